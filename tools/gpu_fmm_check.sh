# FMM: GPU parity tests, timings at C2/C3, and a launch list of one C3 application (p = 4, θ_f = 0.5)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fmm.py -x -q 2>&1 | tail -3
timeout 300 python tools/fmm_bench.py C2 2>&1 | head -6
timeout 600 python tools/fmm_bench.py C3 2>&1 | tee gpurun_out/fmm_bench_C3.txt | head -18
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fmm_launch_C3_p4.csv python tools/fmm_one.py C3 4 0.5 32 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/fmm_launch_C3_p4.csv 2>&1 | head -8
