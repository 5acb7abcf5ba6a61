mkdir -p gpurun_out
python tools/fmm_one.py C3 4 0.5 32 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fmm_launch_C3_p4.csv python tools/fmm_one.py C3 4 0.5 32 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fmm_eval -c 1 -o gpurun_out/fmm_eval_C3 python tools/fmm_one.py C3 4 0.5 32 > gpurun_out/ncu_eval.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fmm_m2l -c 1 -o gpurun_out/fmm_m2l_C3 python tools/fmm_one.py C3 4 0.5 32 > gpurun_out/ncu_m2l.log 2>&1
ls -la gpurun_out
