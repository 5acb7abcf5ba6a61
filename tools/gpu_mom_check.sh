# moment-build check: parity tests touching the moments, step timing of the built variants, ncu of the moment kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_order1.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py -x -q -k "moments or one_iteration or iteration_from or first_iteration or deterministic or graph or order1 or stats or rescale or table5 or edge or tiny or maximum" > gpurun_out/pytest_mom.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_mom.log
for v in $(ls paper_2405_16634_b200/exp); do echo -n "$v: "; WN_LIB=paper_2405_16634_b200/exp/$v/libwn.so timeout 300 python tools/step_bench.py C3 2>&1 | tail -1; done
WN_LIB=paper_2405_16634_b200/exp/base/libwn.so timeout 300 python tools/step_bench.py C5 2>&1 | tail -1
if [ "${NCU:-1}" = "1" ]; then
timeout 300 python tools/prof_one.py C3 1 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mom_" -c 3 -o gpurun_out/${OUT:-mom_prof} python tools/prof_one.py C3 1 > gpurun_out/ncu_mom.log 2>&1; echo "ncu rc=$?"
fi
