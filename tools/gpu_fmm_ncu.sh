# ncu --set full of the FMM leaf pass (k_fmm_eval) and the grouped M2L at C3 (p = 4, θ_f = 0.5, leaf 32)
mkdir -p gpurun_out
python tools/fmm_one.py C3 4 0.5 32 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_fmm_eval -c 1 -o gpurun_out/fmm_eval_C3_v2 python tools/fmm_one.py C3 4 0.5 32 > gpurun_out/ncu_eval.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fmm_m2l_grp -c 1 -o gpurun_out/fmm_m2l_C3_v2 python tools/fmm_one.py C3 4 0.5 32 > gpurun_out/ncu_m2l.log 2>&1
ls gpurun_out
