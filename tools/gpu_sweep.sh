mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py --grid 256 --steps 5 --warmup 3 > gpurun_out/grid256.json 2> gpurun_out/grid.err; echo "grid rc=$?"
cat gpurun_out/grid256.json | head -c 600; echo
WN_SWEEP=1 WN_SWEEP_OUT=gpurun_out/c4_sweep.json timeout 1500 python -m pytest tests/test_gpu_c4_sweep.py -q > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"; tail -5 gpurun_out/sweep.log
