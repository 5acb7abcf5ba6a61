# round-2 GPU check: build, the whole -m gpu suite (parity-floor report), a short bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
nproc
WN_PARITY_REPORT=gpurun_out/parity_floor.json timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.log
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['ms_per_step'], d['value'], d['breakdown_ms_per_step'])"
fi
