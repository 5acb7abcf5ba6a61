# round-2 final evidence: build, whole -m gpu suite, default bench (JSON line), the launch list of the same
# command under ncu (per-launch times, cold cache), one ncu --set full capture of the A traversal
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
WN_PARITY_REPORT=gpurun_out/parity_floor.json timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; rc=$?
echo "bench rc=$rc"; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
if [ $rc -eq 0 ]; then
  timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_small.json 2> /dev/null && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
  echo "ncu launches rc=$?"
  timeout 600 python tools/prof_one.py C3 2 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:trav_kernel -c 1 \
      -o gpurun_out/trav_full python tools/prof_one.py C3 2 > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
