mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_one.py ${CFG:-C3} ${ITERS:-2} > gpurun_out/p.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/prof_one.py ${CFG:-C3} ${ITERS:-2} > gpurun_out/ncu_launches.log 2>&1
echo rc=$?
