mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_one.py C3 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trav_kernel|moments_up" -s 3 -c 4 \
   -o gpurun_out/prof_trav python tools/prof_one.py C3 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python tools/prof_one.py C3 2 > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
