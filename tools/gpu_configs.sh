# bench lines of every BASELINE config (C3 = the driver's default line), then the launch list of the default
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in C3 C1 C2 C4 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 $( [ $c != C3 ] && echo --no-cpu-baseline ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['ms_per_step'],2), round(d['value'],1), d['roofline']['frac'], d['clocks'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
