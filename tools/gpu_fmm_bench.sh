# the FMM solve (bench.py --fmm 4, row f4) at C3 and C2, bench lines into gpurun_out/
mkdir -p gpurun_out
for cfg in C3 C2; do
  timeout 600 python bench.py --fmm 4 --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${cfg}_fmm4.json 2> gpurun_out/bench_${cfg}_fmm4.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_${cfg}_fmm4.json')); print('$cfg', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['kernel'][:90])"
done
