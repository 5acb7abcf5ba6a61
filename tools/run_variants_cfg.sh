# usage: CFG=C2 bash tools/run_variants_cfg.sh — step_bench of every built variant on one config
for v in $(ls paper_2405_16634_b200/exp); do
  echo -n "$v ${CFG:-C3}: "; WN_LIB=paper_2405_16634_b200/exp/$v/libwn.so timeout 300 python tools/step_bench.py ${CFG:-C3} 2>&1 | grep "iterate40"
done
