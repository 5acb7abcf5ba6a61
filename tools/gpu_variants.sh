# step timing (40 iterations, graph) of every built variant on ${CFG:-C3}
for v in $(ls paper_2405_16634_b200/exp); do
  echo -n "$v: "; WN_LIB=paper_2405_16634_b200/exp/$v/libwn.so timeout 300 python tools/step_bench.py ${CFG:-C3} 2>&1 | tail -1
done
