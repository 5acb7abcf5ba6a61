for v in $(ls paper_2405_16634_b200/exp); do
  echo -n "$v: "; WN_LIB=paper_2405_16634_b200/exp/$v/libwn.so timeout 300 python tools/step_bench.py C3 2>&1 | grep "iterate40"
done
