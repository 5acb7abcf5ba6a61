# A/B of the traversal dispatch: persistent warps (heaviest-first / schedule order) vs one block per 128 queries
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for c in C3 C4 C5; do
  echo -n "$c persist-heavy: "; timeout 300 python tools/step_bench.py $c 2>&1 | tail -1
  echo -n "$c persist-sched: "; WN_GROUP_ORDER=sched timeout 300 python tools/step_bench.py $c 2>&1 | tail -1
  echo -n "$c blocks       : "; WN_PERSIST=0 timeout 300 python tools/step_bench.py $c 2>&1 | tail -1
done
