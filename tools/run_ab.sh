python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo -n "hilbert: "; timeout 300 python tools/trav_bench.py C3 20 2>&1 | grep "ms per"
echo -n "morton:  "; WN_EXP_NOHILBERT=1 timeout 300 python tools/trav_bench.py C3 20 2>&1 | grep "ms per"
echo -n "hilbert: "; timeout 300 python tools/trav_bench.py C3 20 2>&1 | grep "ms per"
echo -n "morton:  "; WN_EXP_NOHILBERT=1 timeout 300 python tools/trav_bench.py C3 20 2>&1 | grep "ms per"
