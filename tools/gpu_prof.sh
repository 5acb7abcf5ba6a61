# full ncu capture of selected kernels of a short C3 workload (usage: KREGEX=... bash tools/gpu_prof.sh)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_one.py C3 ${ITERS:-1} > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-trav_kernel}" -s ${SKIP:-0} -c ${COUNT:-1} \
   -o gpurun_out/${OUT:-prof} python tools/prof_one.py C3 ${ITERS:-1} > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
