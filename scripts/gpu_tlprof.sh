# per-warp wait profiles (instrumented build) at the L values in $TL_LS
mkdir -p gpurun_out
PB_NVCC_DEFS="-DPB_TIMELINE=1" python build_pb.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for L in ${TL_LS:-2 8}; do
  PYTHONPATH=. PB_TC_DEBUG=6 PB_TC_PROF=1 timeout -s KILL 120 python scripts/timeline.py --L $L --calls 2 ${TL_ARGS} --out gpurun_out/tlp$L.npy > gpurun_out/tlp$L.txt 2>&1
  echo "== L=$L rc=$?"; python scripts/timeline_an.py gpurun_out/tlp$L.npy | grep -v "^chunk0\|^first pass"
done
