# build variants (PB_NVCC_DEFS) and time them; usage: VARIANTS="-DA=1|-DA=2" bash scripts/gpu_variants.sh
IFS='|' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  PB_NVCC_DEFS="$v" python build_pb.py --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  for m in ${MODES:-0}; do
    for L in ${LS:-8 16}; do
      echo -n "[$v] dbg $m L $L: "
      PYTHONPATH=. PB_TC_DEBUG=$m timeout -s KILL 60 python scripts/timeline.py --L $L --calls 4 --time 20 2>&1 | grep us_per_call
    done
  done
done
python build_pb.py --force > /dev/null 2>&1
