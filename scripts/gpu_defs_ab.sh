# A/B of compile-time knobs: for each "DEFS" in $AB_DEFS ("-" = none) rebuild and sweep
mkdir -p gpurun_out
for d in $AB_DEFS; do
  if [ "$d" = "-" ]; then defs=""; else defs="${d//,/ }"; fi
  PB_NVCC_DEFS="$defs" python build_pb.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
  echo "== $defs"
  PYTHONPATH=. timeout -s KILL 300 python scripts/sweep_L.py ${SWEEP_ARGS:---L 2 4 8 16} 2>&1 | tail -1
done
python build_pb.py --force > /dev/null 2>&1
