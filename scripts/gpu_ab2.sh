# interleaved A/B/A/B of compile-time variants ($AB_DEFS, "-" = none) on one box, 8-call graphs
mkdir -p gpurun_out
i=0
for d in $AB_DEFS; do
  if [ "$d" = "-" ]; then defs=""; else defs="${d//,/ }"; fi
  PB_NVCC_DEFS="$defs" python build_pb.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
  cp paper_2003_00822_b200/libpb.so /tmp/libpb_v$i.so; i=$((i+1))
done
for rep in 1 2; do
  i=0
  for d in $AB_DEFS; do
    cp /tmp/libpb_v$i.so paper_2003_00822_b200/libpb.so; touch paper_2003_00822_b200/libpb.so
    echo "== [$rep] $d"; PYTHONPATH=. timeout -s KILL 300 python scripts/sweep_L.py ${SWEEP_ARGS:---L 2 8 16} 2>&1 | tail -1
    i=$((i+1))
  done
done
python build_pb.py --force > /dev/null 2>&1
