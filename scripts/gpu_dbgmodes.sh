python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for m in 0 1 2 3; do
  for L in 8 16; do
    echo -n "dbg $m L $L: "
    PYTHONPATH=. PB_TC_DEBUG=$m timeout -s KILL 60 python scripts/timeline.py --L $L --calls 4 --time 20 2>&1 | grep us_per_call
  done
done
