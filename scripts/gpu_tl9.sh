python build_pb.py > gpurun_out/build.log 2>&1 || exit 1
for m in 6 9; do
  PYTHONPATH=. PB_TC_DEBUG=$m timeout -s KILL 60 python scripts/timeline.py --calls 4 --out gpurun_out/tl$m.npy > /dev/null 2>&1
  echo "== dbg $m"; python scripts/timeline_an.py gpurun_out/tl$m.npy | grep -E "prologue call 3|^call 3" -A6 | grep -E "prologue|mma0|end "
done
