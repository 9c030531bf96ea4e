# timeline prologue experiments: env settings in $EXP_ENVS
mkdir -p gpurun_out
PB_NVCC_DEFS="-DPB_TIMELINE=1" python build_pb.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for e in $EXP_ENVS; do
  echo "== $e"
  env $e PYTHONPATH=. timeout -s KILL 120 python scripts/timeline.py --L ${EXP_L:-8} --calls 2 --out /tmp/tle.npy > /dev/null 2>&1
  python scripts/timeline_an.py /tmp/tle.npy | grep -A1 "prologue call 1" ; python scripts/timeline_an.py /tmp/tle.npy | grep -A7 "^call 1" | grep "mma0\|bready\|end "
done
