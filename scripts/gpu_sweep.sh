# quick A/B sweep: us/call over L for each env setting in $SWEEP_ENVS (space-separated, "-" = none)
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for e in ${SWEEP_ENVS:--}; do
  if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
  echo "== $envs"
  env $envs PYTHONPATH=. timeout -s KILL 300 python scripts/sweep_L.py ${SWEEP_ARGS} 2>&1 | tail -2
done
if [ -n "$SWEEP_TESTS" ]; then timeout -s KILL 900 python -m pytest $SWEEP_TESTS -m gpu -x -q 2>&1 | tail -3; fi
