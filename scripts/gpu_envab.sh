# interleaved A/B/A/B of runtime env settings ($AB_ENVS, "-" = none) on one box, 8-call graphs
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for rep in 1 2; do
  for e in $AB_ENVS; do
    if [ "$e" = "-" ]; then envs=""; else envs="${e//,/ }"; fi
    echo "== [$rep] $e"; env $envs PYTHONPATH=. timeout -s KILL 300 python scripts/sweep_L.py ${SWEEP_ARGS:---L 2 8 16} 2>&1 | tail -1
  done
done
