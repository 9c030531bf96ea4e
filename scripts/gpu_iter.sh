# one build -> parity -> bench (-> timeline) iteration on the GPU box
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout -s KILL 600 python -m pytest tests -m gpu -x -q ${TEST_ARGS} > gpurun_out/tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/tests.log
timeout -s KILL 300 python bench.py --steps 200 --warmup 10 --no-cpu ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    print("value", d["value"], d["unit"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"])
    for k in ("per_L", "per_kused"):
        if k in d: print(k, [(r.get("L"), r.get("k_used"), round(r["us_per_call"], 1)) for r in d[k]])
except Exception as e:
    print("no json", e)
PY
if [ -n "$TL" ]; then bash scripts/gpu_tl.sh; fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
