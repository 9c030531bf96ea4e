# one build -> parity -> bench iteration on the GPU box
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/tests.log
timeout -s KILL 300 python bench.py --steps 200 --warmup 10 --no-cpu ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    print("value", d["value"], d["unit"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"])
    for k in ("per_L", "per_kused"):
        if k in d: print(k, json.dumps(d[k])[:900])
except Exception as e:
    print("no json", e)
PY
