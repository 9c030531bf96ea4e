python build_pb.py
timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | grep -E "passed|failed|^E " | head -8
for m in 0 3; do echo "mode $m"; PB_TC_DEBUG=$m timeout -s KILL 120 python bench.py --steps 100 --warmup 5 --no-sweep --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['roofline']['avg_launch_us'],1), round(d['roofline']['achieved']))"; done
PB_TC_PROF=1 timeout -s KILL 120 python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu 2>&1 | grep "^warp" | tail -11 | sort -k2,2n
