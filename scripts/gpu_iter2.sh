# iteration: sweep (plain build), parity tests, then the instrumented timeline at L=8
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
PYTHONPATH=. timeout -s KILL 300 python scripts/sweep_L.py ${SWEEP_ARGS:---L 1 2 4 8 16} 2>&1 | tail -2
timeout -s KILL 900 python -m pytest ${ITER_TESTS:-tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_layers.py} -m gpu -x -q 2>&1 | tail -3
TL_LS="${TL_LS:-8}" bash scripts/gpu_tlprof.sh 2>&1 | grep -i "tail\|prologue\|mend\|mma0\|warp  [0-3]"
python build_pb.py --force > /dev/null 2>&1
