python build_pb.py
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "streamk" 2>&1 | tail -25
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
