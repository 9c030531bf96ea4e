python build_pb.py
PB_TC_DEBUG=6 python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu 2>&1 | grep "^cta" | tail -148 > gpurun_out/cta.txt
