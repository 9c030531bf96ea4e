python build_pb.py
PB_TC_DEBUG=6 timeout -s KILL 120 python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu 2>&1 | grep "^cta" | tail -148 > gpurun_out/cta.txt
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bitgemm -c 2 timeout -s KILL 120 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu 2>&1 | grep gpu__time
