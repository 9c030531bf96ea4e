#!/bin/bash
# microbenchmarks + a quick bench line (scratch runs; results land in gpurun_out/)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mxf4_mb scripts/mxf4_mb.cu && timeout 120 /tmp/mxf4_mb > gpurun_out/mxf4_mb.txt 2>&1
python build_pb.py > /dev/null
timeout 600 python bench.py --steps 200 --warmup 10 --no-sweep --no-compare --no-lstm --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
