set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench.cu && /tmp/mb
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 200 --warmup 10 --no-sweep --no-cpu > gpurun_out/bench_nosweep.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
