python build_pb.py
timeout -s KILL 600 python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
tail -2 gpurun_out/bench_tc.err
