python build_pb.py
python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
tail -3 gpurun_out/bench_tc.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_tc.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bitgemm_tc -s 4 -c 1 -o gpurun_out/prof_tc python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_tc.log 2>&1
tail -3 gpurun_out/ncu_tc.log
