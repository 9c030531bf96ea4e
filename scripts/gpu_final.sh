# round-end style evidence run: GPU tests, full bench line, ncu launch list of a short bench run
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/tests_final.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/tests_final.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo "bench rc=$?"; tail -2 gpurun_out/bench_final.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 10 -c 40 --csv \
    --log-file gpurun_out/launches_tc.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"; grep -c bitgemm gpurun_out/launches_tc.csv
