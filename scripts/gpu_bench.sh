set -x
python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bitgemv -s 6 -c 1 -o gpurun_out/prof_gemv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu2.log 2>&1
tail -5 gpurun_out/ncu2.log
