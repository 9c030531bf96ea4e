# ncu evidence for the tensor-engine kernel (one GPU): a full-set capture of one launch at
# the bench configuration (C5 16384x16384, L=8, a=16, B=1) and the launch list of a short bench run
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
PYTHONPATH=. timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bitgemm_tc -s 2 -c 1 \
    -f -o gpurun_out/prof_tc python scripts/timeline.py --L 8 --calls 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_tc.csv python bench.py --steps 16 --warmup 8 --no-sweep --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"; tail -3 gpurun_out/ncu_launch.log
