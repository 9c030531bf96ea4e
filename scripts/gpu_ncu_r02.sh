# round-2 ncu evidence (one GPU): full captures of the C5 bench kernel, the C4 batch-128 wide
# kernel and the persistent LSTM kernel, plus the launch list of a short bench run
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
PYTHONPATH=. timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bitgemm_tc -s 2 -c 1 \
    -f -o gpurun_out/r02_tc_c5 python scripts/timeline.py --L 8 --calls 2 > gpurun_out/ncu_c5.log 2>&1
echo "c5 rc=$?"
PYTHONPATH=. timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bitgemm_tc -s 2 -c 1 \
    -f -o gpurun_out/r02_tc_c4b128 python scripts/timeline.py --R 16384 --K 4096 --B 128 --L 8 --calls 2 > gpurun_out/ncu_c4.log 2>&1
echo "c4 rc=$?"
H=2048 T=32 L=4 B=1 PYTHONPATH=. timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lstm_persist -c 1 \
    -f -o gpurun_out/r02_lstm python scripts/lstm_one.py > gpurun_out/ncu_lstm.log 2>&1
echo "lstm rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 16 --warmup 8 --no-sweep --no-cpu --no-compare --no-lstm --no-extras > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
