# end-of-round evidence: full GPU tests, smoke, default bench line, launch list and ncu captures
# (C5 bench kernel, the local-mode small layer, the LSTM with SMEM-resident A), summarised
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/r02c_launches.csv python bench.py --steps 16 --warmup 8 --no-sweep --no-cpu --no-compare --no-lstm --no-extras > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
PYTHONPATH=. timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bitgemm_tc -s 2 -c 1 \
    -f -o gpurun_out/r02c_tc_c5 python scripts/timeline.py --L 8 --calls 2 > gpurun_out/ncu_c5.log 2>&1
echo "c5 rc=$?"
PYTHONPATH=. timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bitgemm_tc -s 2 -c 1 \
    -f -o gpurun_out/r02c_tc_small python scripts/timeline.py --R 8192 --K 2048 --L 8 --calls 2 > gpurun_out/ncu_small.log 2>&1
echo "small rc=$?"
CFGS="8,1" PYTHONPATH=. timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lstm_persist -c 1 \
    -f -o gpurun_out/r02c_lstm_l8 python scripts/lstm_quick.py > gpurun_out/ncu_lstm.log 2>&1
echo "lstm rc=$?"
for r in r02c_tc_c5 r02c_tc_small r02c_lstm_l8; do
  [ -f gpurun_out/$r.ncu-rep ] && python scripts/ncu_summary.py gpurun_out/$r.ncu-rep gpurun_out/${r}_full.txt > /dev/null 2>&1
done
python scripts/ncu_summary.py --launches gpurun_out/r02c_launches.csv gpurun_out/r02c_launches.txt > /dev/null 2>&1
ls gpurun_out
