# validation run: build, smoke, GPU tests, full bench line
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/tests.log
timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
