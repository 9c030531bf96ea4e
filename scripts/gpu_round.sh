# evidence run: build, smoke, GPU tests, bench line (stdout JSON to gpurun_out/bench.json)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/tests.log
timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err; head -c 3000 gpurun_out/bench.json
