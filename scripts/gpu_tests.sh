set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --durations=8 2>&1 | tail -25
