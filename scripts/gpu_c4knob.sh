python build_pb.py > /dev/null 2>&1
for k in ${KNOBS:-0 256}; do echo "knob=$k: $(PB_TC_KNOB=$k PYTHONPATH=. N=${N:-300} B=128 timeout -s KILL 600 python scripts/c4_repeat.py 2>&1 | tail -1)"; done
