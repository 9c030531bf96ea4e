python build_pb.py > /dev/null
python scripts/c4_prof.py
for d in 1 2 3; do echo "PB_TC_DEBUG=$d"; PB_TC_DEBUG=$d python scripts/c4_prof.py; done
