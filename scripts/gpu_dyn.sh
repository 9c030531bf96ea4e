# dynamic tail share sweep (PB_TC_DYN = % of units claimed one at a time after the static split)
python build_pb.py > /dev/null 2>&1
for rep in 1 2; do for shape in ${SHAPES:-16384,16384,2 16384,16384,8 16384,16384,16}; do set -- ${shape//,/ }
 for d in ${DYNS:-0 2 5 10}; do
  echo "R=$1 K=$2 L=$3 dyn=$d $(PYTHONPATH=. PB_TC_DYN=$d timeout -s KILL 60 python scripts/timeline.py --R $1 --K $2 --L $3 --copies 3 --calls 8 --time 50 --out /tmp/x.npy 2>&1 | grep us_per)"
 done; done; done > gpurun_out/dyn.txt 2>&1
cat gpurun_out/dyn.txt
