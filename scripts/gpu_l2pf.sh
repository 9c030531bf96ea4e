# L2 prefetch depth sweep (PB_TC_L2PF tiles beyond the ring's first fill)
python build_pb.py > /dev/null 2>&1
for rep in 1 2; do for shape in ${SHAPES:-16384,16384,2 16384,16384,4 16384,16384,8 8192,2048,8 2048,16384,8}; do set -- ${shape//,/ }
 for d in ${PFS:-0 8 16 32}; do
  echo "R=$1 K=$2 L=$3 l2pf=$d $(PYTHONPATH=. PB_TC_L2PF=$d timeout -s KILL 60 python scripts/timeline.py --R $1 --K $2 --L $3 --copies 3 --calls 8 --time 50 --out /tmp/x.npy 2>&1 | grep us_per)"
 done; done; done > gpurun_out/l2pf.txt 2>&1
cat gpurun_out/l2pf.txt
