# consumer rate: L2-hot weights (one copy) vs rotating copies, with the PB_TC_DEBUG knobs
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for shape in "16384 16384 2" "16384 8192 4" "16384 4096 8" "16384 16384 8"; do set -- $shape
 for c in 1 3; do for d in 0 1 2 3; do
  echo "R=$1 K=$2 L=$3 copies=$c dbg=$d $(PYTHONPATH=. PB_TC_DEBUG=$d timeout -s KILL 60 python scripts/timeline.py --R $1 --K $2 --L $3 --copies $c --calls 8 --time 50 --out /tmp/x.npy 2>&1 | grep us_per)"
 done; done; done > gpurun_out/hot_knobs.txt 2>&1
