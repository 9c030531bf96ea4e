# us/call under the PB_TC_KNOB profiling knobs (uninstrumented build): 0 normal, 1 no A stores,
# 2 no MMA, 3 neither, 4 converters skip LDS/ALU too (pipeline skeleton)
python build_pb.py > /dev/null 2>&1
for shape in ${SHAPES:-16384,16384,2 16384,16384,8 8192,2048,8}; do set -- ${shape//,/ }
 for c in ${COPIES:-2}; do for d in ${KNOBS:-0 1 2 3 4}; do
  echo "R=$1 K=$2 L=$3 copies=$c knob=$d $(PYTHONPATH=. PB_TC_KNOB=$d timeout -s KILL 60 python scripts/timeline.py --R $1 --K $2 --L $3 --copies $c --calls 8 --time 50 --out /tmp/x.npy 2>&1 | grep us_per)"
 done; done; done > gpurun_out/knobs${TAG}.txt 2>&1
cat gpurun_out/knobs${TAG}.txt
