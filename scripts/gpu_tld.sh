# L=2 timelines under the PB_TC_KNOB profiling knobs (0 normal, 2 no MMA, 3 no MMA + no A stores),
# weights rotating over ${COPIES:-2} copies (1: L2-hot)
PB_NVCC_DEFS="-DPB_TIMELINE=1" python build_pb.py --force > /dev/null 2>&1
for d in ${KNOBS:-0 2 3}; do PYTHONPATH=. PB_TC_DEBUG=6 PB_TC_PROF=${PROF:-0} PB_TC_KNOB=$d timeout -s KILL 120 python scripts/timeline.py --L ${L:-2} --copies ${COPIES:-2} --calls 4 --out gpurun_out/tld$d.npy > /dev/null 2>&1; python scripts/timeline_an.py gpurun_out/tld$d.npy > gpurun_out/tld${TAG}$d.txt 2>&1; done
