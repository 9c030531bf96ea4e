PB_NVCC_DEFS="-DPB_TIMELINE=1" python build_pb.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
PYTHONPATH=. PB_TC_DEBUG=6 PB_TC_PROF=1 timeout -s KILL 120 python scripts/timeline.py ${TL_ARGS} --out gpurun_out/prof.npy > /dev/null 2>&1
python scripts/timeline_an.py gpurun_out/prof.npy | tail -14
python build_pb.py --force > /dev/null 2>&1
