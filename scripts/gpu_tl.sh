# per-CTA timeline: builds with the instrumentation compiled in (-DPB_TIMELINE=1), restores the plain build
PB_NVCC_DEFS="-DPB_TIMELINE=1" python build_pb.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
PYTHONPATH=. PB_TC_DEBUG=6 timeout -s KILL 120 python scripts/timeline.py ${TL_ARGS} --out gpurun_out/tl${TL_TAG}.npy > gpurun_out/tl${TL_TAG}.txt 2>&1
echo rc=$?; tail -3 gpurun_out/tl${TL_TAG}.txt
python scripts/timeline_an.py gpurun_out/tl${TL_TAG}.npy
python build_pb.py --force > /dev/null 2>&1
