PB_NVCC_DEFS="-DPB_TIMELINE=1" python build_pb.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for L in 2 8; do
PYTHONPATH=. PB_TC_DEBUG=6 timeout -s KILL 120 python scripts/timeline.py --L $L --calls 6 --time 20 --out gpurun_out/tlL$L.npy > gpurun_out/tlL$L.txt 2>&1
python scripts/timeline_an.py gpurun_out/tlL$L.npy >> gpurun_out/tlL$L.txt 2>&1
done
python build_pb.py --force > /dev/null 2>&1
PYTHONPATH=. timeout -s KILL 120 python scripts/timeline.py --L 2 --calls 6 --time 20 --out /tmp/x.npy > gpurun_out/tl_plainL2.txt 2>&1
