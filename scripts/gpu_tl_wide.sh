PB_NVCC_DEFS="-DPB_TIMELINE=1" python build_pb.py --force > /dev/null
for B in 1 8; do for L in 2 8; do
echo "== B=$B L=$L"
PB_TC_DEBUG=6 PB_TC_PROF=1 PYTHONPATH=. python scripts/timeline.py --R 16384 --K 4096 --L $L --B $B --calls 1 --out gpurun_out/tl_w.npy > /dev/null 2>&1
python scripts/tl_waits.py gpurun_out/tl_w.npy
done; done
