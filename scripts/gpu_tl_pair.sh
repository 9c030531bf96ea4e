# per-CTA timelines at L=2 and L=8 (instrumented build), plus uninstrumented us/call
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || exit 1
for L in 2 8; do PYTHONPATH=. timeout -s KILL 60 python scripts/timeline.py --L $L --calls 4 --time 50 --out /tmp/x.npy 2>&1 | grep us_per; done
PB_NVCC_DEFS="-DPB_TIMELINE=1" python build_pb.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for L in 2 8; do
  PYTHONPATH=. PB_TC_DEBUG=6 timeout -s KILL 120 python scripts/timeline.py --L $L --calls 4 --out gpurun_out/tlL$L.npy > gpurun_out/tlL$L.txt 2>&1
  echo "== L=$L rc=$?"; python scripts/timeline_an.py gpurun_out/tlL$L.npy
done
