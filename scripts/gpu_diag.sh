# diagnosis: microbenchmarks, consumer-path knobs (PB_TC_DEBUG 1/2/3) at L=2/8, timelines L=2/8
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
bash scripts/gpu_mb.sh
for L in 2 4 8; do for d in 0 1 2 3; do
  echo "L=$L dbg=$d $(PYTHONPATH=. PB_TC_DEBUG=$d timeout -s KILL 60 python scripts/timeline.py --L $L --calls 8 --time 50 --out /tmp/x.npy 2>&1 | grep us_per)"
done; done > gpurun_out/dbg_knobs.txt 2>&1
for L in 2 8; do TL_TAG=_L$L TL_ARGS="--L $L --calls 4" bash scripts/gpu_tl.sh > gpurun_out/tl_an_L$L.txt 2>&1; done
