# one full ncu capture (with source) of the C5 kernel at L=${L:-2}: per-SASS stall samples
mkdir -p gpurun_out
python build_pb.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
PYTHONPATH=. timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bitgemm_tc -s 2 -c 1 \
    -f -o gpurun_out/src_L${L:-2} python scripts/timeline.py --L ${L:-2} --calls 2 > gpurun_out/ncu_src.log 2>&1
echo "rc=$?"
ncu -i gpurun_out/src_L${L:-2}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_L${L:-2}_sass.csv 2>&1
echo "src rc=$?"; ls -la gpurun_out/
