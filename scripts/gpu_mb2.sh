# tensor-core rate microbenchmarks (scratch; results in gpurun_out/)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mxf4_mb scripts/mxf4_mb.cu && timeout 120 /tmp/mxf4_mb > gpurun_out/mxf4_mb.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc_mb scripts/tc_mb.cu && timeout 120 /tmp/tc_mb > gpurun_out/tc_mb.txt 2>&1
cat gpurun_out/mxf4_mb.txt gpurun_out/tc_mb.txt
