nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tcmb scripts/tc_mb.cu && timeout 120 /tmp/tcmb
