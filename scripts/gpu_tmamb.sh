nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmamb scripts/tma_mb.cu && timeout -s KILL 120 /tmp/tmamb
