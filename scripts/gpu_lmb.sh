nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lmb scripts/launch_mb.cu && /tmp/lmb
