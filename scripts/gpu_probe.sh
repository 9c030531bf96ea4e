nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tcp scripts/tc_probe.cu && timeout 60 /tmp/tcp; echo "rc=$?"
