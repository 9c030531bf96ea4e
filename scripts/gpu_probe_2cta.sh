nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tcp2 scripts/tc_probe_2cta.cu && timeout 60 /tmp/tcp2; echo rc=$?
