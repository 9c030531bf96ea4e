nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tcpf4 scripts/tc_probe_f4.cu && timeout 60 /tmp/tcpf4; echo rc=$?
