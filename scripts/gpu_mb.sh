#!/bin/bash
# microbenchmarks behind DESIGN.md §6 (MMA issue rate, TMEM stores, TMA tile streaming, PDL)
mkdir -p gpurun_out
for mb in mxf4_mb mxf4_data_mb tc_mb tma_mb pdl_probe tc_probe_2cta launch_gap; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/$mb scripts/$mb.cu && timeout -s KILL 120 /tmp/$mb > gpurun_out/$mb.txt 2>&1
  echo "$mb rc=$?"
done
