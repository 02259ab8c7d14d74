#!/bin/bash
mkdir -p gpurun_out
nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/host_probe.cu -o /tmp/host_probe -lpthread 2>/dev/null
nproc; lscpu | grep -i "model name\|socket\|numa node(s)\|^CPU(s)"
timeout 300 /tmp/host_probe 2>&1 | tee gpurun_out/host_probe.log
cat /sys/kernel/mm/transparent_hugepage/enabled
timeout 600 python tools/dropin_timing.py 2>&1 | tee gpurun_out/dropin_timing.log
