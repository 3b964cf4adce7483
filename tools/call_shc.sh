#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include tools/sgemm_host_cost.cu -o /tmp/shc -lcuda || exit 1
timeout 60 /tmp/shc | tee gpurun_out/sgemm_host_cost.txt
