#!/bin/bash
# sgemm: host enqueue cost, API costs, phase trace (1-CTA kernel, all-warp split-K reduction)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 120 python tools/prof_gemm.py 30 2>&1 | tail -1
timeout 60 ./tools/api_cost | tee gpurun_out/api_cost.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DSAGE_GEMM_TRACE tools/gemm_phases.cu -o /tmp/gemm_phases2 -lcuda || exit 1
timeout 60 /tmp/gemm_phases2 | tee gpurun_out/phases_epi.txt
