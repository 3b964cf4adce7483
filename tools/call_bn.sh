#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include tools/sgemm_host_cost.cu -o /tmp/shc -lcuda || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include -DSAGE_GEMM_TRACE tools/gemm_phases.cu -o /tmp/gph -lcuda || exit 1
for bn in 0; do echo "== BN=$bn"; SAGE_SGEMM_BN=$bn timeout 60 /tmp/shc | head -1; SAGE_SGEMM_BN=$bn timeout 60 /tmp/gph; done
