#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q -k sgemm 2>&1 | tail -2
SAGE_SGEMM_CR=0 timeout 120 python tools/prof_gemm.py 40
timeout 120 python tools/prof_gemm.py 40
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DSAGE_GEMM_TRACE tools/gemm_phases.cu -o /tmp/gemm_phases -lcuda && /tmp/gemm_phases
SAGE_SGEMM_CR=0 /tmp/gemm_phases | head -1
