#!/bin/bash
# CTA-pair (cta_group::2) 3xTF32 sgemm: parity tests, timing pair vs single, phase trace
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q -k sgemm > gpurun_out/pytest_pair.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pair.log
tail -3 gpurun_out/pytest_pair.log
for pr in 1 0; do
  SAGE_SGEMM_PAIR=$pr timeout 120 python tools/prof_gemm.py 30 2>&1 | tail -1 | sed "s/^/pair=$pr /"
done | tee gpurun_out/pair_timing.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DSAGE_GEMM_TRACE tools/gemm_phases.cu -o /tmp/gemm_phases -lcuda > /dev/null 2>&1
for pr in 1 0; do echo "== pair=$pr"; SAGE_SGEMM_PAIR=$pr timeout 60 /tmp/gemm_phases; done | tee gpurun_out/pair_phases.txt
