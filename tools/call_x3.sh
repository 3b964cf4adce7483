#!/bin/bash
# 3xTF32 sgemm: operand-reading probe, body parity tests, timing per variant
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tf32_probe.cu -o /tmp/tf32_probe && /tmp/tf32_probe > gpurun_out/tf32_probe.jsonl 2>&1
cat gpurun_out/tf32_probe.jsonl | tail -1
for p in 1 3 4; do for bn in 0 128 64; do
  SAGE_SGEMM_PASSES=$p SAGE_SGEMM_BN=$bn timeout 120 python tools/prof_gemm.py 30 2>&1 | tail -1
done; done | tee gpurun_out/x3_timing.jsonl
timeout 900 python -m pytest tests/test_bodies_gpu.py tests/test_issuer_gpu.py -x -q > gpurun_out/pytest_x3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_x3.log
SAGE_SGEMM_PASSES=4 timeout 600 python -m pytest tests/test_bodies_gpu.py -x -q -k sgemm > gpurun_out/pytest_x3_p4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_x3_p4.log
tail -3 gpurun_out/pytest_x3.log gpurun_out/pytest_x3_p4.log
