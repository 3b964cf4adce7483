#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for bn in 0 128 64; do for mc in 0 1; do echo "BN=$bn MC=$mc"; SAGE_SGEMM_BN=$bn SAGE_SGEMM_MC=$mc timeout 120 python tools/prof_gemm.py 40; done; done
SAGE_SGEMM_BN=64 timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q -k sgemm 2>&1 | tail -1
SAGE_SGEMM_BN=128 timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q -k sgemm 2>&1 | tail -1
timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q -k sgemm 2>&1 | tail -1
