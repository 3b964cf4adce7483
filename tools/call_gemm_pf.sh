#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for pf in 0 4 8 16 32; do echo "PF=$pf"; SAGE_SGEMM_PF=$pf timeout 120 python tools/prof_gemm.py 40; done
timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q -k sgemm 2>&1 | tail -1
