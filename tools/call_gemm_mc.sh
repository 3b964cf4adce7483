#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q 2>&1 | tail -3
timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q -k sgemm 2>&1 | tail -1
SAGE_SGEMM_MC=0 timeout 120 python tools/prof_gemm.py 40
SAGE_SGEMM_MC=1 timeout 120 python tools/prof_gemm.py 40
timeout 300 ncu --set full --clock-control none -k regex:sgemm_tf32 -s 5 -c 1 -o gpurun_out/gemm_mc_full -f python tools/prof_gemm.py 8 > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
SAGE_SGEMM_MC=0 timeout 300 ncu --set full --clock-control none -k regex:sgemm_tf32 -s 5 -c 1 -o gpurun_out/gemm_nomc_full -f python tools/prof_gemm.py 8 > gpurun_out/ncu_gemm0.log 2>&1; tail -1 gpurun_out/ncu_gemm0.log
