#!/bin/bash
# round 2: 3xTF32 fix check, conv kernel parity, instance baselines, runtime replays
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for shp in "128 64 32" "128 64 256" "256 256 1024" "4096 256 4096" "1024 192 96"; do
  timeout 30 python tools/x3_debug.py $shp 2>&1 | tail -1
done | tee gpurun_out/x3_debug.txt
for p in 1 3 4; do for bn in 0 128; do
  SAGE_SGEMM_PASSES=$p SAGE_SGEMM_BN=$bn timeout 60 python tools/prof_gemm.py 30 2>&1 | tail -1
done; done | tee gpurun_out/x3_timing.jsonl
timeout 300 python -m pytest tests/test_conv_gpu.py -x -q > gpurun_out/pytest_conv.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_conv.log
timeout 600 python -m pytest tests/test_bodies_gpu.py tests/test_instances_gpu.py tests/test_runtime_gpu.py tests/test_pressure_gpu.py -q > gpurun_out/pytest_r2a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2a.log
tail -5 gpurun_out/pytest_conv.log; tail -15 gpurun_out/pytest_r2a.log
