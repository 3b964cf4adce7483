#!/bin/bash
# compute-sanitizer over the round-2 kernels: land (shuffle fast path), conv (cp.async.mbarrier arrivals,
# short / long kernels), sgemm (3xTF32 split-K cluster); then cfg 4 / cfg 5 re-runs
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SAN="compute-sanitizer --report-api-errors no --error-exitcode 9"
timeout 900 $SAN --tool memcheck --leak-check no python -m pytest tests/test_conv_gpu.py -x -q -k "not 4x56" > gpurun_out/san_conv_mem.log 2>&1; echo "conv memcheck rc=$?"; tail -2 gpurun_out/san_conv_mem.log
timeout 900 $SAN --tool racecheck python -m pytest tests/test_conv_gpu.py -x -q -k "2x14x14x64x64 or 1x7x7x512x512 or 2x28x28x128x512" > gpurun_out/san_conv_race.log 2>&1; echo "conv racecheck rc=$?"; tail -2 gpurun_out/san_conv_race.log
timeout 900 $SAN --tool synccheck python -m pytest tests/test_conv_gpu.py -x -q -k "2x14x14x64x64 or 1x7x7x512x512 or 2x28x28x128x512" > gpurun_out/san_conv_sync.log 2>&1; echo "conv synccheck rc=$?"; tail -2 gpurun_out/san_conv_sync.log
timeout 900 $SAN --tool memcheck --leak-check no python -m pytest tests/test_land_gpu.py tests/test_edges_gpu.py -x -q -k "not two_gib and not hundred and not round_trip" > gpurun_out/san_land_mem.log 2>&1; echo "land memcheck rc=$?"; tail -2 gpurun_out/san_land_mem.log
timeout 900 $SAN --tool memcheck --leak-check no python -m pytest tests/test_bodies_gpu.py -x -q -k "sgemm_tcgen05" > gpurun_out/san_sgemm_mem.log 2>&1; echo "sgemm memcheck rc=$?"; tail -2 gpurun_out/san_sgemm_mem.log
timeout 900 python -m paper_2404_14691_b200.experiments cfg5 cfg4 --out gpurun_out/cfgs > gpurun_out/cfgs/log45.txt 2>&1; echo "cfg45 rc=$?"; tail -c 1500 gpurun_out/cfgs/log45.txt
