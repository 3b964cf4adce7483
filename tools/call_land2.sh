#!/bin/bash
# land: U=8 shuffle fast path, one launch per HBM-resident segment; parity + 1 GiB timing + ncu full capture
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_land_gpu.py tests/test_edges_gpu.py tests/test_fanout_gpu.py tests/test_fanout_p2p_gpu.py tests/test_multigpu_gpu.py tests/test_dedup_gpu.py -x -q > gpurun_out/pytest_land.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_land.log
tail -2 gpurun_out/pytest_land.log
timeout 120 python tools/prof_land_big.py 1 9 | tee gpurun_out/land_big.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:land_kernel -s 128 -c 1 -o gpurun_out/r2_land_1g python tools/prof_land_big.py 1 1 > gpurun_out/ncu_land.log 2>&1
tail -2 gpurun_out/ncu_land.log
