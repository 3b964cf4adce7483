#!/bin/bash
# land kernel variants (vectors per lane U, min blocks per SM) at 1 GiB: aligned + misaligned runs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for cfg in "4 4" "8 4" "8 3" "6 4" "8 2"; do set -- $cfg
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2404_14691_b200/csrc -DSAGE_LAND_U=$1 -DSAGE_LAND_MINB=$2 tools/land_micro.cu -o /tmp/lm_$1_$2 || exit 1
echo "U=$1 MINB=$2"; LM_SHORT=1 timeout 60 /tmp/lm_$1_$2 1073741824 | grep -E '"(memcpy|copy_u4|land_u4|land_sh4|land_sh7)"' | grep '"flush":false'
done | tee gpurun_out/land_u_sweep.txt
timeout 120 python tools/prof_land_big.py 1 7 | tee gpurun_out/land_big.json
timeout 600 python -m pytest tests/test_land_gpu.py tests/test_edges_gpu.py -x -q > gpurun_out/pytest_land.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_land.log
tail -2 gpurun_out/pytest_land.log
