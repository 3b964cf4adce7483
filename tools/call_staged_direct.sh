#!/bin/bash
# staged identity no-verify loads: DMA straight into dst (default) vs through the land (SAGE_STAGED_LAND=1)
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_land_gpu.py tests/test_issuer_gpu.py -x -q -m gpu 2>&1 | tail -4
run() { timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate $1 --gpus 1 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())['cfg3']; g=d['G1']
print('$2', '$1', g['completed'], g['throughput_per_s'], g['setup_p50_ms'], g['setup_p99_ms'], g['wall_s'])"; }
for r in 3500 4000 4500; do
  SAGE_STAGED_LAND=1 run $r land
  run $r direct
  SAGE_STAGED_LAND=1 run $r land
  run $r direct
done | tee gpurun_out/cfgs/staged_direct_ab.txt
