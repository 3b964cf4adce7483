#!/bin/bash
# cfg3 A/B on one box: the tree in _ab (previous commit) vs this tree
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
run() { timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate $1 --gpus 1 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())['cfg3']; g=d['G1']
print('$2', d['workload'][-40:], g['completed'], g['throughput_per_s'], g['setup_p50_ms'], g['setup_p99_ms'], g['wall_s'])"; }
for r in 3000 2500; do
  (cd _ab && run $r old)
  run $r new
done | tee gpurun_out/cfgs/cfg3_ab.txt
(cd _ab && timeout 300 python tools/prof_resnet_native.py 8 16 20 | tail -1)
timeout 300 python tools/prof_resnet_native.py 8 16 20 | tail -1
