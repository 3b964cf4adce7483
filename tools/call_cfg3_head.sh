#!/bin/bash
# cfg3 capacity at HEAD: Poisson arrivals of ResNet-50 BF16 batch-8 invocations, 1 GPU
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for r in 3500 4000 4500 5000; do
  timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate $r --gpus 1 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())['cfg3']; g=d['G1']
print(json.dumps({'offered_per_s': $r, 'completed': g['completed'], 'served_per_s': g['throughput_per_s'], 'setup_p50_ms': g['setup_p50_ms'], 'setup_p99_ms': g['setup_p99_ms'], 'wall_s': g['wall_s']}))"
done | tee gpurun_out/cfgs/cfg3_head.jsonl
