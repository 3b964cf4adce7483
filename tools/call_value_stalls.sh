#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for i in 1 2; do
  echo "== nvml sampler on"; timeout 600 python tools/probe_value_stalls.py 200 1 1 2>&1 | tail -30
  echo "== nvml sampler off"; timeout 600 python tools/probe_value_stalls.py 200 1 0 2>&1 | tail -12
done | tee gpurun_out/value_stalls.txt
echo "== full bench"; timeout 900 python bench.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['step_ms'], d['e2e']['step_ms'])"
