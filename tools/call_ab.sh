#!/bin/bash
# A/B of body kernel variants inside the cfg-2 value leg + e2e timeline
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for L in 0 1 2 3 0; do
  SAGE_BODY_LEGACY=$L timeout 300 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/ab_$L.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_$L.json')); print('legacy=$L', d['value'], d['ms_per_step'], d['setup_p50_ms'], 'e2e', d['e2e']['value'])"
done
timeout 300 python tools/e2e_timeline.py > gpurun_out/e2e_timeline.jsonl 2>&1; tail -1 gpurun_out/e2e_timeline.jsonl
