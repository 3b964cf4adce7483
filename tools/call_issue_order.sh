#!/bin/bash
# issuer order among overdue invocations: e2e A/B (3 runs each) + timeline of one burst
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_issuer_gpu.py tests/test_runtime_gpu.py -q -x 2>&1 | tail -1
for rep in 1 2 3; do
  timeout 600 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/bench_io.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_io.json')); e=d['e2e']; print('e2e', e['value'], e['ms_per_step'], e['roofline']['floor_ms_per_step'], e['roofline']['frac'], 'value', d['value'])"
done
timeout 300 python tools/e2e_timeline.py 10 > gpurun_out/e2e_timeline_io.jsonl 2>&1; tail -1 gpurun_out/e2e_timeline_io.jsonl
