#!/bin/bash
# issuer tiebreak (larger return first among equal H2D-D2H balance): e2e A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for tb in 0 1 0 1; do
  SAGE_ISSUE_BIG_RETURN_FIRST=$tb timeout 600 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/bench_tb$tb.json 2> gpurun_out/bench_tb$tb.err
  python - $tb <<'PY'
import json,sys
d=json.load(open(f'gpurun_out/bench_tb{sys.argv[1]}.json'))
e=d['e2e']
print('tb',sys.argv[1],'e2e',e['value'],e['ms_per_step'],'floor',e['roofline']['floor_ms_per_step'],e['roofline']['frac'],'setup',e['setup_p50_ms'],e['setup_p99_ms'],'value',d['value'])
PY
done
SAGE_ISSUE_BIG_RETURN_FIRST=1 timeout 300 python tools/e2e_timeline.py > gpurun_out/e2e_timeline_tb.jsonl 2>&1; tail -1 gpurun_out/e2e_timeline_tb.jsonl
