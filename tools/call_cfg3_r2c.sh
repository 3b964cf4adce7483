#!/bin/bash
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for r in 4000 4500 5000; do timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate $r --gpus 1 2>&1 | tail -1; done > gpurun_out/cfgs/cfg3_native_r2f.jsonl
python - <<'PY'
import json
for l in open('gpurun_out/cfgs/cfg3_native_r2f.jsonl'):
    try: d=json.loads(l)['cfg3']
    except Exception: print(l[:300]); continue
    g=d['G1']; print(d['workload'][-40:], {k:g.get(k) for k in ('completed','throughput_per_s','setup_p50_ms','setup_p99_ms','latency_p50_ms','wall_s')})
PY
