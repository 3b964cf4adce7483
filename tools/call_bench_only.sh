#!/bin/bash
# the default bench line + the reference arm, for box-to-box spread
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench_rep.json 2> gpurun_out/bench_rep.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_rep_ref.json 2>/dev/null
python - <<'PY'
import json, socket
d = json.load(open('gpurun_out/bench_rep.json')); r = json.load(open('gpurun_out/bench_rep_ref.json'))
e = d['e2e']
print(json.dumps({"host": socket.gethostname(), "value": d['value'], "e2e": e['value'], "e2e_floor_frac": e['roofline']['frac'],
                  "floor_ms": e['roofline']['floor_ms_per_step'], "setup_p50_ms": e['setup_p50_ms'], "setup_p99_ms": e['setup_p99_ms'],
                  "reference_arm": r['value'], "e2e_over_reference": round(e['value'] / r['value'], 1),
                  "cfg1_ratio": d['cfg1_sage_vs_fixedgsl']['p50_setup_ratio_fixedgsl_over_sage'],
                  "roofline": {k: d['roofline'].get(k) for k in ('kernel', 'frac')}, "clocks": d['clocks']}))
PY
