#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for cfg in "SAGE_ISSUE_LOOKAHEAD_MB=32 SAGE_ISSUE_MAX_DEFER_US=3000" "SAGE_ISSUE_LOOKAHEAD_MB=16 SAGE_ISSUE_MAX_DEFER_US=3000" "SAGE_ISSUE_LOOKAHEAD_MB=64 SAGE_ISSUE_MAX_DEFER_US=3000" "SAGE_ISSUE_LOOKAHEAD_MB=32 SAGE_ISSUE_MAX_DEFER_US=1000" "SAGE_ISSUE_LOOKAHEAD_MB=32 SAGE_ISSUE_MAX_DEFER_US=10000" "SAGE_ISSUE_LOOKAHEAD_MB=32 SAGE_ISSUE_MAX_DEFER_US=3000"; do
  env $cfg timeout 300 python bench.py --no-cfg1 --no-cpu-baseline --steps 10 > gpurun_out/sw.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/sw.json')); e=d['e2e']; print(sys.argv[1], e['value'], e['ms_per_step'], e['setup_p50_ms'], e['roofline']['frac'])" "$cfg"
done
