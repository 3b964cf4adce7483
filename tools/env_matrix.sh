#!/bin/bash
# bench (no cfg1 / cpu baseline) under stream-topology knobs; one line per combo
for combo in "$@"; do
  env $combo timeout 300 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/m.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/m.json')); e=d['e2e']; print(sys.argv[1], 'value', d['value'], 'steps', d.get('step_ms'), 'setup', d['setup_p50_ms'], 'e2e', e['value'], e.get('step_ms'), 'pg', e['pageable_db']['value'], 'e2e_setup', e['setup_p50_ms'])" "$combo"
done
