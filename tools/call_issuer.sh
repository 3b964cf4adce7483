#!/bin/bash
# issuer A/B: GPU tests (issuer on), bench legs under issuer off / lookahead sweep, e2e timeline
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for cfg in "SAGE_ISSUER=0" "SAGE_ISSUE_LOOKAHEAD_MB=8" "SAGE_ISSUE_LOOKAHEAD_MB=16" "SAGE_ISSUE_LOOKAHEAD_MB=24" "SAGE_ISSUE_LOOKAHEAD_MB=48" "SAGE_ISSUE_LOOKAHEAD_MB=1000"; do
  env $cfg timeout 300 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/iss.json 2>gpurun_out/iss.err
  python -c "import json,sys; d=json.load(open('gpurun_out/iss.json')); e=d['e2e']; print(sys.argv[1], 'value', d['value'], d['ms_per_step'], d['setup_p50_ms'], 'e2e', e['value'], e['ms_per_step'], e['setup_p50_ms'], e['setup_p99_ms'], 'pg', e['pageable_db']['value'])" "$cfg" || tail -5 gpurun_out/iss.err
done
timeout 300 python tools/e2e_timeline.py > gpurun_out/e2e_timeline_iss.jsonl 2>&1; tail -1 gpurun_out/e2e_timeline_iss.jsonl
