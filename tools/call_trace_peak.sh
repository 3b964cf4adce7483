#!/bin/bash
mkdir -p gpurun_out/peak
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_trace_gpu.py -x -q 2>&1 | tail -5
timeout 900 python -m paper_2404_14691_b200.experiments peak --workload cfg3 --out gpurun_out/peak/cfg3 > gpurun_out/peak/cfg3.log 2>&1; python -c "import json; d=json.load(open('gpurun_out/peak/cfg3/peak.json')); print('cfg3 peak', d['peak_rate_per_s'], d['trajectory'])" || tail -5 gpurun_out/peak/cfg3.log
timeout 900 python -m paper_2404_14691_b200.experiments peak --workload cfg2 --out gpurun_out/peak/cfg2 > gpurun_out/peak/cfg2.log 2>&1; python -c "import json; d=json.load(open('gpurun_out/peak/cfg2/peak.json')); print('cfg2 peak', d['peak_rate_per_s'], d['trajectory'])" || tail -5 gpurun_out/peak/cfg2.log
