#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python tools/prof_host.py 2>&1 | tee gpurun_out/prof_host.txt
timeout 300 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/bq.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bq.json')); print('value', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'])"
