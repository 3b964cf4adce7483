#!/bin/bash
# full validation of HEAD: GPU tests, smoke, default bench line
mkdir -p gpurun_out/val
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/val/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/val/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/val/bench.json 2> gpurun_out/val/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/val/bench.json')); e=d['e2e']
print(d['value'], e['value'], e['roofline']['frac'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])"
