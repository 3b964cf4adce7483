#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python tools/prof_submit.py > gpurun_out/prof_submit.txt 2>&1
timeout 300 python tools/prof_cfg2.py value > gpurun_out/prof_cfg2_value.txt 2>&1
head -5 gpurun_out/prof_submit.txt; head -3 gpurun_out/prof_cfg2_value.txt
