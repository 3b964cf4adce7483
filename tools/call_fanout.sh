#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_fanout_gpu.py -x -q > gpurun_out/pytest_fanout.log 2>&1; tail -15 gpurun_out/pytest_fanout.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
mkdir -p gpurun_out/cfgs; timeout 600 python -m paper_2404_14691_b200.experiments cfg3 --rate 300 --gpus 1,2 --out gpurun_out/cfgs > gpurun_out/cfgs/log3.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/cfgs/cfg3.json'))
for g in ('G1','G2'): print(g, {k: d[g][k] for k in ('completed','setup_p50_ms','setup_p99_ms','throughput_per_s','graph_captures')})"
