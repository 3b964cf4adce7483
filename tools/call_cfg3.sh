#!/bin/bash
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for r in 300 600; do
timeout 600 python -m paper_2404_14691_b200.experiments cfg3 --rate $r --gpus 1,2 --out gpurun_out/cfgs/r$r > gpurun_out/cfgs/log3_$r.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/cfgs/r$r/cfg3.json'))
for g in ('G1','G2'): print($r, g, {k: d[g][k] for k in ('completed','setup_p50_ms','setup_p99_ms','throughput_per_s','graph_captures')})" || tail -5 gpurun_out/cfgs/log3_$r.txt
done
