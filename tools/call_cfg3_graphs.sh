#!/bin/bash
# cfg 3 (BF16 channels-last) capacity at 2000/s offered vs graphs per landed segment
mkdir -p gpurun_out/gps
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for n in 2 4 8 12; do
  SAGE_DNN_GRAPHS_PER_SEGMENT=$n timeout 600 python -m paper_2404_14691_b200.experiments cfg3 --rate 2000 --gpus 1 --dtype bf16 --out gpurun_out/gps/g$n > gpurun_out/gps/log_$n.txt 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/gps/g$n/cfg3.json'))
print('graphs $n', {k: d['G1'][k] for k in ('completed','latency_p50_ms','throughput_per_s','graph_captures')})" || tail -5 gpurun_out/gps/log_$n.txt
done
