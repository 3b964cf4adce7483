#!/bin/bash
# BF16 channels-last ResNet-50: the dnn tests, then cfg 3 capacity at 1000 / 2000 per s (bf16) and 1000 (fp32)
mkdir -p gpurun_out/cl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_dnn_gpu.py -x -q 2>&1 | tail -2
for spec in "bf16 1000" "bf16 2000" "fp32 1000"; do
  set -- $spec
  timeout 600 python -m paper_2404_14691_b200.experiments cfg3 --rate $2 --gpus 1 --dtype $1 --out gpurun_out/cl/${1}_r$2 > gpurun_out/cl/log_${1}_$2.txt 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/cl/${1}_r$2/cfg3.json'))
print('$1', $2, {k: d['G1'][k] for k in ('completed','setup_p50_ms','latency_p50_ms','throughput_per_s')})" || tail -5 gpurun_out/cl/log_${1}_$2.txt
done
