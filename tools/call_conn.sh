#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/conn
for c in 8 32 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 300 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/conn/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/conn/b.json')); print('conn=$c bench value', d['value'], 'e2e', d['e2e']['value'])"
done
for c in 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 600 python -m paper_2404_14691_b200.experiments cfg3 --rate 1200 --gpus 1 --out gpurun_out/conn/c$c > /dev/null 2>&1
  python -c "import json; d=json.load(open('gpurun_out/conn/c$c/cfg3.json'))['G1']; print('conn=$c cfg3@1200', d['throughput_per_s'], d['setup_p50_ms'])"
done
