#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2404_14691_b200/csrc tools/land_micro.cu -o /tmp/land_micro
timeout 120 /tmp/land_micro > gpurun_out/land_micro2.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/land_micro2.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l); continue
    print(d['kernel'], d['flush'], d['mean_us'], d['GBps_mean'], d['checksum_ok'])
PY
