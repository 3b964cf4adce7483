#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for b in 8; do for s in 1 4 8; do timeout 120 python tools/prof_resnet_native.py $b $s 20 2>&1 | tail -1; done; done | tee gpurun_out/resnet_native_body.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/resnet_native_launches.csv python tools/prof_resnet_native.py 8 1 2 > /dev/null 2>&1
for r in 1000 2000 4000; do timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate $r --gpus 1 2>&1 | tail -1; done | tee gpurun_out/cfg3_native.jsonl
timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --engine torch --rate 2000 --gpus 1 2>&1 | tail -1 | tee gpurun_out/cfg3_torch.jsonl
