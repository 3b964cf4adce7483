#!/bin/bash
# round-2 configuration sweeps (cfg1 rows, cfg3 native vs cuDNN, cfg4 density, cfg5 contention)
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m paper_2404_14691_b200.experiments cfg1 --out gpurun_out/cfgs > gpurun_out/cfgs/log.txt 2>&1
for r in 1000 2000 2500; do timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate $r --gpus 1 2>&1 | tail -1; done > gpurun_out/cfgs/cfg3_native.jsonl
for r in 1000 2000; do timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --engine torch --rate $r --gpus 1 2>&1 | tail -1; done > gpurun_out/cfgs/cfg3_torch.jsonl
timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate 1000 --gpus 2,4 2>&1 | tail -1 > gpurun_out/cfgs/cfg3_native_logical.jsonl
timeout 900 python -m paper_2404_14691_b200.experiments cfg5 cfg4 --out gpurun_out/cfgs >> gpurun_out/cfgs/log.txt 2>&1
tail -c 2500 gpurun_out/cfgs/log.txt
