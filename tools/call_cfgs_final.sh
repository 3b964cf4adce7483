#!/bin/bash
# final round-2 configuration runs: cfg1 rows, cfg3 (1 GPU rates + logical G=2/4), cfg2 Poisson peak
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m paper_2404_14691_b200.experiments cfg1 --out gpurun_out/cfgs > gpurun_out/cfgs/log1.txt 2>&1; echo "cfg1 rc=$?"
for r in 2000 3500; do timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate $r --gpus 1 2>&1 | tail -1; done > gpurun_out/cfgs/cfg3_final.jsonl
timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate 2000 --gpus 2,4 2>&1 | tail -1 > gpurun_out/cfgs/cfg3_final_logical.jsonl
echo "cfg3 done"; tail -c 600 gpurun_out/cfgs/cfg3_final_logical.jsonl
