#!/bin/bash
# host profile (cProfile) of cfg 3 above capacity
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -m cProfile -o gpurun_out/cfg3_5000.prof -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate 5000 --gpus 1 2>&1 | tail -1 | cut -c1-300
timeout 300 python -m cProfile -o gpurun_out/cfg3_5000b.prof -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate 5000 --gpus 1 2>&1 | tail -1 | cut -c1-300
