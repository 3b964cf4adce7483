#!/bin/bash
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m paper_2404_14691_b200.experiments cfg1 cfg5 cfg4 --out gpurun_out/cfgs > gpurun_out/cfgs/log.txt 2>&1
timeout 600 python -m paper_2404_14691_b200.experiments cfg3 --rate 300 --gpus 1,2,4 --out gpurun_out/cfgs >> gpurun_out/cfgs/log.txt 2>&1
tail -c 3000 gpurun_out/cfgs/log.txt
