#!/bin/bash
# per-layer launch list of one native ResNet-50 forward (ops launched one by one) + concurrent throughput
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python tools/prof_resnet_native.py 8 8 20 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 130 --csv --log-file gpurun_out/resnet_layers.csv env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
wc -l gpurun_out/resnet_layers.csv
