#!/bin/bash
# conv: coalesced im2col gather -- parity, throughput, per-layer launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_conv_gpu.py tests/test_dnn_gpu.py -x -q > gpurun_out/pytest_conv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_conv.log
tail -2 gpurun_out/pytest_conv.log
timeout 300 python tools/prof_resnet_native.py 8 8 20 | tail -1
timeout 300 python tools/prof_resnet_native.py 8 16 20 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 130 --csv --log-file gpurun_out/resnet_layers4.csv env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
