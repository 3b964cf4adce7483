#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 240 python -m pytest tests/test_conv_gpu.py tests/test_dnn_gpu.py -x -q > gpurun_out/pytest_s2d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s2d.log; tail -2 gpurun_out/pytest_s2d.log
grep -q "rc=0" gpurun_out/pytest_s2d.log || exit 1
for i in 1 2; do timeout 120 python tools/prof_resnet_native.py 8 16 20 | tail -1; done; timeout 120 python tools/stress.py 40 16 2 | tail -1
timeout 120 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 130 --csv --log-file gpurun_out/resnet_layers12.csv env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
