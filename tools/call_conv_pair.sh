#!/bin/bash
# conv CTA pair (SAGE_CONV_PAIR=1): parity, throughput (short timeouts: a hang must not eat the call)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SAGE_CONV_PAIR=1 timeout 90 python -m pytest tests/test_conv_gpu.py -x -q > gpurun_out/pytest_cpair.log 2>&1; echo "pytest conv rc=$?" >> gpurun_out/pytest_cpair.log; tail -3 gpurun_out/pytest_cpair.log
grep -q "rc=0" gpurun_out/pytest_cpair.log || exit 1
SAGE_CONV_PAIR=1 timeout 240 python -m pytest tests/test_dnn_gpu.py -x -q > gpurun_out/pytest_cpair_dnn.log 2>&1; echo "pytest dnn rc=$?" >> gpurun_out/pytest_cpair_dnn.log; tail -2 gpurun_out/pytest_cpair_dnn.log
for p in 0 1; do echo "pair=$p $(SAGE_CONV_PAIR=$p timeout 90 python tools/prof_resnet_native.py 8 16 20 | tail -1)"; done | tee gpurun_out/conv_pair.txt
SAGE_CONV_PAIR=1 timeout 120 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 130 --csv --log-file gpurun_out/resnet_layers5.csv env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
