#!/bin/bash
# pool + classifier rewrite: parity (ResNet tests) + per-kernel ncu durations + forward throughput
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_dnn_gpu.py -x -q 2>&1 | tail -2 | tee gpurun_out/fc_pytest.txt
timeout 300 python tools/prof_resnet_native.py 8 1 20 | tail -2
timeout 300 python tools/prof_resnet_native.py 8 16 20 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fc_kernel|avgpool|maxpool" -c 8 --csv env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 2>/dev/null | grep -E "fc_kernel|avgpool|maxpool" | awk -F'","' '{print $5, $NF}' | tee gpurun_out/fc_ncu.txt
(cd _ab && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1) && (cd _ab && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxpool" -c 4 --csv env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 2>/dev/null | grep maxpool | awk -F'","' '{print "old", $5, $NF}')
