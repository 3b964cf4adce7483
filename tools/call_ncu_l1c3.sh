#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_bf16 -s 4 -c 1 -o gpurun_out/r2f_conv_l1c3 env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
ls -la gpurun_out/r2f_conv_l1c3.ncu-rep
