#!/bin/bash
# ncu --set full of the layer4 3x3 convolution (8 CTAs, 72 K-blocks) of one native forward
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_bf16 -s 45 -c 1 -o gpurun_out/r2_conv_l4 env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > gpurun_out/ncu_conv.log 2>&1
tail -2 gpurun_out/ncu_conv.log
