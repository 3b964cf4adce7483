#!/bin/bash
# ncu --set full of the final kernels: 3xTF32 sgemm, spmv, conv (layer4 3x3 long-K, layer1 1x1 short-K)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sgemm_tf32 -s 2 -c 1 -o gpurun_out/r2f_sgemm python tools/prof_gemm.py 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmv4 -s 2 -c 1 -o gpurun_out/r2f_spmv python tools/prof_spmv.py 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_bf16 -s 45 -c 1 -o gpurun_out/r2f_conv_l4 env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_bf16 -s 3 -c 1 -o gpurun_out/r2f_conv_l1 env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
