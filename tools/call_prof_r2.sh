#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_dedup_gpu.py tests/test_fanout_bcast_gpu.py tests/test_bench_n2_gpu.py -q > gpurun_out/pytest_r2d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2d.log
timeout 120 python tools/prof_land_big.py 1 5 > gpurun_out/land_big.json 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:land_kernel -s 128 -c 1 -o gpurun_out/r2_land_big python tools/prof_land_big.py 1 1 > gpurun_out/ncu_land.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sgemm_tf32 -s 2 -c 1 -o gpurun_out/r2_sgemm_x3 python tools/prof_gemm.py 3 > gpurun_out/ncu_sgemm.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_bf16 -s 29 -c 1 -o gpurun_out/r2_conv_l3c2 env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > gpurun_out/ncu_conv.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2_resnet_launches.csv env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
tail -3 gpurun_out/pytest_r2d.log; cat gpurun_out/land_big.json; ls -la gpurun_out/*.ncu-rep
