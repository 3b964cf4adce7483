#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for s in 1 4; do timeout 120 python tools/prof_resnet_native.py 8 $s 20 2>&1 | tail -1; done | tee gpurun_out/resnet_native_body2.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/resnet_native_launches2.csv python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_bf16 -s 46 -c 1 -o gpurun_out/conv_l4c3 python tools/prof_resnet_native.py 8 1 1 > gpurun_out/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_bf16 -s 29 -c 1 -o gpurun_out/conv_l3c2 python tools/prof_resnet_native.py 8 1 1 > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out/*.ncu-rep
