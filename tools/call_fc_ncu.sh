#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"fc_kernel|avgpool" -c 2 -o gpurun_out/fc_full -f env SAGE_NET_GRAPHS=0 python tools/prof_resnet_native.py 8 1 1 > /dev/null 2>&1
ncu -i gpurun_out/fc_full.ncu-rep --page details --csv > gpurun_out/fc_full_details.csv 2>&1; wc -l gpurun_out/fc_full_details.csv
