mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2404_14691_b200/csrc tools/land_micro.cu -o /tmp/land_micro
timeout 120 /tmp/land_micro > gpurun_out/land_micro.jsonl 2>&1
timeout 120 /tmp/land_micro 104857600 >> gpurun_out/land_micro.jsonl 2>&1
timeout 120 python tools/probe_bidir.py > gpurun_out/bidir.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:land_kernel -s 17 -c 1 -o gpurun_out/land_full -f python tools/prof_land.py 3 > gpurun_out/ncu_land.log 2>&1
cat gpurun_out/land_micro.jsonl gpurun_out/bidir.json; tail -3 gpurun_out/ncu_land.log
