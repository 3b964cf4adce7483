#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 120 python tools/probe_h2d_mix.py > gpurun_out/probe_h2d_mix.json 2>&1; cat gpurun_out/probe_h2d_mix.json
for cfg in "SAGE_LAND_TMA=0" "SAGE_LAND_TMA=1"; do
  env $cfg timeout 300 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/lt.json 2>gpurun_out/lt.err
  python -c "import json,sys; d=json.load(open('gpurun_out/lt.json')); e=d['e2e']; r=d['roofline']; print(sys.argv[1], 'land', r['achieved'], r['frac'], r['avg_launch_us'], 'd2d', r['same_size_d2d_GBps'], 'value', d['value'], 'e2e', e['value'])" "$cfg" || tail -5 gpurun_out/lt.err
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:land_tma_kernel -s 1 -c 1 -o gpurun_out/land_tma_full -f python tools/prof_land.py 3 > gpurun_out/ncu_land_tma.log 2>&1; tail -2 gpurun_out/ncu_land_tma.log
