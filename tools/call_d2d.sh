#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_land_gpu.py tests/test_edges_gpu.py tests/test_runtime_gpu.py tests/test_issuer_gpu.py tests/test_bodies_gpu.py -x -q > gpurun_out/pytest_d2d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_d2d.log; tail -2 gpurun_out/pytest_d2d.log
for i in 1 2; do
  timeout 600 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/bench_d2d.json 2> gpurun_out/bench_d2d.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_d2d.json')); r=d['roofline']
print('value',d['value'],d['ms_per_step'],'e2e',d['e2e']['value'],'dom',r['kernel'],r['frac'],{k:(v['frac'],v['avg_launch_us'],v['launches']) for k,v in d['rooflines'].items()})"
done
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 3000 --csv --log-file gpurun_out/launches_d2d.csv python bench.py --steps 2 --warmup 3 --no-cfg1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_d2d.csv | tail -9
