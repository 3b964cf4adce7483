#!/bin/bash
# sgemm epilogue change + bench value leg under compute-concurrency gates
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_bodies_gpu.py -x -q -k sgemm > gpurun_out/pytest_sg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sg.log
tail -2 gpurun_out/pytest_sg.log
timeout 120 python tools/prof_gemm.py 30 2>&1 | tail -1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DSAGE_GEMM_TRACE tools/gemm_phases.cu -o /tmp/gemm_phases -lcuda > /dev/null 2>&1
timeout 60 /tmp/gemm_phases | tee gpurun_out/phases_epi.txt
for cc in 0 1 2; do
  timeout 600 python bench.py --no-cfg1 --no-cpu-baseline --compute-concurrency $cc > gpurun_out/bench_cc$cc.json 2> gpurun_out/bench_cc$cc.err
  python - $cc <<'PY'
import json,sys
d=json.load(open(f'gpurun_out/bench_cc{sys.argv[1]}.json'))
r=d['roofline']
print('cc',sys.argv[1],'value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],d['e2e']['ms_per_step'],'dom',r['kernel'],r['frac'],'iso',r.get('isolated',{}).get('frac'),{k:(v['frac'],v['avg_launch_us']) for k,v in d['rooflines'].items()})
PY
done
