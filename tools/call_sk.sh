#!/bin/bash
# stream-K 3xTF32 sgemm: parity, isolated timing, bench value leg with / without
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_bodies_gpu.py tests/test_conv_gpu.py -x -q > gpurun_out/pytest_sk.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sk.log; tail -2 gpurun_out/pytest_sk.log
for sk in 0 1; do SAGE_SGEMM_SK=$sk timeout 120 python tools/prof_gemm.py 30 | tail -1 | sed "s/^/sk=$sk /"; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include tools/sgemm_host_cost.cu -o /tmp/shc -lcuda || exit 1
for sk in 0 1; do echo "sk=$sk"; SAGE_SGEMM_SK=$sk timeout 60 /tmp/shc | head -1; done
for sk in 0 1; do
  SAGE_SGEMM_SK=$sk timeout 600 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/bench_sk$sk.json 2> gpurun_out/bench_sk$sk.err
  python - $sk <<'PY'
import json,sys
d=json.load(open(f'gpurun_out/bench_sk{sys.argv[1]}.json'))
r=d['roofline']
print('sk',sys.argv[1],'value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'dom',r['kernel'],r['frac'],'iso',r.get('isolated',{}).get('frac'),{k:(v['frac'],v['avg_launch_us']) for k,v in d['rooflines'].items()})
PY
done
