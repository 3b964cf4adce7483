#!/bin/bash
# sgemm split-K reduction in the burst: DSMEM cluster (default) vs red.add (no cluster) -- bench value leg
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for cr in 1 0 1 0; do
  SAGE_SGEMM_CR=$cr timeout 600 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/bench_cr$cr.json 2> gpurun_out/bench_cr$cr.err
  python - $cr <<'PY'
import json,sys
d=json.load(open(f'gpurun_out/bench_cr{sys.argv[1]}.json'))
r=d['roofline']
print('cr',sys.argv[1],'value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'dom',r['kernel'],r['frac'],{k:(v['frac'],v['avg_launch_us']) for k,v in d['rooflines'].items()})
PY
done
