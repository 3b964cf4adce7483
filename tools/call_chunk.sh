#!/bin/bash
# staged-load chunk size A/B (3 runs each): e2e, setup latency, pageable leg
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for rep in 1 2 3; do for c in 8 16 32; do
  timeout 600 python bench.py --no-cfg1 --no-cpu-baseline --chunk-mb $c > gpurun_out/bench_ch$c.json 2> gpurun_out/bench_ch$c.err
  python - $c <<'PY'
import json,sys
d=json.load(open(f'gpurun_out/bench_ch{sys.argv[1]}.json'))
e=d['e2e']
print('chunk',sys.argv[1],'e2e',e['value'],e['ms_per_step'],'frac',e['roofline']['frac'],'setup',e['setup_p50_ms'],e['setup_p99_ms'],
      'pageable',e['pageable_db']['value'],e['pageable_db']['setup_p50_ms'],'value',d['value'])
PY
done; done | tee gpurun_out/chunk_ab.txt
