#!/bin/bash
# full round check: tests, smoke, default bench, reference arm, launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cfg1 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'setup', d['setup_p50_ms'], d['setup_p99_ms'], 'launches', d['gpu_launches'])
e=d['e2e']; print('e2e', e['value'], e['ms_per_step'], e['setup_p50_ms'], e['setup_p99_ms'], 'pg', e['pageable_db']['value'])
print('roofline', {k: d['roofline'].get(k) for k in ('kernel','achieved','frac','traffic','limiter')})
print('roofline_land', {k: d['roofline_land'][k] for k in ('achieved','frac','traffic','same_size_d2d_GBps','frac_of_same_size_d2d')})
print('cfg1', d.get('cfg1_sage_vs_fixedgsl', {}).get('p50_setup_ratio_fixedgsl_over_sage'), 'cpu', d.get('cpu_baseline'))
print(open('gpurun_out/bench_ref.json').read())
PY
