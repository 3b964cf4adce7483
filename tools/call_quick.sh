#!/bin/bash
# quick GPU iteration: build, body + land tests, short bench, launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cfg1 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_quick.csv python bench.py --steps 2 --warmup 3 --no-cfg1 --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench_quick.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_quick.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'setup', d['setup_p50_ms'], d['setup_p99_ms'])
print('e2e', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['setup_p50_ms'], 'pg', d['e2e']['pageable_db']['value'])
print('roofline', {k: d['roofline'][k] for k in ('achieved','frac','traffic','same_size_d2d_GBps','frac_of_same_size_d2d')})
for k,v in d['rooflines'].items(): print(k, v['achieved'], v['frac'], v['avg_launch_us'], v['share_of_kernel_time'])
PY
python tools/launch_summary.py gpurun_out/launches_quick.csv
