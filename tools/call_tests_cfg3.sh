#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for r in 300 1000; do
  timeout 600 python -m paper_2404_14691_b200.experiments cfg3 --rate $r --gpus 1 > gpurun_out/cfg3_r$r.json 2> gpurun_out/cfg3_r$r.err
  python -c "import json; d=json.load(open('gpurun_out/cfg3_r$r.json'))['cfg3']; print($r, {k: d['G1'][k] for k in ('completed','setup_p50_ms','setup_p99_ms','throughput_per_s')})" || tail -5 gpurun_out/cfg3_r$r.err
done
SAGE_DNN_GRAPHS=0 timeout 600 python -m paper_2404_14691_b200.experiments cfg3 --rate 300 --gpus 1 > gpurun_out/cfg3_eager.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/cfg3_eager.json'))['cfg3']; print('eager 300', {k: d['G1'][k] for k in ('completed','setup_p50_ms','setup_p99_ms','throughput_per_s')})"
timeout 300 python tools/prof_submit.py > gpurun_out/prof_submit.txt 2>&1; head -60 gpurun_out/prof_submit.txt
