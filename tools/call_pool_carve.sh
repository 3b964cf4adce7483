#!/bin/bash
# chunk-carved private segments: full GPU suite, cfg5 first-burst probe, cfg3 overload, cfg4
mkdir -p gpurun_out/cfgs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_cfg5.py 128 2; timeout 300 python tools/probe_cfg5.py 512 2
for r in 3500 5000; do timeout 300 python -m paper_2404_14691_b200.experiments cfg3 --dtype bf16 --rate $r --gpus 1 2>&1 | tail -1 | cut -c1-420; done
