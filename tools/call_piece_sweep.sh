#!/bin/bash
# e2e burst length across SAGE_ISSUE_PIECE_MB (0 = whole-load issue), then the issuer tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/piece
for pc in 0 8 16 24; do
  SAGE_ISSUE_PIECE_MB=$pc timeout 300 python tools/e2e_timeline.py > gpurun_out/piece/p${pc}.jsonl 2>&1
  echo "piece $pc $(grep bursts_us gpurun_out/piece/p${pc}.jsonl | cut -c1-200)"
done
timeout 900 python -m pytest tests/test_issuer_gpu.py tests/test_runtime_gpu.py tests/test_land_gpu.py tests/test_pressure_gpu.py -x -q 2>&1 | tail -3
