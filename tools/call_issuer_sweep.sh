#!/bin/bash
# e2e burst length (tools/e2e_timeline.py, 6 bursts) across issuer knobs
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/sweep
for d in 3000 6000 20000; do
  for la in 16 32 64; do
    SAGE_ISSUE_MAX_DEFER_US=$d SAGE_ISSUE_LOOKAHEAD_MB=$la timeout 300 python tools/e2e_timeline.py > gpurun_out/sweep/d${d}_l${la}.jsonl 2>&1
    echo "defer $d lookahead $la $(grep bursts_us gpurun_out/sweep/d${d}_l${la}.jsonl)"
  done
done
