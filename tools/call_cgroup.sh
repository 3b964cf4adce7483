#!/bin/bash
# is the container CPU-quota throttled while the bench runs?  (cgroup v2 cpu.max / cpu.stat)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
{
echo "nproc $(nproc)"; echo "cpu.max $(cat /sys/fs/cgroup/cpu.max 2>/dev/null)"; 
echo "before:"; cat /sys/fs/cgroup/cpu.stat 2>/dev/null
timeout 900 python bench.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'median-step', d.get('value_at_median_step'), d['step_ms'], 'e2e', d['e2e']['value'], d['e2e']['step_ms'])"
echo "after:"; cat /sys/fs/cgroup/cpu.stat 2>/dev/null
} 2>&1 | tee gpurun_out/cgroup.txt
