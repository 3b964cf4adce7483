#!/bin/bash
# the N > 1 bench path (one process per rank, p2p fan-out) with both ranks on this pool's one GPU
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
SAGE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --no-cfg1 --no-cpu-baseline > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_n2.json')); f=d['fanout']
print('n_gpus', d['n_gpus'], 'value', d['value'], 'e2e', d['e2e']['value'], 'pcie/step', d['e2e']['h2d_bytes_per_step'])
print(json.dumps(f))" || tail -30 gpurun_out/bench_n2.err
