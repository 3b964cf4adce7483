"""Cross-process fan-out with peer landing (fanout.PeerFanout), two real
rank processes on one GPU: each function's home rank lands its segment over
PCIe and hands the pages + an interprocess "landed" event to the other rank,
whose cold leader lands them with ONE `land` launch reading the home's
segment (NVLink on a multi-GPU box; here the same device) and verifies the
checksum.  Homes are split (sgemm, stencil -> rank 0; spmv -> rank 1) so both
directions run; two cold bursts each, results checked against the oracle in
each rank."""
import json
import os
import socket
import subprocess
import sys
import uuid
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

RANK = r"""
import json, os, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch.distributed as dist
rank, world, port, job = int(sys.argv[2]), 2, sys.argv[3], sys.argv[4]
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
from oracle import oracle as O
from paper_2404_14691_b200 import device as D
from paper_2404_14691_b200.fanout import PeerFanout
from paper_2404_14691_b200.parboil import cfg2_functions
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
table, data = cfg2_functions(scale=4)
names = [sorted(table)[k % 3] for k in range(12)]
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=3, function_data=data)
box = PeerFanout(rank, world, table, homes={"sgemm": 0, "stencil": 0, "spmv": 1}, job=job, barrier=dist.barrier)
sim.dataplane.box = box
sim.dataplane.pin_host_store()
out, ok = [], True
for rep in range(2):
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
    dist.barrier()
    invs = sim.submit_many(names)
    sim.drain()
    box.reap()
    for i in invs:
        fd = data[i.spec.name]
        lay = fd.layout
        seg, want = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        x = fd.input
        if fd.body == "sgemm":
            m, n, k = fd.args
            ref = O.sgemm_ref(seg[:m * k * 4].view(np.float32).reshape(m, k), x.view(np.float32).reshape(n, k).T)
            good = np.allclose(i.result.view(np.float32).reshape(m, n), ref, rtol=1e-3, atol=1e-4 * np.abs(ref).max())
        elif fd.body == "stencil":
            nx, ny, nz, bits = fd.args
            ref = O.stencil_ref(seg.view(np.float32)[:nx * ny * nz].reshape(nz, ny, nx),
                                x.view(np.float32).reshape(nz, ny, nx), float(np.int32(bits).view(np.float32)))
            good = np.allclose(i.result.view(np.float32).reshape(nz, ny, nx), ref, rtol=1e-3, atol=1e-5)
        else:
            rows, nnz, o_rp, o_col, o_val = fd.args
            ref = O.spmv_ref(seg[o_rp:o_rp + 4 * (rows + 1)].view(np.int32), seg[o_col:o_col + 4 * nnz].view(np.int32),
                             seg[o_val:o_val + 4 * nnz].view(np.float32), x.view(np.float32))
            good = np.allclose(i.result.view(np.float32)[:rows], ref, rtol=1e-3, atol=1e-4)
        ok = ok and bool(good) and i.outcome == "completed" and i.ro_checksum in (None, want)
        out.append([i.spec.name, i.warmth.label(), i.ro_source, int(i.measured.get("pcie_bytes", 0)),
                    int(i.measured.get("nvlink_bytes", 0))])
stats = box.stats()
sim.dataplane.unpin_host_store()
dist.barrier()
box.close()
sim.close()
dist.destroy_process_group()
print("RANK " + json.dumps({"rank": rank, "ok": ok, "invs": out, "stats": stats}))
"""


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_peer_fanout_two_processes(built):
    from conftest import gpu_available
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    port, job = str(_free_port()), uuid.uuid4().hex[:8]
    procs = [subprocess.Popen([sys.executable, "-c", RANK, str(ROOT), str(r), port, job], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True, env=dict(os.environ)) for r in range(2)]
    res = []
    for p in procs:
        out, err = p.communicate(timeout=600)
        assert p.returncode == 0, err[-3000:]
        res.append(json.loads([ln for ln in out.splitlines() if ln.startswith("RANK ")][-1][len("RANK "):]))
    homes = {"sgemm": 0, "stencil": 0, "spmv": 1}
    for r in res:
        assert r["ok"], r
        leaders = [inv for inv in r["invs"] if inv[1] == "Cold"]
        assert len(leaders) == 6                                   # 3 functions x 2 bursts
        for name, _, src, pcie, nvl in leaders:
            if homes[name] == r["rank"]:
                assert src == "pcie" and nvl == 0
            else:
                assert src == "nvlink" and nvl > 0                 # landed from the home's pages
        assert r["stats"]["received"] == 2 * sum(h != r["rank"] for h in homes.values())
        assert r["stats"]["sent"] == 2 * sum(h == r["rank"] for h in homes.values())
