"""Stress / determinism check (not a benchmark).
1. The native ResNet-50 program: one reference forward, then R rounds of S
   concurrent forwards on S streams (different graph instances, device-side
   frames) -- every output must be bit-identical to the reference (the conv
   kernels have no atomics: any difference is a race).
2. B cold bursts of the scaled cfg-2 mix through the public API with every
   landed checksum and every output checked against the CPU oracle.
python tools/stress.py [rounds] [streams] [bursts]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2404_14691_b200 import _lib, dnn  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
streams = int(sys.argv[2]) if len(sys.argv) > 2 else 16
bursts = int(sys.argv[3]) if len(sys.argv) > 3 else 20
t0 = time.time()
_lib.init(n_gpus=1, pool_bytes=32 << 30)
spec, fd = dnn.resnet50_native(batch=8, seed=0)
h = dnn.native_handle(fd)
seg = D.pool_alloc(0, fd.layout.seg_bytes, _lib.CLASS_READ_ONLY)
op = D.load(0, seg.dptr, fd.db, fd.layout)
op.wait()
op.release()
in_b = (fd.input_bytes + 16 + 255) // 256 * 256
wr, bodies = [], []
for _ in range(streams):
    w = D.pool_alloc(0, spec.writable_bytes, _lib.CLASS_WRITABLE)
    up = D.load(0, w.dptr, fd.input, None)
    up.wait()
    up.release()
    wr.append(w)
    bodies.append(D.body_desc(_lib.BODY_RESNET50, ro=seg.dptr, ro_bytes=fd.layout.seg_bytes, inp=w.dptr,
                              inp_bytes=(fd.input_bytes + 15) // 16 * 16, out=w.dptr + in_b,
                              out_bytes=fd.out_bytes, args=(h, 8)))
slots = [D.Slot(0) for _ in range(streams)]
b, e = slots[0].launch(bodies[0])
e.sync()
ref = D.read_device(0, wr[0].dptr + in_b, fd.out_bytes).copy()
b.release(); e.release()
mism = 0
for r in range(rounds):
    evs = [slots[s].launch(bodies[s]) for s in range(streams)]
    for bb, ee in evs:
        ee.sync()
    for s in range(streams):
        got = D.read_device(0, wr[s].dptr + in_b, fd.out_bytes)
        mism += int(not np.array_equal(got, ref))
    for bb, ee in evs:
        bb.release(); ee.release()
for s in slots:
    s.release()
for w in wr:
    w.free()
seg.free()
_lib.shutdown()
res = {"resnet_forwards": rounds * streams, "resnet_mismatches": mism}

from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402
table, data = cfg2_functions(scale=4)
names = [sorted(table)[k % 3] for k in range(48)]
want = {}
for n, f in data.items():
    lay = f.layout
    want[n] = O.land_c(f.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
bad = 0
with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=2, function_data=data) as sim:
    outs = {}
    for k in range(bursts):
        for r in list(sim.sharing.residents.values()):
            sim.sharing.evict(r)
        invs = sim.submit_many(names)
        sim.drain()
        for i in invs:
            n = i.spec.name
            if i.outcome != "completed" or i.ro_checksum not in (None, want[n][1]):
                bad += 1
                continue
            key = (n, k == 0)
            if n not in outs:
                outs[n] = i.result.copy()
                f = data[n]
                seg_b = want[n][0]
                if f.body == "sgemm":
                    m, nn, kk = f.args
                    r_ = O.sgemm_ref(seg_b[:m * kk * 4].view(np.float32).reshape(m, kk),
                                     f.input.view(np.float32).reshape(nn, kk).T)
                    g_ = i.result.view(np.float32).reshape(m, nn)
                    bad += int(not np.allclose(g_, r_, rtol=1e-3, atol=1e-4 * np.abs(r_).max()))
            elif data[n].body != "sgemm":   # stencil / spmv: deterministic, bit-identical run to run
                bad += int(not np.array_equal(i.result, outs[n]))
res.update({"cfg2_bursts": bursts, "cfg2_invocations": bursts * len(names), "cfg2_bad": bad,
            "elapsed_s": round(time.time() - t0, 1)})
print(json.dumps(res))
