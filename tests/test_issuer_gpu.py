"""The invocation issuer (csrc/invoke.cu) changes only WHEN an admitted
invocation's DAG is enqueued, never what it computes.  The same cold cfg-2
burst (scaled down), run once with the issuer off (enqueue at admission) and
once on, must produce identical warmth classes, RO-load sources, landed
checksums, input checksums and results (bit-identical but for sgemm split-K
summation order), each equal to the CPU
oracle; followers must still compute only after their leader's segment landed.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2404_14691_b200 import device as D
from paper_2404_14691_b200.functions import Stage
from paper_2404_14691_b200.parboil import cfg2_functions
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
table, data = cfg2_functions(scale=4)
names = [sorted(table)[k % 3] for k in range(24)]
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=3, function_data=data)
pls = []
for n in names:
    pb = D.PinnedBuffer(data[n].input_bytes)
    pb.view()[:] = data[n].input
    pls.append(pb)
sim.dataplane.pin_host_store()
sim.dataplane.verify_inputs = True   # the input checksums are compared across runs
out, res = [], []
for rep in range(2):
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
    invs = sim.submit_many(names, payloads=pls)
    sim.drain()
    land = {}
    for i in invs:
        if i.ro_landed_us is not None and i.warmth.label() != "Stage1Hot":
            land[i.spec.name] = i.ro_landed_us
    for i in invs:
        assert i.outcome == "completed", i.fail_reason
        c = i.stages[Stage.COMPUTE][0]
        assert c >= land[i.spec.name], ("follower computed before its leader's RO landed", i.id)
        out.append([i.spec.name, i.warmth.label(), i.ro_source, i.ro_checksum, i.input_checksum])
        res.append(np.array(i.result, copy=True))
sim.dataplane.unpin_host_store()
sim.close()
np.savez(sys.argv[2], *res)
print("RESULT " + json.dumps(out))
"""


def run_child(issuer: str, tmp, piece_mb: str = "0"):
    import numpy as np
    env = dict(os.environ, SAGE_ISSUER=issuer, SAGE_ISSUE_PIECE_MB=piece_mb)
    npz = str(tmp / f"issuer{issuer}_p{piece_mb}.npz")
    res = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), npz], capture_output=True, text=True, env=env,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    z = np.load(npz)
    return json.loads(line[len("RESULT "):]), [z[f"arr_{k}"] for k in range(len(z.files))]


def test_issuer_changes_order_not_results(built, tmp_path):
    """Metadata and every landed / input checksum identical; stencil and spmv
    outputs bit-identical; sgemm outputs equal up to the fp32 summation order
    of the tcgen05 kernel's split-K red.add epilogue (not run-to-run fixed)."""
    import numpy as np
    from conftest import gpu_available
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    off, r_off = run_child("0", tmp_path)
    on, r_on = run_child("1", tmp_path)
    assert len(off) == len(on) == 48
    assert off == on
    for meta, a, b in zip(off, r_off, r_on):
        if meta[0] == "sgemm":
            np.testing.assert_allclose(a.view(np.float32), b.view(np.float32), rtol=1e-5, atol=1e-4)
        else:
            assert np.array_equal(a, b), meta


def test_piecewise_cold_loads_change_order_not_results(built, tmp_path):
    """SAGE_ISSUE_PIECE_MB=1: every staged cold load is enqueued one ring
    chunk at a time, alternating with the followers of landed segments; the
    same metadata, checksums and results as enqueueing at admission, and
    followers still compute after their leader's segment landed (checked in
    the child)."""
    import numpy as np
    from conftest import gpu_available
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    off, r_off = run_child("0", tmp_path)
    pc, r_pc = run_child("1", tmp_path, piece_mb="1")
    assert off == pc
    for meta, a, b in zip(off, r_off, r_pc):
        if meta[0] == "sgemm":
            np.testing.assert_allclose(a.view(np.float32), b.view(np.float32), rtol=1e-5, atol=1e-4)
        else:
            assert np.array_equal(a, b), meta


def test_issuer_results_match_oracle(built):
    """Every returned output equals the numpy body on the oracle-landed bytes
    (one invocation per function, issuer on)."""
    import numpy as np

    from oracle import oracle as O
    from paper_2404_14691_b200 import device as D
    from paper_2404_14691_b200.parboil import cfg2_functions
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
    from conftest import gpu_available
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    table, data = cfg2_functions(scale=8)
    names = [sorted(table)[k % 3] for k in range(12)]
    with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=5, function_data=data) as sim:
        invs = sim.submit_many(names)
        sim.drain()
        for i in invs:
            fd = data[i.spec.name]
            lay = fd.layout
            seg, want_sum = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
            assert i.ro_checksum is None or i.ro_checksum == want_sum
            x = fd.input
            if fd.body == "sgemm":
                m, n, k = fd.args
                want = O.sgemm_ref(seg[:m * k * 4].view(np.float32).reshape(m, k), x.view(np.float32).reshape(n, k).T)
                got = i.result.view(np.float32).reshape(m, n)
                np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-4 * np.abs(want).max())
            elif fd.body == "stencil":
                nx, ny, nz, bits = fd.args
                beta = float(np.int32(bits).view(np.float32))
                want = O.stencil_ref(seg.view(np.float32)[:nx * ny * nz].reshape(nz, ny, nx),
                                     x.view(np.float32).reshape(nz, ny, nx), beta)
                np.testing.assert_allclose(i.result.view(np.float32).reshape(nz, ny, nx), want, rtol=1e-3, atol=1e-5)
            else:
                rows, nnz, o_rp, o_col, o_val = fd.args
                want = O.spmv_ref(seg[o_rp:o_rp + 4 * (rows + 1)].view(np.int32),
                                  seg[o_col:o_col + 4 * nnz].view(np.int32), seg[o_val:o_val + 4 * nnz].view(np.float32),
                                  x.view(np.float32))
                np.testing.assert_allclose(i.result.view(np.float32)[:rows], want, rtol=1e-3, atol=1e-4)


def test_issuer_backlog_beyond_scan_window():
    """A burst far larger than the issuer's pick window (256 waiting
    invocations): two functions, so the window fills with followers while a
    leader waits further back; every invocation completes, each function's
    segment crosses PCIe once, every landed copy is the oracle's."""
    code = r"""
import sys
sys.path.insert(0, sys.argv[1])
from oracle import oracle as O
from paper_2404_14691_b200.experiments import synthetic_function
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
a, da = synthetic_function("fa", 8, 1, 0.0625, tensors=7)
b, db = synthetic_function("fb", 24, 1, 0.0625, tensors=9)
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {"fa": a, "fb": b}, seed=5,
                 function_data={"fa": da, "fb": db}, copy_results=False)
try:
    names = ["fa"] * 400 + ["fb"] * 400
    invs = sim.submit_many(names)
    sim.drain()
    assert all(i.outcome == "completed" for i in invs), [i.fail_reason for i in invs if i.outcome != "completed"][:3]
    for fn, fd in (("fa", da), ("fb", db)):
        lay = fd.layout
        _, want = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        mine = [i for i in invs if i.spec.name == fn]
        assert sim.sharing.ro_loads_performed[(fn, 0)] == 1   # PCIe once for the burst
        assert any(i.ro_checksum == want for i in mine)
        assert all(i.ro_checksum in (None, want) for i in mine)
    sim.check_no_leaks()
finally:
    sim.close()
print("ok")
"""
    r = subprocess.run([sys.executable, "-c", code, str(ROOT)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]


def test_admission_window_bounds_concurrency():
    """ClusterSpec.admission_window: no more than the window's invocations of
    a GPU are started and unfinished at once; the rest wait in the
    dispatcher's FIFO and every invocation completes, in arrival order of
    admission, with the same landed bytes."""
    code = r"""
import sys
sys.path.insert(0, sys.argv[1])
from oracle import oracle as O
from paper_2404_14691_b200.experiments import synthetic_function
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
a, da = synthetic_function("fa", 4, 1, 0.0625, tensors=5)
sim = Simulation(ClusterSpec(gpus=1, admission_window=3), policy_preset("SAGE"), {"fa": a}, seed=5,
                 function_data={"fa": da}, copy_results=False)
peak = [0]
orig = sim.start_invocation
def start(inv, *x, **k):
    orig(inv, *x, **k)
    peak[0] = max(peak[0], sim._in_flight_gpu[inv.gpu])
sim.start_invocation = start
try:
    invs = sim.submit_many(["fa"] * 40)
    sim.drain()
    assert all(i.outcome == "completed" for i in invs)
    assert peak[0] == 3, peak[0]
    starts = [i.start_us for i in invs]
    assert starts == sorted(starts)          # FIFO admission
    lay = da.layout
    _, want = O.land_c(da.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    assert any(i.ro_checksum == want for i in invs)
    sim.check_no_leaks()
finally:
    sim.close()
print("ok")
"""
    r = subprocess.run([sys.executable, "-c", code, str(ROOT)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]


def test_prewarm_leaves_a_cold_plane():
    """Simulation.prewarm(n): the warm-up burst runs and is forgotten -- no
    invocation records, no resident segment (the next arrival is cold and
    loads its RO bytes over PCIe), no memory held."""
    code = r"""
import sys
sys.path.insert(0, sys.argv[1])
from paper_2404_14691_b200.experiments import synthetic_function
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
a, da = synthetic_function("fa", 4, 1, 0.0625, tensors=5)
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {"fa": a}, seed=5, function_data={"fa": da},
                 copy_results=False)
try:
    sim.prepare()
    sim.prewarm(24)
    assert sim.invocations == [] and not sim.sharing.residents
    sim.check_no_leaks()
    inv = sim.submit_many(["fa"])[0]
    sim.drain()
    assert inv.outcome == "completed" and inv.warmth.name == "COLD" and inv.ro_source == "pcie"
finally:
    sim.close()
print("ok")
"""
    r = subprocess.run([sys.executable, "-c", code, str(ROOT)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
