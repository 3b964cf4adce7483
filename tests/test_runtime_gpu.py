"""The real plane replays the reference's scenarios on a B200.

Control-plane parity: warmth, leader/follower waits, planned bytes, read-only
load counts and ledger allocations equal the reference simulator's decisions
(tests/golden/sim_parity.json, generated from gslsim).  Data-plane parity:
every landed segment's checksum, the bytes the TOUCH body reads and every
function body's output match the CPU oracle.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_14691_b200 import parboil
from paper_2404_14691_b200.functions import Stage, builtin_spec_table, load_spec_table, umb_to_bytes
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, SequenceSource, Simulation

pytestmark = pytest.mark.gpu
GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "sim_parity.json").read_text())["scenarios"]


@pytest.fixture(scope="module")
def built_lib(built):
    from conftest import gpu_available
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    return True


def allocs(ledger):
    return sorted([a.cls.name.lower(), a.requested, a.effective] for a in ledger.allocations())


def want_allocs(u):
    return sorted([c, umb_to_bytes(r), umb_to_bytes(e)] for c, r, e in u["allocs"])


def check_against(invs, want):
    """Exact parity on warmth, stage set and planned bytes.  Whether a follower
    still has to WAIT depends on the leader's progress at its admission: the
    reference's GPU_CTX takes a modelled 285 ms (functions.py:59) while the
    pooled context bind here takes microseconds, so the real plane may find a
    token ready where the model did not -- never the reverse.  The invariant
    that matters (tests/test_policies.py:188-201) is checked instead: no
    follower computes before its leader's read-only segment landed."""
    assert len(invs) == len(want)
    for g, w in zip(invs, want):
        assert g.outcome == w["outcome"], (g, g.fail_reason)
        assert g.warmth.label() == w["warmth"], (g.id, w)
        if Stage.SYNC_WAIT in g.stages:
            assert w["sync_wait"], (g.id, w)
        assert (Stage.GPU_CTX in g.stages) == w["has_gpu_ctx"], (g.id, w)
        assert g.pcie_bytes_umb == w["pcie_bytes_umb"] and g.host_bytes_umb == w["host_bytes_umb"], (g.id, w)
    leaders = {}
    for g in invs:
        if g.warmth.label() != "Stage1Hot" and g.ro_landed_us is not None:
            leaders[(g.spec.name, g.gpu)] = g.ro_landed_us
        elif g.warmth.label() == "Stage1Hot" and (g.spec.name, g.gpu) in leaders:
            assert g.stages[Stage.COMPUTE][0] >= leaders[(g.spec.name, g.gpu)], g


def oracle_touch(fd):
    """What the TOUCH body must return: checksums of the landed RO segment and
    of the landed input (both via the oracle)."""
    lay = fd.layout
    _, ro = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    inp = np.zeros((fd.input_bytes + 15) // 16 * 16, np.uint8)
    inp[:fd.input_bytes] = fd.input
    return ro, O.checksum_c(inp)


@pytest.mark.parametrize("policy", ["SAGE", "SAGE_NR", "FixedGSL", "DGSF"])
def test_burst16_parity(built_lib, policy):
    sc = GOLD[f"burst16_{policy}"]
    table = load_spec_table(sc["functions"])
    sim = Simulation(ClusterSpec(gpus=1, gpu_mem_mb=40960), policy_preset(policy), table, seed=1)
    try:
        invs = sim.submit_many([fn for _, fn in sc["arrivals_ms"]])
        assert allocs(sim.gpu_ledgers[0]) == want_allocs(sc["usage_t0"])
        sim.gpu_ledgers[0].check_native()
        sim.drain()
        check_against(invs, sc["invocations"])
        fd = sim.dataplane.data["fn100"]
        want_ro, want_in = oracle_touch(fd)
        for inv in invs:
            assert inv.ro_checksum == want_ro or (inv.ro_checksum is None and inv.warmth.label() == "Stage1Hot")
            got = inv.result.view(np.uint64)
            assert int(got[0]) == want_ro and int(got[1]) == want_in, inv
            assert inv.setup_us is not None and inv.setup_us >= 0
        if sim.sharing is not None:
            assert {f"{k[0]}@{k[1]}": v for k, v in sim.sharing.ro_loads_performed.items()} == sc["ro_loads"]
        if sim.policy_cfg.ro_sharing:
            # PCIe once: the leader alone moved the read-only bytes (plus the
            # 16-byte chunk-overlap prefix each staged chunk after the first carries)
            moved = sum(i.measured["pcie_bytes"] for i in invs)
            chunk = int(sim.cluster.chunk_mb * (1 << 20))
            extra = 16 * ((fd.layout.packed_bytes + chunk - 1) // chunk - 1)
            assert moved == fd.layout.packed_bytes + extra + 16 * fd.input_bytes
        sim.check_no_leaks()
    finally:
        sim.close()


@pytest.mark.parametrize("name", ["table5_SAGE", "conservation_SAGE"])
def test_decay_sequence_parity_scaled(built_lib, name):
    """Every time / 50: 0.6 s decay windows, arrivals centred in them."""
    sc = GOLD[name]
    arrivals = [(t_ms * 20, fn) for t_ms, fn in sc["arrivals_ms"]]   # ms/50 in µs
    sim = Simulation(ClusterSpec(gpus=1, gpu_mem_mb=40960),
                     policy_preset("SAGE").with_overrides(stage_interval_s=0.6), builtin_spec_table(), seed=1)
    try:
        sim.prepare(["resnet50"])           # registration (data + layout upload) before the clock starts
        src = SequenceSource([(t + sim.engine.tick(), fn) for t, fn in arrivals])
        src.attach(sim)
        sim.source = src
        sim.drain()
        check_against(sim.invocations, sc["invocations"])
        assert {f"{k[0]}@{k[1]}": v for k, v in sim.sharing.ro_loads_performed.items()} == sc["ro_loads"]
        sums = {i.ro_checksum for i in sim.invocations if i.ro_checksum is not None}
        assert len(sums) == 1                  # every reload (DB or Stage-2 cache) landed identical bytes
        if name == "table5_SAGE":
            srcs = [i.ro_source for i in sim.invocations]
            assert srcs[2] == "cache" and srcs[3] == "cache"    # Stage2 / Stage3 rejoin from the pinned cache
            assert srcs[4] == "pcie" and srcs[5] == "pcie"      # Stage4 / Cold reload from the DB
        sim.sharing.check_consistency()
    finally:
        sim.close()


def test_parboil_bodies_match_oracle(built_lib):
    table, data = parboil.cfg2_functions(scale=4)
    sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data)
    try:
        invs = sim.submit_many(["sgemm", "stencil", "spmv", "sgemm", "spmv"])
        sim.drain()
        for inv in invs:
            fd = data[inv.spec.name]
            lay = fd.layout
            seg, cs = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
            if inv.ro_checksum is not None:
                assert inv.ro_checksum == cs
            x = fd.input
            if fd.body == "sgemm":
                m, n, k = fd.args
                want = O.sgemm_ref(seg[:m * k * 4].view(np.float32).reshape(m, k), x.view(np.float32).reshape(n, k).T)
                got = inv.result.view(np.float32).reshape(m, n)
                # FP32 contract (3xTF32 tcgen05): rtol 1e-3, atol 1e-4 * max|C|
                np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-4 * np.abs(want).max())
            elif fd.body == "stencil":
                nx, ny, nz, bits = fd.args
                beta = float(np.int32(bits).view(np.float32))
                want = O.stencil_ref(seg.view(np.float32)[:nx * ny * nz].reshape(nz, ny, nx),
                                     x.view(np.float32).reshape(nz, ny, nx), beta)
                np.testing.assert_allclose(inv.result.view(np.float32).reshape(nz, ny, nx), want, rtol=1e-3, atol=1e-5)
            else:
                rows, nnz, o_rp, o_col, o_val = fd.args
                want = O.spmv_ref(seg[o_rp:o_rp + 4 * (rows + 1)].view(np.int32),
                                  seg[o_col:o_col + 4 * nnz].view(np.int32), seg[o_val:o_val + 4 * nnz].view(np.float32),
                                  x.view(np.float32))
                np.testing.assert_allclose(inv.result.view(np.float32), want, rtol=1e-3, atol=1e-4)
    finally:
        sim.close()


def test_full_size_cfg2_burst(built_lib):
    """The bench workload itself (64 concurrent, full sizes): every output is
    checked against the oracle for one invocation per function."""
    table, data = parboil.cfg2_functions()
    sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data)
    try:
        names = [sorted(table)[k % 3] for k in range(64)]
        invs = sim.submit_many(names)
        sim.drain()
        assert all(i.outcome == "completed" for i in invs)
        assert sum(i.warmth.label() == "Cold" for i in invs) == 3
        seen = set()
        for inv in invs:
            if inv.spec.name in seen:
                continue
            seen.add(inv.spec.name)
            fd = data[inv.spec.name]
            lay = fd.layout
            seg, cs = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
            if fd.body == "spmv":
                rows, nnz, o_rp, o_col, o_val = fd.args
                want = O.spmv_ref(seg[o_rp:o_rp + 4 * (rows + 1)].view(np.int32),
                                  seg[o_col:o_col + 4 * nnz].view(np.int32), seg[o_val:o_val + 4 * nnz].view(np.float32),
                                  fd.input.view(np.float32))
                np.testing.assert_allclose(inv.result.view(np.float32), want, rtol=1e-3, atol=1e-4)
            elif fd.body == "sgemm":
                m, n, k = fd.args
                A = seg[:m * k * 4].view(np.float32).reshape(m, k)
                BT = fd.input.view(np.float32).reshape(n, k)
                rows = np.arange(0, m, 97)
                want = (A[rows].astype(np.float64) @ BT.T.astype(np.float64)).astype(np.float32)
                got = inv.result.view(np.float32).reshape(m, n)[rows]
                np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-4 * np.abs(want).max())
        sim.check_no_leaks()
    finally:
        sim.close()


@pytest.mark.parametrize("fmt", ["csr", "csb"])
def test_spmv_function_formats_through_the_runtime(built_lib, fmt):
    """The same ragged matrix registered as a CSR function and as a
    column-sliced block (CSB) function: a cold burst through the public API
    lands each record bit-exactly (checksum vs the oracle's land) and every
    invocation's y matches the CSR reference of the matrix."""
    rows = 20_000
    counts = np.random.default_rng(4).integers(0, 30, rows)
    counts[::9] = 0
    spec, fd = parboil.spmv(rows=rows, seed=21, name=f"spmv_{fmt}", fmt=fmt, row_counts=counts)
    _, csr = parboil.spmv(rows=rows, seed=21, name="ref", fmt="csr", row_counts=counts)
    lay = csr.layout
    seg, _ = O.land_c(csr.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
    r, nnz, o_rp, o_col, o_val = csr.args
    want = O.spmv_ref(seg[o_rp:o_rp + 4 * (r + 1)].view(np.int32), seg[o_col:o_col + 4 * nnz].view(np.int32),
                      seg[o_val:o_val + 4 * nnz].view(np.float32), csr.input.view(np.float32))
    _, land_sum = O.land_c(fd.db, fd.layout.src_off, fd.layout.dst_off, fd.layout.length, fd.layout.seg_bytes)
    with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=2,
                    function_data={spec.name: fd}) as sim:
        invs = sim.submit_many([spec.name] * 6)
        sim.drain()
        assert [i.warmth.label() for i in invs] == ["Cold"] + ["Stage1Hot"] * 5
        assert invs[0].ro_checksum == land_sum
        for i in invs:
            assert i.outcome == "completed"
            np.testing.assert_allclose(i.result.view(np.float32)[:rows], want, rtol=1e-3, atol=1e-4)
