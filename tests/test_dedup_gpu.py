"""Content deduplication of shared RO segments (north_star: the checksum lets
the data-sharing manager "deduplicate and verify shared segments").  Two
functions registered with byte-identical RO records: with content_dedup the
second's cold start maps the first's landed segment (found through the
native table's content index, keyed by the checksum the record has once
landed) instead of loading it -- no RO bytes cross PCIe, the ledger holds one
segment -- and both compute correct results; the owner's segment outlives
its own decay while the other function still maps it."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_14691_b200.parboil import cfg2_functions
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation

pytestmark = pytest.mark.gpu


def test_identical_records_share_one_segment(built):
    table, data = cfg2_functions(scale=8)
    name = "sgemm"
    spec, fd = table[name], data[name]
    import dataclasses
    twin = dataclasses.replace(spec, name="sgemm_twin")
    table2 = {name: spec, "sgemm_twin": twin}
    data2 = {name: fd, "sgemm_twin": fd}
    cfg = policy_preset("SAGE").with_overrides(content_dedup=True, stage_interval_s=0.2)
    with Simulation(ClusterSpec(gpus=1), cfg, table2, seed=1, function_data=data2) as sim:
        a = sim.submit(name)
        sim.drain()
        ro_after_a = sim.gpu_ledgers[0].usage_by_class()
        b = sim.submit("sgemm_twin")
        sim.drain()
        assert a.ro_source == "pcie" and b.ro_source == "dedup"
        assert b.warmth.label() == "Cold"                      # its own context was still made
        lay = fd.layout
        assert b.measured["pcie_bytes"] < lay.packed_bytes       # only its input crossed PCIe
        from paper_2404_14691_b200.resources import AllocClass
        ro_now = sim.gpu_ledgers[0].usage_by_class()
        assert ro_now[AllocClass.READ_ONLY] == ro_after_a[AllocClass.READ_ONLY]   # one RO segment
        ra, rb = sim.sharing.residents[(name, 0)], sim.sharing.residents[("sgemm_twin", 0)]
        assert rb.shares is ra and ra.borrowers == 1 and rb.gpu_ro is ra.gpu_ro
        seg, _ = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        m, n, k = fd.args
        want = O.sgemm_ref(seg[:m * k * 4].view(np.float32).reshape(m, k), fd.input.view(np.float32).reshape(n, k).T)
        for inv in (a, b):
            np.testing.assert_allclose(inv.result.view(np.float32).reshape(m, n), want, rtol=1e-3,
                                       atol=1e-4 * np.abs(want).max())
        sim.sharing.check_consistency()
        # the owner decays first (its RO leaves the table) while the twin still maps
        # the pages: they stay in the ledger until the twin's RO goes too
        sim.run(until=sim.engine.now + 300_000)
        sim.sharing.check_consistency()
        sim.check_no_leaks()
        c = sim.submit(name)                                   # both decayed past Stage1: a fresh load
        sim.drain()
        assert c.outcome == "completed"
        sim.check_no_leaks()
