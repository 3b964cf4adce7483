"""Edge cases on the real plane (the reference's own edge cases, SURVEY.md
§8c / functions.py:62-67, policies.py:290-293): a function with no read-only
data, a function with no input, an oversized function (fails permanently,
nothing allocated), a 1-byte read-only record, and all of them mixed in one
burst with normal functions -- results, warmth and ledger stay consistent."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_edge_functions_in_one_burst(built):
    from conftest import gpu_available
    from paper_2404_14691_b200.functions import load_spec_table
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    table = load_spec_table({
        "no_ro": {"ro_mem_mb": 0, "writable_mem_mb": 4, "compute_ms": 1, "input_bytes_host_mb": 1,
                  "input_bytes_pcie_mb": 1},
        "no_input": {"ro_mem_mb": 8, "writable_mem_mb": 1, "compute_ms": 1, "input_bytes_host_mb": 0,
                     "input_bytes_pcie_mb": 0},
        "tiny_ro": {"ro_mem_mb": 0.000001, "writable_mem_mb": 1, "compute_ms": 1},
        "normal": {"ro_mem_mb": 32, "writable_mem_mb": 2, "compute_ms": 1},
        "huge": {"ro_mem_mb": 4000, "writable_mem_mb": 1, "compute_ms": 1},
    })
    names = ["no_ro", "no_input", "tiny_ro", "normal", "huge"] * 3
    with Simulation(ClusterSpec(gpus=1, gpu_mem_mb=3000), policy_preset("SAGE"), table, seed=1) as sim:
        invs = sim.submit_many(names)
        sim.drain()
        for inv in invs:
            if inv.spec.name == "huge":
                assert inv.outcome == "failed" and "larger than GPU memory" in inv.fail_reason
                continue
            assert inv.outcome == "completed", (inv.spec.name, inv.fail_reason)
            fd = sim.dataplane.data[inv.spec.name]
            lay = fd.layout
            digest = np.frombuffer(bytes(inv.result[:16]), dtype=np.uint64)
            if lay.seg_bytes:
                _, want_ro = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
                assert int(digest[0]) == want_ro
            else:
                assert int(digest[0]) == 0
            if fd.input_bytes:
                x = np.zeros(-(-fd.input_bytes // 16) * 16, np.uint8)
                x[:fd.input_bytes] = fd.input
                assert int(digest[1]) == O.checksum_c(x)
            else:
                assert int(digest[1]) == 0
        warm = {n: [i.warmth.label() for i in invs if i.spec.name == n] for n in table if n != "huge"}
        assert all(w[0] == "Cold" and w[1:] == ["Stage1Hot", "Stage1Hot"] for w in warm.values()), warm
        assert not any(i.spec.name == "huge" and i.allocations for i in invs)
        sim.sharing.check_consistency()
        sim.check_no_leaks()
