"""Memory pressure on the real plane: a budget that holds two residents, four
functions cycled -- every admission past the second forces the LRU demotion
of a decayed resident (sharing.py:271-298) while the issuer may still have
work queued.  The plane's warmth / allocation decisions must equal the
product classes' decisions on CPU (FakeSim, tests/test_host_logic.py) for
the same sequence, every landed segment must verify against the oracle, every
TOUCH result must be the oracle checksums of the bytes it read, and nothing
may leak."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _table():
    from paper_2404_14691_b200.functions import load_spec_table
    return load_spec_table({f"f{k}": {"ro_mem_mb": 300, "writable_mem_mb": 16, "compute_ms": 1, "context_mem_mb": 64,
                                      "input_bytes_host_mb": 2, "input_bytes_pcie_mb": 2} for k in range(4)})


SEQ = [f"f{k % 4}" for k in range(10)] + ["f3", "f3", "f1"]


def _cpu_decisions():
    from test_host_logic import FakeSim
    sim = FakeSim("SAGE", _table(), cap_mb=800)
    out = []
    for name in SEQ:
        inv = sim.submit(name)
        sim.complete_all()
        out.append((name, inv.warmth.label(), sim.gpu_ledgers[0].usage))
    return out


def test_force_demotion_cycle_matches_host_logic_and_oracle(built):
    from conftest import gpu_available
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    want = _cpu_decisions()
    assert any(w != "Stage1Hot" for _, w, _ in want[4:])      # the budget really forces demotions
    table = _table()
    with Simulation(ClusterSpec(gpus=1, gpu_mem_mb=800), policy_preset("SAGE"), table, seed=1) as sim:
        got = []
        for name in SEQ:
            inv = sim.submit(name)
            sim.drain()
            assert inv.outcome == "completed", inv.fail_reason
            got.append((name, inv.warmth.label(), sim.gpu_ledgers[0].usage))
            fd = sim.dataplane.data[name]
            lay = fd.layout
            _, want_ro = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
            if inv.ro_checksum is not None:
                assert inv.ro_checksum == want_ro
            digest = np.frombuffer(bytes(inv.result[:16]), dtype=np.uint64)
            assert int(digest[0]) == want_ro                      # TOUCH read the landed bytes
            x = np.zeros(-(-fd.input_bytes // 16) * 16, np.uint8)
            x[:fd.input_bytes] = fd.input
            assert int(digest[1]) == O.checksum_c(x)
            sim.sharing.check_consistency()
            sim.check_no_leaks()
        assert got == want
