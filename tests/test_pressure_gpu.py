"""Memory pressure on the real plane: a budget that holds two residents, four
functions cycled -- every admission past the second forces the LRU demotion
of a decayed resident (sharing.py:271-298) while the issuer may still have
work queued.  The plane's warmth / allocation decisions must equal the
reference simulator's for the same sequence (tests/golden/pressure_golden.json,
made by tests/golden/make_pressure_golden.py), every landed segment must
verify against the oracle, every
TOUCH result must be the oracle checksums of the bytes it read, and nothing
may leak."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "pressure_golden.json").read_text())
SEQ = GOLD["sequence"]


def _table():
    from paper_2404_14691_b200.functions import load_spec_table
    return load_spec_table(GOLD["functions"])


def test_force_demotion_cycle_matches_host_logic_and_oracle(built):
    from conftest import gpu_available
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    table = _table()
    with Simulation(ClusterSpec(gpus=1, gpu_mem_mb=GOLD["gpu_mem_mb"]), policy_preset("SAGE"), table, seed=1) as sim:
        got = []
        for name in SEQ:
            inv = sim.submit(name)
            sim.drain()
            assert inv.outcome == "completed", inv.fail_reason
            got.append(inv.warmth.label())
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
        assert got == GOLD["warmth"]
        assert {k[0]: v for k, v in sim.sharing.ro_loads_performed.items()} == GOLD["ro_loads"]
