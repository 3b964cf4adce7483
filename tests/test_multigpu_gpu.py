"""Multi-GPU control plane + PCIe-once fan-out.

This pool exposes one physical B200 per call, so the runtime is started with
two LOGICAL GPUs (SAGE_INIT_SHARE_DEVICE: two independent planes -- pools,
rings, streams, residents -- on one device).  Placement, per-GPU residents and
the fan-out decision are exactly the multi-GPU code; the peer land reads the
other plane's segment through the same kernel path an NVLink peer read uses.
"""
import json
from pathlib import Path

import pytest

from oracle import oracle as O
from paper_2404_14691_b200.functions import builtin_spec_table
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation

pytestmark = pytest.mark.gpu
GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "sim_parity.json").read_text())["scenarios"]


@pytest.mark.parametrize("fanout", [True, False])
def test_two_gpu_placement_and_pcie_once(built, fanout):
    sc = GOLD["mixed_2gpu_SAGE"]
    sim = Simulation(ClusterSpec(gpus=2, gpu_mem_mb=40960), policy_preset("SAGE").with_overrides(fanout=fanout),
                     builtin_spec_table(), seed=1)
    try:
        sim.prepare(["resnet50", "vgg11"])
        invs = sim.submit_many([fn for _, fn in sc["arrivals_ms"]])
        sim.drain()
        assert [i.gpu for i in invs] == [w["gpu"] for w in sc["invocations"]]
        for g, w in zip(invs, sc["invocations"]):
            assert g.outcome == "completed" and g.warmth.label() == w["warmth"]
            assert g.pcie_bytes_umb == w["pcie_bytes_umb"]          # planned bytes: reference semantics
        for name in ("resnet50", "vgg11"):
            fd = sim.dataplane.data[name]
            lay = fd.layout
            _, want = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
            loads = [i for i in invs if i.spec.name == name and i.ro_checksum is not None]
            assert loads and all(i.ro_checksum == want for i in loads)
            srcs = sorted(i.ro_source for i in loads)
            gpus = {i.gpu for i in invs if i.spec.name == name}
            if fanout and len(gpus) == 2:
                # the segment crossed PCIe once for the box; the other GPU landed it from its peer
                assert srcs == ["nvlink", "pcie"], srcs
                peer = next(i for i in loads if i.ro_source == "nvlink")
                assert peer.measured["nvlink_bytes"] == lay.seg_bytes
                # only the (pageable, staged) input crossed PCIe: its bytes + the
                # 16-B overlap prefix of each staged chunk after the first
                chunks = -(-fd.input_bytes // int(sim.cluster.chunk_mb * (1 << 20)))
                assert peer.measured["pcie_bytes"] == fd.input_bytes + 16 * (chunks - 1)
            else:
                assert set(srcs) == {"pcie"}
        sim.check_no_leaks()
        for s in sim.sharing.residents.values():
            assert s.state.label == "Stage1"
        sim.sharing.check_consistency()
    finally:
        sim.close()
