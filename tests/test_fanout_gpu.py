"""PCIe once per box across processes (paper_2404_14691_b200/fanout.py) on one
GPU: the collective is replaced by a loopback that moves the same bytes on
the stream the data plane hands it, so both sides of the fan-out run through
the real data plane.

  home      the cold leader loads over PCIe; the bytes handed to the "send"
            (copied out on the send stream) must be the landed segment --
            proving the send is ordered after the land.
  receiver  the cold leader's segment arrives by the "receive" (a D2D of the
            home's landed bytes on the receive stream), then lands from HBM
            with a checksum: ro_source "nccl", checksum = oracle, no RO bytes
            on PCIe, every output equal to the oracle.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _oracle_segments(data):
    out = {}
    for name, fd in data.items():
        lay = fd.layout
        seg, cs = O.land_c(fd.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        out[name] = (seg, cs)
    return out


def _check_outputs(invs, data, segs):
    for i in invs:
        fd = data[i.spec.name]
        seg = segs[i.spec.name][0]
        x = fd.input
        if fd.body == "sgemm":
            m, n, k = fd.args
            want = O.sgemm_ref(seg[:m * k * 4].view(np.float32).reshape(m, k), x.view(np.float32).reshape(n, k).T)
            np.testing.assert_allclose(i.result.view(np.float32).reshape(m, n), want, rtol=1e-3,
                                       atol=1e-4 * np.abs(want).max())
        elif fd.body == "stencil":
            nx, ny, nz, bits = fd.args
            want = O.stencil_ref(seg.view(np.float32)[:nx * ny * nz].reshape(nz, ny, nx),
                                 x.view(np.float32).reshape(nz, ny, nx), float(np.int32(bits).view(np.float32)))
            np.testing.assert_allclose(i.result.view(np.float32).reshape(nz, ny, nx), want, rtol=1e-3, atol=1e-5)
        else:
            rows, nnz, o_rp, o_col, o_val = fd.args
            want = O.spmv_ref(seg[o_rp:o_rp + 4 * (rows + 1)].view(np.int32), seg[o_col:o_col + 4 * nnz].view(np.int32),
                              seg[o_val:o_val + 4 * nnz].view(np.float32), x.view(np.float32))
            np.testing.assert_allclose(i.result.view(np.float32)[:rows], want, rtol=1e-3, atol=1e-4)


def _d2d(stream: int, dst: int, src: int, nbytes: int) -> None:
    import torch

    from paper_2404_14691_b200.dnn import view
    dev = torch.device("cuda", 0)
    with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=dev)):
        view(dst, nbytes, dev).copy_(view(src, nbytes, dev))


@pytest.mark.parametrize("role", ["home", "receiver"])
def test_box_fanout_loopback(built, role):
    from conftest import gpu_available
    from paper_2404_14691_b200 import device as D
    from paper_2404_14691_b200 import _lib
    from paper_2404_14691_b200.fanout import BoxFanout
    from paper_2404_14691_b200.parboil import cfg2_functions
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    table, data = cfg2_functions(scale=4)
    segs = _oracle_segments(data)
    names = [sorted(table)[k % 3] for k in range(18)]
    sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=2, function_data=data)
    sent, refs = {}, {}
    try:
        if role == "receiver":
            # what the home rank would send: each function's landed segment
            for name, fd in data.items():
                seg = D.pool_alloc(0, fd.layout.seg_bytes, _lib.CLASS_WRITABLE, unaccounted=True)
                op = D.load(0, seg.dptr, fd.db, fd.layout)
                assert op.wait().checksum == segs[name][1]
                op.release()
                refs[fd.layout.seg_bytes] = seg

        def loopback(gpu, stream, dptr, nbytes, src):
            if role == "home":          # the send: copy out what is at dptr, in stream order
                cap = D.pool_alloc(0, nbytes, _lib.CLASS_WRITABLE, unaccounted=True)
                _d2d(stream, cap.dptr, dptr, nbytes)
                sent[nbytes] = cap
            else:                       # the receive: the home's bytes arrive at dptr
                _d2d(stream, dptr, refs[nbytes].dptr, nbytes)

        world = 2
        box = BoxFanout(rank=0 if role == "home" else 1, world=world, names=table,
                        homes={n: 0 for n in table}, broadcast=loopback)
        sim.dataplane.box = box
        invs = sim.submit_many(names)
        sim.drain()
        assert all(i.outcome == "completed" for i in invs)
        leaders = [i for i in invs if i.warmth.label() == "Cold"]
        assert len(leaders) == 3
        for i in leaders:
            fd = data[i.spec.name]
            assert i.ro_checksum == segs[i.spec.name][1]
            if role == "home":
                assert i.ro_source == "pcie"
            else:
                assert i.ro_source == "nccl"
                assert i.measured["nvlink_bytes"] == fd.layout.seg_bytes
                assert i.measured["pcie_bytes"] == fd.input_bytes       # only the input crossed PCIe
        _check_outputs(invs, data, segs)
        if role == "home":
            assert box.sent == 3 and box.received == 0
            for name, fd in data.items():
                cap = sent[fd.layout.seg_bytes]
                assert D.segment_checksum(0, cap.dptr, fd.layout.seg_bytes) == segs[name][1]
        else:
            assert box.received == 3 and box.sent == 0
    finally:
        for s in list(sent.values()) + list(refs.values()):
            s.free()
        sim.close()
