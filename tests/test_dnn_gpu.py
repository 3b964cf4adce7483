"""ResNet-50 as a SAGE function: weights landed by `land` into one shared RO
segment, COMPUTE by PyTorch on the invocation stream over zero-copy views.
Outputs must equal the same network run directly with its own parameters."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation

pytestmark = pytest.mark.gpu


def test_resnet50_function_matches_torch(built):
    import torch
    import torchvision
    from paper_2404_14691_b200 import dnn
    spec, data = dnn.resnet50(batch=8, seed=0)
    sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=1,
                     function_data={spec.name: data})
    try:
        invs = sim.submit_many([spec.name] * 6)
        sim.drain()
        assert [i.warmth.label() for i in invs] == ["Cold"] + ["Stage1Hot"] * 5
        lay = data.layout
        _, want_cs = O.land_c(data.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        assert invs[0].ro_checksum == want_cs
        torch.manual_seed(0)
        ref = torchvision.models.resnet50(weights=None).eval().cuda()
        x = torch.from_numpy(data.input.view(np.float32).reshape(8, 3, 224, 224).copy()).cuda()
        with torch.inference_mode():
            want = ref(x).float().cpu().numpy()
        for inv in invs:
            got = inv.result.view(np.float32).reshape(8, 1000)
            np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-3 * np.abs(want).max())
    finally:
        sim.close()


def test_resnet50_graph_replays_distinct_inputs(built):
    """Ten concurrent invocations with ten different request payloads: the
    captured CUDA graphs (4 per segment, reused round robin) must read each
    invocation's own input and return its own logits."""
    import torch
    import torchvision
    from paper_2404_14691_b200 import device as D
    from paper_2404_14691_b200 import dnn
    spec, data = dnn.resnet50(batch=8, seed=0)
    rng = np.random.default_rng(7)
    xs = [rng.standard_normal((8, 3, 224, 224), dtype=np.float32) for _ in range(10)]
    pls = []
    for x in xs:
        pb = D.PinnedBuffer(x.nbytes)
        pb.view()[:] = x.reshape(-1).view(np.uint8)
        pls.append(pb)
    sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=1,
                     function_data={spec.name: data})
    try:
        invs = sim.submit_many([spec.name] * 10, payloads=pls)
        sim.drain()
        torch.manual_seed(0)
        ref = torchvision.models.resnet50(weights=None).eval().cuda()
        for inv, x in zip(invs, xs):
            with torch.inference_mode():
                want = ref(torch.from_numpy(x).cuda()).float().cpu().numpy()
            got = inv.result.view(np.float32).reshape(8, 1000)
            np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-3 * np.abs(want).max())
    finally:
        for pb in pls:           # before close(): shutdown frees every pinned buffer
            pb.free()
        sim.close()


def test_resnet50_bf16_function_within_rtol(built):
    """The BF16 variant (51 MB of bfloat16 weights landed, bf16 input, fp32
    logits): within the north star's BF16 tolerance of the fp32 network on the
    same (bf16-rounded) input."""
    import torch
    import torchvision
    from paper_2404_14691_b200 import dnn
    spec, data = dnn.resnet50(batch=8, seed=0, dtype="bf16")
    assert data.layout.seg_bytes < 52 << 20
    with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=1,
                    function_data={spec.name: data}) as sim:
        invs = sim.submit_many([spec.name] * 5)
        sim.drain()
        assert [i.warmth.label() for i in invs] == ["Cold"] + ["Stage1Hot"] * 4
        torch.manual_seed(0)
        ref = torchvision.models.resnet50(weights=None).eval().cuda()
        assert data.meta["layout"] == "nhwc"                   # the record is packed channels-last
        x = torch.from_numpy(data.input.copy()).view(torch.bfloat16).float().view(8, 224, 224, 3)
        x = x.permute(0, 3, 1, 2).contiguous().cuda()
        with torch.inference_mode():
            want = ref(x).float().cpu().numpy()
        for inv in invs:
            got = inv.result.view(np.float32).reshape(8, 1000)
            np.testing.assert_allclose(got, want, rtol=1e-2, atol=2e-2 * np.abs(want).max())
