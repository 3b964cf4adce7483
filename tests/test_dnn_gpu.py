"""ResNet-50 as a SAGE function, checked against torch-CPU fp32.

BF16 record (BASELINE cfg 3, the default engine): the body is the native
program of tcgen05 implicit-GEMM convolutions (csrc/resnet.cu, conv_tc.cu),
no PyTorch on the device path; logits within the BF16 tolerance of
torchvision's network run on the CPU in fp32 with the same bf16-rounded
weights and input.  FP32 record: PyTorch / cuDNN over zero-copy views of the
landed segment with TF32 disabled, within the FP32 tolerance of the CPU."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation

pytestmark = pytest.mark.gpu


def cpu_fp32_reference(x_nchw: np.ndarray, seed: int = 0) -> np.ndarray:
    import torch
    import torchvision
    torch.manual_seed(seed)
    model = torchvision.models.resnet50(weights=None).eval()
    with torch.inference_mode():
        return model(torch.from_numpy(x_nchw)).numpy()


def test_resnet50_native_bf16_matches_torch_cpu(built):
    from paper_2404_14691_b200 import dnn
    spec, data = dnn.resnet50(batch=8, seed=0, dtype="bf16")
    assert data.body == "resnet50_native" and data.layout.seg_bytes < 52 << 20
    with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=1,
                    function_data={spec.name: data}) as sim:
        sim.prepare()
        invs = sim.submit_many([spec.name] * 6)
        sim.drain()
        assert [i.warmth.label() for i in invs] == ["Cold"] + ["Stage1Hot"] * 5
        lay = data.layout
        _, want_cs = O.land_c(data.db, lay.src_off, lay.dst_off, lay.length, lay.seg_bytes)
        assert invs[0].ro_checksum == want_cs
        want = dnn.reference_cpu(data, data.input)
        for inv in invs:
            got = inv.result.view(np.float32).reshape(8, 1000)
            np.testing.assert_allclose(got, want, rtol=1e-2, atol=1e-2 * np.abs(want).max())
            assert (got.argmax(1) == want.argmax(1)).mean() >= 0.75
        sim.check_no_leaks()


def test_resnet50_native_distinct_requests(built):
    """Concurrent invocations with different request images: each reads its
    own input and workspace and returns its own logits."""
    import torch
    from paper_2404_14691_b200 import device as D
    from paper_2404_14691_b200 import dnn
    spec, data = dnn.resnet50(batch=4, seed=0, dtype="bf16")
    rng = np.random.default_rng(7)
    xs = [torch.from_numpy(rng.standard_normal((4, 224, 224, 3), dtype=np.float32)).to(torch.bfloat16)
          .view(torch.int16).numpy().reshape(-1).view(np.uint8) for _ in range(6)]
    pls = []
    for x in xs:
        pb = D.PinnedBuffer(x.nbytes)
        pb.view()[:] = x
        pls.append(pb)
    sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=1,
                     function_data={spec.name: data})
    try:
        invs = sim.submit_many([spec.name] * 6, payloads=pls)
        sim.drain()
        for inv, x in zip(invs, xs):
            want = dnn.reference_cpu(data, x)
            got = inv.result.view(np.float32).reshape(4, 1000)
            np.testing.assert_allclose(got, want, rtol=1e-2, atol=1e-2 * np.abs(want).max())
    finally:
        for pb in pls:           # before close(): shutdown frees every pinned buffer
            pb.free()
        sim.close()


def test_resnet50_fp32_torch_engine_matches_cpu_without_tf32(built):
    import torch
    from paper_2404_14691_b200 import dnn
    spec, data = dnn.resnet50(batch=8, seed=0, dtype="fp32")
    with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=1,
                    function_data={spec.name: data}) as sim:
        invs = sim.submit_many([spec.name] * 4)
        sim.drain()
        assert not torch.backends.cudnn.allow_tf32       # FP32 computed in FP32
        want = cpu_fp32_reference(data.input.view(np.float32).reshape(8, 3, 224, 224).copy())
        for inv in invs:
            got = inv.result.view(np.float32).reshape(8, 1000)
            np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-3 * np.abs(want).max())


def test_resnet50_bf16_torch_engine_within_rtol(built):
    """The cuDNN A/B engine on the same BF16 record format (channels-last)."""
    from paper_2404_14691_b200 import dnn
    spec, data = dnn.resnet50(batch=8, seed=0, dtype="bf16", engine="torch")
    assert data.meta["layout"] == "nhwc"
    with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=1,
                    function_data={spec.name: data}) as sim:
        invs = sim.submit_many([spec.name] * 3)
        sim.drain()
        native_like = dnn.resnet50(batch=8, seed=0, dtype="bf16")[1]
        want = dnn.reference_cpu(native_like, data.input)
        for inv in invs:
            got = inv.result.view(np.float32).reshape(8, 1000)
            np.testing.assert_allclose(got, want, rtol=1e-2, atol=2e-2 * np.abs(want).max())
