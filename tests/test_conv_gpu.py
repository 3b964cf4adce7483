"""The tcgen05 implicit-GEMM convolution (csrc/conv_tc.cu) through the C-ABI
(sage_conv) against torch-CPU fp32 on the same bf16 values: every ResNet-50
convolution shape class (1x1 stride 1 / 2, 3x3 stride 1 / 2, conv1's 7x7
stride 2 in the C4 mode), folded batch-norm, residual add, ReLU, ragged M
(rows past the last full 128-pixel tile), the 2-stage short-K and 4-stage
long-K BN = 256 kernels.  BF16 outputs: rtol 1e-2 with
atol 1e-2 * max|y| (BASELINE.json north_star BF16 tolerance)."""
import ctypes as C

import numpy as np
import pytest

from paper_2404_14691_b200 import _lib
from paper_2404_14691_b200 import device as D

pytestmark = pytest.mark.gpu


def bf16_bytes(t):
    import torch
    return t.contiguous().to(torch.bfloat16).view(torch.int16).numpy().view(np.uint8).reshape(-1)


def upload(b: np.ndarray):
    seg = D.pool_alloc(0, max(256, b.size + 256), _lib.CLASS_WRITABLE, unaccounted=True)
    if b.size:
        op = D.load(0, seg.dptr, b, None)
        op.wait()
        op.release()
    return seg


def run_conv(x_nhwc, w_ohwi, bn, res_nhwc, stride, pad, relu, mode=_lib.CONV_NHWC, r=None, s=None, cin=None):
    import torch
    n, h, w, c = x_nhwc.shape
    cout = w_ohwi.shape[0]
    r = r or w_ohwi.shape[1]
    s = s or w_ohwi.shape[2]
    p = (h + 2 * pad - r) // stride + 1
    q = (w + 2 * pad - s) // stride + 1
    if mode == _lib.CONV_S2D:      # pad 2 before, 1 after: the output keeps the input's size
        p, q = h, w
    segs = [upload(bf16_bytes(x_nhwc)), upload(bf16_bytes(w_ohwi))]
    out = D.pool_alloc(0, n * p * q * cout * 2 + 256, _lib.CLASS_WRITABLE, unaccounted=True)
    d = _lib.ConvDesc()
    d.x, d.w, d.out = segs[0].dptr, segs[1].dptr, out.dptr
    if res_nhwc is not None:
        segs.append(upload(bf16_bytes(res_nhwc)))
        d.residual = segs[-1].dptr
    if bn is not None:
        for name, t in zip(("bn_gamma", "bn_beta", "bn_mean", "bn_var"), bn):
            segs.append(upload(bf16_bytes(t)))
            setattr(d, name, segs[-1].dptr)
        d.bn_eps = 1e-5
    d.n, d.h, d.w_, d.cin, d.cout, d.r, d.s = n, h, w, cin or c, cout, r, s
    d.stride, d.pad, d.relu, d.mode = stride, pad, int(relu), mode
    slot = D.Slot(0)
    _lib.check(_lib.lib().sage_conv(slot.h, C.byref(d)), "sage_conv")
    e = slot.record()
    e.sync()
    e.release()
    slot.release()
    raw = D.read_device(0, out.dptr, n * p * q * cout * 2)
    got = torch.from_numpy(raw.view(np.int16).copy()).view(torch.bfloat16).float().view(n, p, q, cout)
    for sg in segs + [out]:
        sg.free()
    return got


def reference(x_nhwc, w_ohwi, bn, res_nhwc, stride, pad, relu):
    """torch-CPU fp32 on the bf16-rounded operands."""
    import torch
    import torch.nn.functional as F
    rb = lambda t: t.to(torch.bfloat16).float()
    x = rb(x_nhwc).permute(0, 3, 1, 2)
    w = rb(w_ohwi).permute(0, 3, 1, 2)
    y = F.conv2d(x, w, stride=stride, padding=pad)
    if bn is not None:
        g, b, m, v = (rb(t) for t in bn)
        sc = g / torch.sqrt(v + 1e-5)
        y = y * sc[None, :, None, None] + (b - m * sc)[None, :, None, None]
    y = y.permute(0, 2, 3, 1)
    if res_nhwc is not None:
        y = y + rb(res_nhwc)
    return torch.relu(y) if relu else y


SHAPES = [  # n, h, w, cin, cout, k, stride, pad, bn, residual, relu
    (2, 14, 14, 64, 64, 1, 1, 0, True, False, True),        # 1x1, M = 392 (ragged last tile)
    (2, 28, 28, 128, 512, 1, 1, 0, True, True, True),       # 1x1 expand + residual + ReLU
    (2, 28, 28, 256, 512, 1, 2, 0, True, False, False),     # downsample 1x1 stride 2
    (2, 14, 14, 64, 64, 3, 1, 1, True, False, True),        # 3x3 stride 1 (padding taps)
    (2, 15, 15, 128, 128, 3, 2, 1, False, False, False),    # 3x3 stride 2, odd size, no BN
    (1, 7, 7, 512, 2048, 1, 1, 0, True, True, True),        # layer4 expand: M = 49
    (3, 9, 11, 192, 320, 3, 1, 1, True, True, True),        # non power-of-two channels (Cout % 64)
    (2, 14, 14, 256, 256, 3, 1, 1, True, False, True),      # BN = 256, 36 K-blocks: the 4-stage kernel
    (1, 7, 7, 512, 512, 3, 1, 1, True, True, True),         # layer4 3x3: 72 K-blocks, 4 M tiles
    (2, 28, 28, 256, 256, 3, 2, 1, True, False, True),      # 3x3 stride 2, BN = 256, long K
    (4, 56, 56, 64, 256, 1, 1, 0, True, True, True),        # layer1 expand: 1 K-block, 98 M tiles (2-stage kernel)
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s[:8])))
def test_conv_matches_torch_cpu(dp, shape):
    import torch
    n, h, w, cin, cout, k, stride, pad, use_bn, use_res, relu = shape
    torch.manual_seed(sum(shape[:8]))
    x = torch.randn(n, h, w, cin)
    wt = torch.randn(cout, k, k, cin) * (2.0 / (k * k * cin)) ** 0.5
    bn = None
    if use_bn:
        bn = (torch.rand(cout) + 0.5, torch.randn(cout) * 0.1, torch.randn(cout) * 0.1, torch.rand(cout) + 0.5)
    p = (h + 2 * pad - k) // stride + 1
    q = (w + 2 * pad - k) // stride + 1
    res = torch.randn(n, p, q, cout) if use_res else None
    got = run_conv(x, wt, bn, res, stride, pad, relu)
    want = reference(x, wt, bn, res, stride, pad, relu)
    np.testing.assert_allclose(got.numpy(), want.numpy(), rtol=1e-2, atol=1e-2 * float(want.abs().max()))


def test_conv1_c4_mode_matches_torch_cpu(dp):
    """ResNet-50's stem: 7x7 stride 2, 3 input channels padded to 4, filter
    K padded to 256 (16 taps x 4 channels per 64-wide K-block)."""
    import torch
    torch.manual_seed(7)
    n, h, w, cout = 2, 32, 30, 64
    x3 = torch.randn(n, h, w, 3)
    w3 = torch.randn(cout, 7, 7, 3) * 0.1
    bn = (torch.rand(cout) + 0.5, torch.randn(cout) * 0.1, torch.randn(cout) * 0.1, torch.rand(cout) + 0.5)
    x4 = torch.zeros(n, h, w, 4)
    x4[..., :3] = x3
    wpad = torch.zeros(cout, 256)
    wpad[:, :49 * 4] = torch.cat([w3, torch.zeros(cout, 7, 7, 1)], dim=3).reshape(cout, 196)
    got = run_conv(x4, wpad.view(cout, 1, 1, 256), bn, None, 2, 3, True, mode=_lib.CONV_C4, r=7, s=7, cin=4)
    want = reference(x3, w3, bn, None, 2, 3, True)
    np.testing.assert_allclose(got.numpy(), want.numpy(), rtol=1e-2, atol=1e-2 * float(want.abs().max()))


def test_conv1_s2d_mode_matches_torch_cpu(dp):
    """The stem as the S2D mode: the 7x7 stride-2 pad-3 convolution of a
    3-channel image run as a 4x4 stride-1 implicit GEMM over its 2x2
    space-to-depth input (16 channels), against torch-CPU fp32 of the
    original convolution (BN + ReLU fused)."""
    import torch
    from paper_2404_14691_b200 import dnn
    g = torch.Generator().manual_seed(11)
    n, h = 2, 40
    x = torch.randn(n, h, h, 3, generator=g)
    w = torch.randn(64, 3, 7, 7, generator=g) * 0.1
    bn = (torch.rand(64, generator=g) + 0.5, torch.randn(64, generator=g), torch.randn(64, generator=g) * 0.1,
          torch.rand(64, generator=g) + 0.5)
    rb = lambda t: t.to(torch.bfloat16).float()
    xs = dnn.stem_s2d_input(rb(x).numpy())
    ws = dnn.stem_s2d_filter(rb(w).numpy()).reshape(64, 4, 4, 16)
    got = run_conv(torch.from_numpy(xs), torch.from_numpy(ws), bn, None, 1, 2, True, mode=_lib.CONV_S2D)
    want = reference(x, w.permute(0, 2, 3, 1), bn, None, 2, 3, True)
    assert got.shape == want.shape == (n, h // 2, h // 2, 64)
    m = float(want.abs().max())
    np.testing.assert_allclose(got.numpy(), want.numpy(), rtol=1e-2, atol=1e-2 * m)


def test_conv_rejects_bad_shapes(dp):
    import torch
    with pytest.raises(_lib.SageError):
        run_conv(torch.randn(1, 8, 8, 48), torch.randn(64, 1, 1, 48), None, None, 1, 0, False)   # Cin % 64


def test_conv_cta_pair_variant():
    """SAGE_CONV_PAIR=1 (BN = 256 tiles as cta_group::2 CTA pairs, half the
    filter tile per SM; opt-in, measured slower): the same parity, in its own
    process because the variant is chosen at library load."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-m", "pytest", str(root / "tests" / "test_conv_gpu.py"), "-x", "-q",
                        "-k", "matches_torch_cpu"], env={**os.environ, "SAGE_CONV_PAIR": "1"}, cwd=str(root),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
