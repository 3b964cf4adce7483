"""The native ResNet-50 program (dnn.resnet50_native) on CPU: its structure
is torchvision's resnet50 (53 convolutions in module order with their
batch-norms, the stem pooling, avg pool + classifier), no op writes a buffer
it reads, the workspace fits the function's writable segment, the record
holds every filter OHWI (the stem padded for the C4 gather), and the library
accepts the program (sage_net_create needs no device)."""
import numpy as np

from paper_2404_14691_b200 import _lib, dnn


def test_program_mirrors_torchvision_resnet50(built):
    import torch
    import torchvision
    spec, fd = dnn.resnet50_native(batch=2, seed=0)
    ops, bufs = fd.meta["program"]
    convs = [o for o in ops if o["kind"] == _lib.NET_CONV]
    model = torchvision.models.resnet50(weights=None)
    tv = [m for m in model.modules() if isinstance(m, torch.nn.Conv2d)]
    assert len(convs) == len(tv) == 53
    off = dict(zip(fd.meta["names"], fd.layout.dst_off))
    by_off = {v: k for k, v in off.items()}
    order = [by_off[o["w_off"]] for o in convs]
    tv_names = [n + ".weight" for n, m in model.named_modules() if isinstance(m, torch.nn.Conv2d)]
    # module order within a block differs only by where the downsample runs (first)
    assert sorted(order) == sorted(tv_names)
    for o, name in zip(convs, order):
        m = dict(model.named_modules())[name[:-len(".weight")]]
        if name == "conv1.weight":   # the stem runs as a 4x4 stride-1 conv over its space-to-depth input
            assert (o["cout"], o["r"], o["stride"], o["pad"], o["cin"], o["mode"]) == (64, 4, 1, 2, 16,
                                                                                      _lib.CONV_S2D)
            continue
        assert (o["cout"], o["r"], o["stride"], o["pad"]) == (m.out_channels, m.kernel_size[0], m.stride[0],
                                                                m.padding[0]), name
        assert o["cin"] == m.in_channels
        assert o["src"] != o["dst"] and o["res"] != o["dst"]
    assert [o["kind"] for o in ops[:3]] == [_lib.NET_S2D_INPUT, _lib.NET_CONV, _lib.NET_MAXPOOL]
    assert ops[-1]["kind"] == _lib.NET_POOL_FC and ops[-1]["cout"] == 1000 and ops[-1]["dst"] == _lib.NET_BUF_OUT
    # residual adds only on the third conv of each bottleneck
    assert sum(o["res"] >= 0 for o in convs) == 16
    # the stem filter: [64][4][4][2][2][4] = w[c][2a+dr-1][2b+ds-1] (zero outside 7x7 and for c = 3)
    lay = fd.layout
    i = fd.meta["names"].index("conv1.weight")
    w = fd.db[lay.src_off[i]:lay.src_off[i] + lay.length[i]].view(np.int16).reshape(64, 4, 4, 2, 2, 4)
    assert lay.length[i] == 64 * 256 * 2
    assert not w[..., 3].any()
    assert not w[:, 0, :, 0].any() and not w[:, :, 0, :, 0].any()     # a = 0, dr = 0 -> r = -1 (outside)
    torch.manual_seed(0)
    ref = torchvision.models.resnet50(weights=None).conv1.weight.detach().to(torch.bfloat16).view(torch.int16).numpy()
    for a_, b_, dr, ds in [(1, 1, 0, 0), (2, 3, 1, 0), (3, 3, 1, 1), (0, 2, 1, 1)]:
        r, sx = 2 * a_ + dr - 1, 2 * b_ + ds - 1
        assert np.array_equal(w[:, a_, b_, dr, ds, :3], ref[:, :, r, sx])
    assert spec.writable_bytes >= fd.input_bytes + fd.out_bytes + fd.scratch_bytes


def test_stem_s2d_equals_the_7x7_stride2_conv():
    """The rewrite itself (CPU, fp32): conv2d(x, w, stride 2, pad 3) ==
    conv2d(s2d(x), s2d(w), stride 1, pad (2 before, 1 after))."""
    import torch
    import torch.nn.functional as F
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 32, 40, 3), dtype=np.float32)
    w = rng.standard_normal((64, 3, 7, 7), dtype=np.float32)
    want = F.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w), stride=2, padding=3)
    xs = torch.from_numpy(dnn.stem_s2d_input(x)).permute(0, 3, 1, 2)
    ws = torch.from_numpy(dnn.stem_s2d_filter(w).reshape(64, 4, 4, 16)).permute(0, 3, 1, 2)
    got = F.conv2d(F.pad(xs, (2, 1, 2, 1)), ws)
    np.testing.assert_allclose(got.numpy(), want.numpy(), rtol=1e-4, atol=1e-4)


def test_library_accepts_the_program(built):
    _, fd = dnn.resnet50_native(batch=2, seed=0)
    h = dnn.native_handle(fd)
    assert h and fd.args == (h, 2)
    assert _lib.lib().sage_net_destroy(h) == 0
    assert _lib.lib().sage_net_destroy(h) == _lib.SAGE_ESTATE
