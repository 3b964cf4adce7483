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
        assert (o["cout"], o["r"], o["stride"], o["pad"]) == (m.out_channels, m.kernel_size[0], m.stride[0],
                                                                m.padding[0]), name
        assert o["cin"] == (4 if name == "conv1.weight" else m.in_channels)
        assert o["src"] != o["dst"] and o["res"] != o["dst"]
    assert [o["kind"] for o in ops[:3]] == [_lib.NET_PAD_INPUT, _lib.NET_CONV, _lib.NET_MAXPOOL]
    assert ops[-1]["kind"] == _lib.NET_POOL_FC and ops[-1]["cout"] == 1000 and ops[-1]["dst"] == _lib.NET_BUF_OUT
    # residual adds only on the third conv of each bottleneck
    assert sum(o["res"] >= 0 for o in convs) == 16
    # the stem filter: [64][256] with the 4th channel and the K tail zero
    lay = fd.layout
    i = fd.meta["names"].index("conv1.weight")
    w = fd.db[lay.src_off[i]:lay.src_off[i] + lay.length[i]].view(np.int16).reshape(64, 256)
    assert lay.length[i] == 64 * 256 * 2
    assert not w[:, 196:].any() and not w[:, 3:196:4].any()
    assert spec.writable_bytes >= fd.input_bytes + fd.out_bytes + fd.scratch_bytes


def test_library_accepts_the_program(built):
    _, fd = dnn.resnet50_native(batch=2, seed=0)
    h = dnn.native_handle(fd)
    assert h and fd.args == (h, 2)
    assert _lib.lib().sage_net_destroy(h) == 0
    assert _lib.lib().sage_net_destroy(h) == _lib.SAGE_ESTATE
