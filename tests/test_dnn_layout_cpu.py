"""The ResNet-50 function records (dnn.resnet50): the FP32 record packs the
state dict as is; the BF16 record packs filters OHWI and the input NHWC, and
dnn._as_logical / _input_view turn the flat bytes back into the logical
(OIHW / NCHW) tensors PyTorch's forward expects (CPU: no device needed)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytest.importorskip("torchvision")


def _flat(fd, k):
    lay = fd.layout
    return torch.from_numpy(fd.db[lay.src_off[k]:lay.src_off[k] + lay.length[k]].copy())


def test_bf16_record_is_channels_last_and_views_restore_logical_tensors():
    from paper_2404_14691_b200 import dnn
    _, fd32 = dnn.resnet50(batch=2, seed=0, dtype="fp32")
    _, fd16 = dnn.resnet50(batch=2, seed=0, dtype="bf16", engine="torch")
    assert fd32.meta["layout"] == "nchw" and fd16.meta["layout"] == "nhwc"
    assert fd16.layout.seg_bytes < fd32.layout.seg_bytes * 0.51
    names = fd32.meta["names"]
    checked = 0
    for k, (n, shp) in enumerate(zip(names, fd32.meta["shapes"])):
        if fd32.meta["dtypes"][k] != "<f4":
            continue
        want = _flat(fd32, k).view(torch.float32).view(shp).to(torch.bfloat16)
        got = dnn._as_logical(_flat(fd16, k).view(torch.bfloat16), shp, fd16)
        assert tuple(got.shape) == tuple(shp), n
        assert torch.equal(got, want), n
        if len(shp) == 4:
            assert got.is_contiguous(memory_format=torch.channels_last), n
            checked += 1
    assert checked == 53                                   # every convolution filter of ResNet-50
    x32 = torch.from_numpy(fd32.input.copy()).view(torch.float32).view(2, 3, 224, 224).to(torch.bfloat16)
    x16 = dnn._input_view(torch.from_numpy(fd16.input.copy()).view(torch.bfloat16), 2, fd16)
    assert torch.equal(x16, x32) and x16.is_contiguous(memory_format=torch.channels_last)
