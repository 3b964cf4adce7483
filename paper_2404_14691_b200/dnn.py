"""ResNet-50 inference as a SAGE function (BASELINE cfg 3).

The reference's resnet50 is a calibrated record (97.7 MB RO, 11.9 MB
writable, 24.3 ms compute; functions.py:154, ref PAPER.md Table 3).  Here it
is a real function: random-init torchvision ResNet-50 weights (params +
BN buffers, 102,440,608 B fp32) are the packed DB record, landed as one RO
segment by the `land` kernel; COMPUTE runs the network with PyTorch on the
invocation's pooled stream over ZERO-COPY views of that segment
(`torch.func.functional_call` with tensors built from
`__cuda_array_interface__`), so concurrent invocations share one copy of the
weights -- the RO sharing SAGE is about.  PyTorch (cuDNN convolutions) is used
only for the DNN body, as the north star allows; activations come from
PyTorch's caching allocator, outside the segment pool.
"""
from __future__ import annotations

import numpy as np

from .dataplane import FunctionData
from .functions import FunctionSpec
from .layout import SegmentLayout

MIB = 1 << 20


def _mb(nbytes: int) -> float:
    return -(-nbytes * 1_000_000 // MIB) / 1_000_000


def _state(seed: int):
    import torch
    import torchvision
    torch.manual_seed(seed)
    model = torchvision.models.resnet50(weights=None).eval()
    sd = model.state_dict()
    names = list(sd.keys())
    arrays = [sd[n].detach().cpu().contiguous().numpy() for n in names]
    return names, arrays


def _bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bit patterns (round to nearest even, torch's cast)."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).view(torch.int16).numpy()


def resnet50(batch: int = 8, seed: int = 0, name: str = "resnet50_real", dtype: str = "fp32",
             engine: str | None = None):
    """(FunctionSpec, FunctionData) for ResNet-50 inference on a batch of
    224x224 images; the DB record packs the state dict back to back.
    dtype "fp32": 102.4 MB of weights, fp32 input; "bf16": the weights and
    the input in bfloat16 (51.2 MB, half the PCIe bytes), packed
    channels-last (filters OHWI, input NHWC: meta["layout"] == "nhwc"),
    logits returned in fp32 (BASELINE.json: BF16 outputs within rtol 1e-2).
    engine: "native" (BF16 default) runs the body as the registered program of
    tcgen05 convolutions (csrc/resnet.cu, csrc/conv_tc.cu); "torch" (FP32
    default) runs PyTorch / cuDNN over zero-copy views, with TF32 off."""
    if dtype not in ("fp32", "bf16"):
        raise ValueError(f"resnet50: dtype must be fp32 or bf16, not {dtype!r}")
    engine = engine or ("native" if dtype == "bf16" else "torch")
    if engine == "native":
        if dtype != "bf16":
            raise ValueError("resnet50: the native engine runs the BF16 record")
        return resnet50_native(batch, seed, name)
    names, arrays = _state(seed)
    shapes = [a.shape for a in arrays]            # logical (NCHW / OIHW) shapes
    dtypes = [a.dtype.str for a in arrays]
    if dtype == "bf16":
        # channels-last record: conv filters stored OHWI, the input NHWC, so
        # the zero-copy views feed cuDNN's NHWC tensor-core kernels (a batch-8
        # graph replay: 1.12 ms vs 1.38 ms NCHW, profiles/r1_resnet50_body_formats.jsonl)
        arrays = [_bf16_bits(a.transpose(0, 2, 3, 1) if a.ndim == 4 else a) if a.dtype == np.float32 else a
                  for a in arrays]
        dtypes = ["bf16" if d.endswith("f4") else d for d in dtypes]
    sizes = [a.nbytes for a in arrays]
    layout = SegmentLayout.packed(sizes, align=256, names=tuple(names))
    db = layout.pack(arrays)
    rng = np.random.Generator(np.random.PCG64(seed + 1))
    x = rng.standard_normal((batch, 3, 224, 224), dtype=np.float32)
    if dtype == "bf16":
        x = _bf16_bits(x.transpose(0, 2, 3, 1))
    out_bytes = batch * 1000 * 4
    data = FunctionData(layout, db, body="resnet50", args=(batch,), input=x.reshape(-1).view(np.uint8),
                        out_bytes=out_bytes)
    data.meta = {"shapes": shapes, "dtypes": dtypes, "names": names, "compute": dtype,
                 "layout": "nhwc" if dtype == "bf16" else "nchw"}
    spec = FunctionSpec(name=name, ro_mem_mb=_mb(layout.seg_bytes),
                        writable_mem_mb=_mb(x.nbytes + out_bytes + 4096), compute_ms=24.3,
                        input_bytes_host_mb=_mb(x.nbytes), input_bytes_pcie_mb=_mb(x.nbytes), body="resnet50")
    return spec, data


_STAGES = ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2))   # (planes, blocks, stride) of layer1..4


def stem_s2d_filter(w: np.ndarray) -> np.ndarray:
    """The stem's 7x7 stride-2 pad-3 filter [64][3][7][7] (OIHW) as the 4x4
    stride-1 filter over the 2x2 space-to-depth input (SAGE_CONV_S2D):
    [64][a][b][dr][ds][c] = w[c][2a+dr-1][2b+ds-1], zero outside the 7x7
    window and for the padded channel c = 3; flattened to [64][256]."""
    o = w.shape[0]
    out = np.zeros((o, 4, 4, 2, 2, 4), np.float32)
    for a_ in range(4):
        for dr in range(2):
            r = 2 * a_ + dr - 1
            if not 0 <= r < 7:
                continue
            for b_ in range(4):
                for ds in range(2):
                    sx = 2 * b_ + ds - 1
                    if 0 <= sx < 7:
                        out[:, a_, b_, dr, ds, :3] = w[:, :, r, sx]
    return out.reshape(o, 256)


def stem_s2d_input(x_nhwc: np.ndarray) -> np.ndarray:
    """NHWC [N, H, W, 3] -> [N, H/2, W/2, 16] with channel (dr*2+ds)*4 + c
    = x[2i+dr, 2j+ds, c] (c = 3 zero): what the program's S2D_INPUT op
    computes on the device (numpy form for tests)."""
    n, h, w, _ = x_nhwc.shape
    out = np.zeros((n, h // 2, w // 2, 2, 2, 4), x_nhwc.dtype)
    for dr in range(2):
        for ds in range(2):
            out[:, :, :, dr, ds, :3] = x_nhwc[:, dr::2, ds::2, :]
    return out.reshape(n, h // 2, w // 2, 16)


def resnet50_native(batch: int = 8, seed: int = 0, name: str = "resnet50_real"):
    """The BF16 ResNet-50 function whose body is a native program (no
    PyTorch at run time).  Record: every conv filter OHWI bf16 in place, the
    stem's filter as the 4x4 stride-1 filter over its 2x2 space-to-depth
    input ([64][4][4][16], `stem_s2d_filter`: the S2D mode of
    csrc/conv_tc.cu), batch-norm parameters and the classifier in bf16.
    Request: the images NHWC bf16.  Writable: the image, the fp32 logits and
    the activation workspace of the program."""
    names, arrays = _state(seed)
    sd = dict(zip(names, arrays))
    rec_names, rec = [], []
    for n in names:
        a = sd[n]
        if a.dtype != np.float32:
            continue                    # num_batches_tracked: not used at inference
        if n == "conv1.weight":
            a = stem_s2d_filter(a)
        elif a.ndim == 4:
            a = a.transpose(0, 2, 3, 1)   # OIHW -> OHWI
        rec_names.append(n)
        rec.append(_bf16_bits(a))
    layout = SegmentLayout.packed([a.nbytes for a in rec], align=256, names=tuple(rec_names))
    db = layout.pack(rec)
    off = dict(zip(rec_names, layout.dst_off))
    ops, bufs = _native_program(off, batch)
    rng = np.random.Generator(np.random.PCG64(seed + 1))
    x = _bf16_bits(rng.standard_normal((batch, 3, 224, 224), dtype=np.float32).transpose(0, 2, 3, 1))
    out_bytes = batch * 1000 * 4
    ws = sum(-(-b // 256) * 256 for b in bufs)
    data = FunctionData(layout, db, body="resnet50_native", args=(0, batch), input=x.reshape(-1).view(np.uint8),
                        out_bytes=out_bytes)
    data.scratch_bytes = ws
    data.meta = {"names": rec_names, "compute": "bf16", "layout": "nhwc", "program": (ops, bufs),
                 "state_seed": seed}
    spec = FunctionSpec(name=name, ro_mem_mb=_mb(layout.seg_bytes),
                        writable_mem_mb=_mb(x.nbytes + 16 + out_bytes + ws + 4096), compute_ms=24.3,
                        input_bytes_host_mb=_mb(x.nbytes), input_bytes_pcie_mb=_mb(x.nbytes),
                        body="resnet50_native")
    return spec, data


def _native_program(off: dict, batch: int):
    """The op list of one forward (sage_net_op fields as dicts) and the
    workspace buffer sizes.  Buffers rotate so a bottleneck's input stays
    live until its residual add."""
    from . import _lib
    N = batch
    act = N * 112 * 112 * 64 * 2          # the largest activation (stem out = layer1 out)
    bufs = [N * 112 * 112 * 16 * 2] + [act] * 5 + [N * 2048 * 4]
    s2d_in, feat = _lib.NET_BUF_WS0, _lib.NET_BUF_WS0 + 6
    A = [_lib.NET_BUF_WS0 + 1 + i for i in range(5)]
    ops = [dict(kind=_lib.NET_S2D_INPUT, src=_lib.NET_BUF_INPUT, dst=s2d_in, n=N, h=224, w=224)]

    def conv(src, dst, prefix, bn, cin, cout, k, stride, pad, h, relu, res=-1, mode=0):
        g = bn + "."
        ops.append(dict(kind=_lib.NET_CONV, src=src, dst=dst, res=res, w_off=off[prefix + ".weight"],
                        g_off=off[g + "weight"], b_off=off[g + "bias"], m_off=off[g + "running_mean"],
                        v_off=off[g + "running_var"], eps=1e-5, n=N, h=h, w=h, cin=cin, cout=cout, r=k, s=k,
                        stride=stride, pad=pad, relu=int(relu), mode=mode))

    # the stem: 7x7 stride 2 over 224^2 x 3 == 4x4 stride 1 over the 112^2 x 16 space-to-depth input
    conv(s2d_in, A[0], "conv1", "bn1", 16, 64, 4, 1, 2, 112, True, mode=_lib.CONV_S2D)
    ops.append(dict(kind=_lib.NET_MAXPOOL, src=A[0], dst=A[1], n=N, h=112, w=112, cin=64))
    cur, h, cin = A[1], 56, 64
    for li, (planes, blocks, stride) in enumerate(_STAGES):
        for bi in range(blocks):
            s = stride if bi == 0 else 1
            p = f"layer{li + 1}.{bi}."
            t1, t2, o, ds = [b for b in A if b != cur][:4]
            res = cur
            if bi == 0:
                conv(cur, ds, p + "downsample.0", p + "downsample.1", cin, 4 * planes, 1, s, 0, h, False)
                res = ds
            conv(cur, t1, p + "conv1", p + "bn1", cin, planes, 1, 1, 0, h, True)
            conv(t1, t2, p + "conv2", p + "bn2", planes, planes, 3, s, 1, h, True)
            h //= s
            conv(t2, o, p + "conv3", p + "bn3", planes, 4 * planes, 1, 1, 0, h, True, res=res)
            cur, cin = o, 4 * planes
    ops.append(dict(kind=_lib.NET_POOL_FC, src=cur, dst=_lib.NET_BUF_OUT, res=feat, w_off=off["fc.weight"],
                    b_off=off["fc.bias"], n=N, h=h, w=h, cin=cin, cout=1000))
    return ops, bufs


def native_handle(fd: FunctionData) -> int:
    """The library handle of the function's program (created once)."""
    h = fd.meta.get("net_handle")
    if h:
        return h
    from . import _lib
    ops, bufs = fd.meta["program"]
    arr = (_lib.NetOp * len(ops))()
    for i, op in enumerate(ops):
        for k in ("g_off", "b_off", "m_off", "v_off", "w_off"):
            op.setdefault(k, (1 << 64) - 1 if k == "g_off" else 0)
        op.setdefault("res", -1)
        for k, v in op.items():
            setattr(arr[i], k, v)
    out, ws = _lib.H(0), _lib.u64(0)
    _lib.check(_lib.lib().sage_net_create(arr, len(ops), (_lib.u64 * len(bufs))(*bufs), len(bufs),
                                          _lib.C.byref(out), _lib.C.byref(ws)), "sage_net_create")
    if ws.value > fd.scratch_bytes:
        raise RuntimeError(f"native resnet workspace {ws.value} B exceeds the reserved {fd.scratch_bytes} B")
    fd.meta["net_handle"] = out.value
    fd.args = (out.value, fd.args[1])
    return out.value


def reference_cpu(fd: FunctionData, x_bytes: np.ndarray):
    """torch-CPU fp32 logits of the function's network on its (bf16) weights
    and a (bf16 NHWC) request -- the parity reference of tests/ (not used on
    the product path)."""
    import torch
    import torchvision
    torch.manual_seed(fd.meta["state_seed"])
    model = torchvision.models.resnet50(weights=None).eval()
    with torch.no_grad():
        for p in list(model.parameters()) + list(model.buffers()):
            if p.dtype == torch.float32:
                p.copy_(p.to(torch.bfloat16).float())
    n = fd.args[1]
    x = torch.from_numpy(np.ascontiguousarray(x_bytes).view(np.int16).copy()).view(torch.bfloat16).float()
    x = x.view(n, 224, 224, 3).permute(0, 3, 1, 2).contiguous()
    with torch.inference_mode():
        return model(x).numpy()


def _as_logical(t, shp, fd: FunctionData):
    """A flat parameter view shaped to its logical (PyTorch) shape; 4-D
    filters of a channels-last record become OIHW views with NHWC strides."""
    if len(shp) == 4 and fd.meta.get("layout") == "nhwc":
        o, i, h, w = shp
        return t.view(o, h, w, i).permute(0, 3, 1, 2)
    return t.view(shp) if len(shp) else t.view(())


def _input_view(t, batch: int, fd: FunctionData):
    if fd.meta.get("layout") == "nhwc":
        return t.view(batch, 224, 224, 3).permute(0, 3, 1, 2)
    return t.view(batch, 3, 224, 224)


def _torch_dtype(tag: str):
    import torch
    return torch.int64 if tag.endswith("i8") else torch.bfloat16 if tag == "bf16" else torch.float32


def _compute_dtype(fd: FunctionData):
    import torch
    dt = torch.bfloat16 if fd.meta.get("compute") == "bf16" else torch.float32
    if dt is torch.float32:
        # the FP32 function computes in FP32: cuDNN / cuBLAS would otherwise
        # run its convolutions in TF32 (10-bit mantissa) by default
        torch.backends.cudnn.allow_tf32 = False
        torch.backends.cuda.matmul.allow_tf32 = False
    return dt


class _CudaBuf:
    """Minimal __cuda_array_interface__ over a raw device range (zero copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                         "strides": None}


_MODELS: dict = {}


def _skeleton():
    import torch
    import torchvision
    m = _MODELS.get("resnet50")
    if m is None:
        with torch.device("meta"):
            m = torchvision.models.resnet50(weights=None).eval()
        _MODELS["resnet50"] = m
    return m


def view(ptr: int, nbytes: int, device):
    import torch
    return torch.as_tensor(_CudaBuf(ptr, nbytes), device=device)


def _params(fd: FunctionData, ro_ptr: int, dev, plane: int):
    """Zero-copy parameter views over the landed segment (cached per segment
    and logical GPU -- several logical planes may share one device)."""
    import torch
    key = (id(fd), ro_ptr, plane)
    params = _PARAMS.get(key)
    if params is None:
        meta, lay = fd.meta, fd.layout
        seg = view(ro_ptr, lay.seg_bytes, dev)
        params = {}
        for n, off, ln, shp, dt in zip(meta["names"], lay.dst_off, lay.length, meta["shapes"], meta["dtypes"]):
            params[n] = _as_logical(seg[off:off + ln].view(_torch_dtype(dt)), shp, fd)
        for k in [k for k in _PARAMS if k[0] == key[0] and k[2] == key[2]]:
            del _PARAMS[k]         # the function's segment moved on this GPU
        _PARAMS[key] = params
    return params


class _GraphEntry:
    """One captured forward: static input / output, the executable graph, and
    the event that ends its last use (reuses of an entry are ordered)."""

    __slots__ = ("graph", "x", "y", "done")

    def __init__(self, graph, x, y):
        self.graph, self.x, self.y, self.done = graph, x, y, None


class _GraphPool:
    """CUDA graphs of the ResNet-50 forward over ONE landed weight segment.
    Launches of one executable graph serialise, so GRAPHS_PER_SEGMENT entries
    are used round robin to let concurrent invocations overlap."""

    def __init__(self):
        self.entries: list[_GraphEntry] = []
        self.next = 0


import os as _os
GRAPHS_PER_SEGMENT = int(_os.environ.get("SAGE_DNN_GRAPHS_PER_SEGMENT", "4"))
_GRAPHS: dict = {}
CAPTURES = {"count": 0, "seconds": 0.0}   # graph captures so far (reported by experiments.cfg3)


_WARM: set = set()


def prewarm(fd: FunctionData, device_index: int) -> None:
    """Registration-time warm-up (Simulation.prepare): one eager forward and
    one throwaway graph capture with the function's weights copied to the
    device, so cuDNN / cuBLAS initialisation and kernel loading (measured
    ~2 s on a fresh process) happen before the first invocation instead of
    inside its COMPUTE.  Invocations still capture their own graphs over the
    landed segment (its address is known only then)."""
    import numpy as np
    import torch
    if (id(fd), device_index) in _WARM:
        return
    dev = torch.device("cuda", device_index)
    meta, lay = fd.meta, fd.layout
    params = {}
    for n, off, ln, shp, dt in zip(meta["names"], lay.src_off, lay.length, meta["shapes"], meta["dtypes"]):
        raw = torch.from_numpy(fd.db[off:off + ln].copy()).view(_torch_dtype(dt))
        params[n] = _as_logical(raw, shp, fd).to(dev)
    model = _skeleton()
    side = torch.cuda.Stream(device=dev)
    x = _static_input(fd.args[0], dev, fd)
    with torch.cuda.stream(side), torch.inference_mode():
        for _ in range(2):
            torch.func.functional_call(model, params, (x,))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
            torch.func.functional_call(model, params, (x,))
        g.replay()
    side.synchronize()
    del g, params
    _WARM.add((id(fd), device_index))


def _graphs_enabled() -> bool:
    import os
    return os.environ.get("SAGE_DNN_GRAPHS", "1") != "0"


def _static_input(batch: int, dev, fd: FunctionData):
    import torch
    x = torch.zeros((batch, 3, 224, 224), device=dev, dtype=_compute_dtype(fd))
    return x.contiguous(memory_format=torch.channels_last) if fd.meta.get("layout") == "nhwc" else x


def _capture(model, params, batch: int, dev, ext, fd: FunctionData) -> _GraphEntry:
    """Warm up (cuDNN algorithm choice, allocations) and capture one forward
    on a side stream ordered after the invocation's stream (the segment has
    landed there).  Capture is thread-local: the library's issuer and
    completion threads keep calling CUDA meanwhile."""
    import torch
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(ext)
    x = _static_input(batch, dev, fd)
    with torch.cuda.stream(side), torch.inference_mode():
        for _ in range(2):
            torch.func.functional_call(model, params, (x,))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
            y = torch.func.functional_call(model, params, (x,))
    ext.wait_stream(side)
    return _GraphEntry(g, x, y)


def run_resnet50(fd: FunctionData, ro_ptr: int, in_ptr: int, out_ptr: int, stream_ptr: int, device_index: int,
                 plane: int = 0) -> None:
    """Enqueue one ResNet-50 forward on the invocation's stream, reading the
    weights in place from the landed segment and writing logits to out.

    Default: replay a CUDA graph captured over this segment (one graph launch
    + two 16-B-vector copies instead of ~300 eager kernel launches from
    Python); the first invocations over a newly landed segment capture the
    graphs.  SAGE_DNN_GRAPHS=0 runs the forward eagerly."""
    import torch
    dev = torch.device("cuda", device_index)
    params = _params(fd, ro_ptr, dev, plane)
    batch = fd.args[0]
    x = _input_view(view(in_ptr, fd.input_bytes, dev).view(_compute_dtype(fd)), batch, fd)
    out = view(out_ptr, fd.out_bytes, dev).view(torch.float32).view(batch, 1000)
    model = _skeleton()
    ext = torch.cuda.ExternalStream(stream_ptr, device=dev)
    if not _graphs_enabled():
        with torch.cuda.stream(ext), torch.inference_mode():
            out.copy_(torch.func.functional_call(model, params, (x,)).float())
        return
    key = (id(fd), ro_ptr, plane)
    pool = _GRAPHS.get(key)
    if pool is None:
        for k in [k for k in _GRAPHS if k[0] == key[0] and k[2] == key[2]]:
            del _GRAPHS[k]         # graphs over a segment that has gone
        pool = _GRAPHS[key] = _GraphPool()
    if len(pool.entries) < GRAPHS_PER_SEGMENT:
        import time
        t0 = time.perf_counter()
        pool.entries.append(_capture(model, params, batch, dev, ext, fd))
        CAPTURES["count"] += 1
        CAPTURES["seconds"] += time.perf_counter() - t0
    entry = pool.entries[pool.next % len(pool.entries)]
    pool.next += 1
    with torch.cuda.stream(ext):
        if entry.done is not None:
            ext.wait_event(entry.done)
        entry.x.copy_(x)
        entry.graph.replay()
        out.copy_(entry.y)
        entry.done = torch.cuda.Event()
        entry.done.record(ext)


_PARAMS: dict = {}
