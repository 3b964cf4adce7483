"""ResNet-50 batch-8 inference on one B200: CUDA-graph replay throughput by
dtype / memory format / cudnn.benchmark, one stream and 8 concurrent streams
(probe for dnn.py's body choices; torchvision model, random weights)."""
import json
import sys

import torch
import torchvision

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def bench(dtype, cl, benchmark, streams):
    torch.backends.cudnn.benchmark = benchmark
    m = torchvision.models.resnet50(weights=None).eval().cuda().to(dtype)
    fmt = torch.channels_last if cl else torch.contiguous_format
    m = m.to(memory_format=fmt)
    graphs = []
    for s in range(streams):
        x = torch.randn(B, 3, 224, 224, device="cuda", dtype=dtype).to(memory_format=fmt)
        st = torch.cuda.Stream()
        with torch.no_grad(), torch.cuda.stream(st):
            for _ in range(3):
                m(x)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.no_grad(), torch.cuda.graph(g, stream=st):
            y = m(x)
        graphs.append((g, st, x, y))
    torch.cuda.synchronize()
    reps = 40
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        cur = torch.cuda.current_stream()
        for g, st, _, _ in graphs:
            st.wait_stream(cur)
        for _ in range(reps):
            for g, st, _, _ in graphs:
                g.replay()
        for g, st, _, _ in graphs:
            cur.wait_stream(st)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    n = reps * streams
    return {"dtype": str(dtype).split(".")[-1], "channels_last": cl, "cudnn_benchmark": benchmark, "streams": streams,
            "batch": B, "ms_per_inv": round(ms / n, 4), "img_per_s": round(n * B / ms * 1e3)}


for dtype in (torch.float32, torch.bfloat16):
    for cl in (False, True):
        for bm in (False, True):
            for streams in (1, 8):
                print(json.dumps(bench(dtype, cl, bm, streams)), flush=True)
