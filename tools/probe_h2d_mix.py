"""PCIe ceiling for the cfg-2 e2e transfer mix (plumbing probe, torch copies):
64 x 4 MiB H2D back to back on one stream, alone and with 4 MiB / 16 MiB D2H
copies streaming concurrently on another; pinned memory from cudaHostAlloc
(torch pin_memory) vs cudaHostRegister'd numpy."""
import json
import numpy as np
import torch

MiB = 1 << 20
n, c = 64, 4 * MiB
h_in = torch.empty(n * c, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n * 16 * MiB, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n * c, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n * 16 * MiB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(d2h_chunk=0, d2h_n=0):
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    with torch.cuda.stream(s1):
        for k in range(n):
            d_in[k * c:(k + 1) * c].copy_(h_in[k * c:(k + 1) * c], non_blocking=True)
        e1.record()
    with torch.cuda.stream(s2):
        for k in range(d2h_n):
            h_out[k * d2h_chunk:(k + 1) * d2h_chunk].copy_(d_out[k * d2h_chunk:(k + 1) * d2h_chunk], non_blocking=True)
        e2.record()
    torch.cuda.synchronize()
    t_h = e0.elapsed_time(e1)
    t_d = e0.elapsed_time(e2)
    return {"h2d_GBps": round(n * c / t_h / 1e6, 1), "h2d_ms": round(t_h, 3),
            "d2h_GBps": round(d2h_n * d2h_chunk / t_d / 1e6, 1) if d2h_n else None, "d2h_ms": round(t_d, 3)}


for _ in range(2):
    run()
out = {"h2d_4MiB_alone": run(), "h2d_with_d2h_4MiB": run(4 * MiB, 64), "h2d_with_d2h_16MiB": run(16 * MiB, 16),
       "h2d_with_d2h_16MiB_x32": run(16 * MiB, 32)}
print(json.dumps(out))
