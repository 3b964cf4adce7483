"""Is PCIe H2D + D2H concurrency full duplex on this box?  (plumbing probe,
torch copies only).  Prints GB/s for H2D alone, D2H alone, both at once on
separate streams, and the 64 x 8 MiB chunked pattern of the cfg-2 burst."""
import json
import torch

MiB = 1 << 20
n = 512 * MiB
h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)


def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


def chunked():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    c = 8 * MiB
    for k in range(64):
        with torch.cuda.stream(s1):
            d_a[k * c:(k + 1) * c].copy_(h_src[k * c:(k + 1) * c], non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst[k * c:(k + 1) * c].copy_(d_b[k * c:(k + 1) * c], non_blocking=True)


out = {}
t = timeit(h2d)
out["h2d_GBps"] = round(n / t / 1e9, 2)
t = timeit(d2h)
out["d2h_GBps"] = round(n / t / 1e9, 2)
t = timeit(both)
out["both_total_GBps"] = round(2 * n / t / 1e9, 2)
out["both_ms"] = round(t * 1e3, 2)
t = timeit(chunked)
out["chunked_total_GBps"] = round(2 * n / t / 1e9, 2)
print(json.dumps(out))
