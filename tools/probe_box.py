"""One-off probe of the GPU box: host cores, PCIe H2D bandwidth (pinned/pageable),
cuCtxCreate cost. Prints a JSON blob; used to size the data plane."""
import json, os, subprocess, time, ctypes
import torch
out = {"nproc": os.cpu_count()}
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()[:16]
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
    out["smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,memory.total,pcie.link.gen.max,pcie.link.width.max,clocks.sm,clocks.max.sm", "--format=csv"], capture_output=True, text=True).stdout
    out["free"] = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout
except Exception as e:
    out["err"] = str(e)
dev = torch.device("cuda:0")
torch.cuda.init()
for nbytes in (1 << 20, 16 << 20, 100 << 20, 1 << 30):
    h_pin = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_pag = torch.empty(nbytes, dtype=torch.uint8); h_pag.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for name, h in (("pinned", h_pin), ("pageable", h_pag)):
        d.copy_(h, non_blocking=False); torch.cuda.synchronize()
        t = time.perf_counter(); reps = 5
        for _ in range(reps):
            d.copy_(h, non_blocking=(name == "pinned"))
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / reps
        out[f"h2d_{name}_{nbytes>>20}MiB_GBps"] = round(nbytes / dt / 1e9, 2)
    h_pin2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5):
        h_pin2.copy_(d, non_blocking=True)
    torch.cuda.synchronize(); out[f"d2h_pinned_{nbytes>>20}MiB_GBps"] = round(nbytes * 5 / (time.perf_counter() - t) / 1e9, 2)
    # host memcpy bandwidth (1 thread)
    a = torch.empty(nbytes, dtype=torch.uint8); a.fill_(3); b = torch.empty_like(a)
    torch.set_num_threads(1); t = time.perf_counter(); b.copy_(a); out[f"memcpy1t_{nbytes>>20}MiB_GBps"] = round(nbytes / (time.perf_counter() - t) / 1e9, 2)
    del h_pin, h_pag, d, h_pin2, a, b
cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
devh = ctypes.c_int()
cuda.cuDeviceGet(ctypes.byref(devh), 0)
ts = []
for i in range(4):
    ctx = ctypes.c_void_p()
    t = time.perf_counter()
    r = cuda.cuCtxCreate_v2(ctypes.byref(ctx), 0, devh)
    free = ctypes.c_size_t(); tot = ctypes.c_size_t()
    cuda.cuMemGetInfo_v2(ctypes.byref(free), ctypes.byref(tot))
    t1 = time.perf_counter()
    cuda.cuCtxDestroy_v2(ctx)
    t2 = time.perf_counter()
    ts.append((r, round((t1 - t) * 1e3, 2), round((t2 - t1) * 1e3, 2)))
out["cuCtxCreate_ms(ret,create,destroy)"] = ts
print(json.dumps(out, indent=1))
