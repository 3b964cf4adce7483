"""How does the copy engine arbitrate H2D copies queued on different streams?
(plumbing probe, torch copies only).  Stream A gets 17 x 8 MiB H2D chunks,
stream B then 10 x 4 MiB; per-copy completion times show FIFO vs interleave.
Variants: B enqueued first, B with higher stream priority, D2H traffic on a
third stream."""
import json
import torch

MiB = 1 << 20
hA = torch.empty(17 * 8 * MiB, dtype=torch.uint8).pin_memory()
hB = torch.empty(10 * 4 * MiB, dtype=torch.uint8).pin_memory()
hC = torch.empty(64 * MiB, dtype=torch.uint8).pin_memory()
dA = torch.empty_like(hA, device="cuda")
dB = torch.empty_like(hB, device="cuda")
dC = torch.empty(64 * MiB, dtype=torch.uint8, device="cuda")
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)


def run(order="AB", prio_b=0, d2h=False):
    sA, sB, sC = torch.cuda.Stream(), torch.cuda.Stream(priority=prio_b), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in (sA, sB, sC):
        s.wait_event(t0)
    evA, evB = [], []

    def qa():
        with torch.cuda.stream(sA):
            for k in range(17):
                dA[k * 8 * MiB:(k + 1) * 8 * MiB].copy_(hA[k * 8 * MiB:(k + 1) * 8 * MiB], non_blocking=True)
                e = torch.cuda.Event(enable_timing=True); e.record(); evA.append(e)

    def qb():
        with torch.cuda.stream(sB):
            for k in range(10):
                dB[k * 4 * MiB:(k + 1) * 4 * MiB].copy_(hB[k * 4 * MiB:(k + 1) * 4 * MiB], non_blocking=True)
                e = torch.cuda.Event(enable_timing=True); e.record(); evB.append(e)
    if d2h:
        with torch.cuda.stream(sC):
            for k in range(4):
                hC.copy_(dC, non_blocking=True)
    for c in order:
        (qa if c == "A" else qb)()
    torch.cuda.synchronize()
    return {"A_ms": [round(t0.elapsed_time(e), 3) for e in evA], "B_ms": [round(t0.elapsed_time(e), 3) for e in evB]}


out = {"priority_range": [lo, hi]}
for _ in range(2):
    run()
out["AB"] = run("AB")
out["BA"] = run("BA")
out["AB_prioB"] = run("AB", prio_b=hi)
out["AB_d2h"] = run("AB", d2h=True)
print(json.dumps(out))
