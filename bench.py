"""Benchmark of the B200 SAGE data plane (driver contract: one JSON line).

Workload (BASELINE.json configs[1], "cfg 2"): a burst of 64 concurrent
invocations of the Parboil-style sgemm / stencil / spmv mix on one GPU with
shared read-only segments (paper_2404_14691_b200/parboil.py).  One STEP = one
burst submitted at one instant through the public API
(`Simulation.submit_many`) and drained, starting from COLD (no resident
segment: each step performs the three leader read-only loads and 64 input
loads, parallel setup, 64 kernels, 64 result returns).

  value  invocations/s with every DB record and input already resident in
         HBM (loads land from HBM, no PCIe) -- the device pipeline
  e2e    invocations/s through the same API with HOST buffers: pageable DB
         records + request payloads, CPU_LOAD memcpy + H2D + land inside the
         timed region, results D2H into pinned memory
Both are whole-job aggregates over all ranks (max-over-ranks device time).

Extra keys: p50/p99 setup latency (compute_begin - arrival), the cfg-1
SAGE-vs-FixedGSL setup comparison (16 concurrent 100 MiB cold starts,
`--cfg1`), per-kernel rooflines measured live with CUDA events, and the CPU
baseline (oracle/cpu_path.py: the same burst served on the host cores, each
invocation's copy + unpack + checksum and fp32 body on its own core).

`--impl reference` times that host-only serving path as the reference arm
(full bursts, all cores) and prints its own line.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "invocations/sec (p50/p99 setup latency alongside)"
UNIT = "invocations/s"


def _rank_env():
    """One process per GPU: every device stays visible (peers' exported pages
    then map over NVLink like NCCL's own), this rank's library planes start
    at device LOCAL_RANK (SAGE_DEVICE_OFFSET)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not _shared_gpu():
        os.environ["SAGE_DEVICE_OFFSET"] = str(local)
    return rank, world, local


def _my_device() -> int:
    """Physical device index of this rank (torch / NVML numbering)."""
    return int(os.environ.get("SAGE_DEVICE_OFFSET", "0"))


def _shared_gpu() -> bool:
    """Test mode (SAGE_BENCH_SHARE_GPU=1): every rank on device 0 and gloo for
    the rank plumbing, so the N > 1 path (fan-out included) runs on a
    one-GPU box.  Not a measurement mode."""
    return os.environ.get("SAGE_BENCH_SHARE_GPU") == "1"


def _reduce_device(dist) -> str:
    import torch
    return "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"


# --------------------------------------------------------------- clocks -------
class ClockSampler:
    """SM clock + throttle reasons sampled DURING a timed region: NVML polled
    every 5 ms from a thread (the value leg lasts only tens of ms), else
    `nvidia-smi -lms 100`."""
    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, gpu: int = 0):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple] = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._nvml = (pynvml, h, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            return self
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu),
                                          "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                                          "clocks_event_reasons.hw_thermal_slowdown,"
                                          "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv, h, _ = self._nvml
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), r))
            except Exception:
                pass
            self._stop.wait(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        sm, smax, reasons = [], None, set()
        if self._nvml is not None:
            self._stop.set()
            self._t.join(timeout=2)
            nv, _, smax = self._nvml
            for clk, r in self.samples:
                sm.append(clk)
                for name, attr in self.REASONS.items():
                    if r & getattr(nv, attr, 0):
                        reasons.add(name)
            src = "nvml 5 ms"
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            for ln in self.lines:
                p = [x.strip() for x in ln.split(",")]
                if len(p) < 6:
                    continue
                try:
                    sm.append(float(p[0]))
                    smax = float(p[1])
                except ValueError:
                    continue
                for n, v in zip(self.REASONS, p[2:6]):
                    if v.lower() == "active":
                        reasons.add(n)
            src = "nvidia-smi 100 ms"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": src}


# ------------------------------------------------------------- our arm --------
def burst_names(table, burst: int):
    names = sorted(table)
    return [names[k % len(names)] for k in range(burst)]


def run_steps(sim, names, steps: int, payloads=None, marks=None):
    """`steps` cold bursts; returns the invocations.  `marks`: a list that
    receives one device mark (event handle) after each burst."""
    from paper_2404_14691_b200 import _lib
    out = []
    for _ in range(steps):
        if sim.sharing is not None:   # start every burst cold (no resident segment)
            for r in list(sim.sharing.residents.values()):
                sim.sharing.evict(r)
        invs = sim.submit_many(names, payloads=payloads)
        sim.drain()
        box = getattr(sim.dataplane, "box", None)
        if box is not None:
            box.reap()           # received segments are no longer read
        bad = [i for i in invs if i.outcome != "completed"]
        if bad:
            raise RuntimeError(f"{len(bad)} invocations did not complete: {bad[0].fail_reason}")
        out += invs
        if marks is not None:
            m = _lib.H()
            _lib.check(_lib.lib().sage_mark(0, _lib.C.byref(m)), "mark")
            marks.append(m.value)
    return out


def timed(sim, names, steps, warmup, dist, payloads=None):
    from paper_2404_14691_b200 import _lib
    from paper_2404_14691_b200 import device as D
    L = _lib.lib()
    run_steps(sim, names, warmup, payloads)
    # no cyclic-GC pass inside the timed region (a serving process tunes its
    # collector the same way); refcounting still frees every finished record
    gc.collect()
    gc.disable()
    _lib.check(L.sage_stats_reset(), "stats_reset")
    box = getattr(sim.dataplane, "box", None)
    box_in0 = box.bytes_in if box is not None else 0
    barrier(dist)
    _lib.check(L.sage_device_sync(0), "device_sync")
    a = _lib.H()
    _lib.check(L.sage_mark(0, _lib.C.byref(a)), "mark")
    marks = [a.value]
    invs = run_steps(sim, names, steps, payloads, marks)
    _lib.check(L.sage_device_sync(0), "device_sync")
    b = _lib.H()
    _lib.check(L.sage_mark(0, _lib.C.byref(b)), "mark")
    D.Event(b.value).sync()
    us = _lib.C.c_double()
    _lib.check(L.sage_event_elapsed(a.value, b.value, _lib.C.byref(us)), "event_elapsed")
    step_ms = []
    for m0, m1 in zip(marks[:-1], marks[1:]):
        _lib.check(L.sage_event_elapsed(m0, m1, _lib.C.byref(d_us := _lib.C.c_double())), "event_elapsed")
        step_ms.append(round(d_us.value / 1e3, 3))
    for m in marks + [b.value]:
        D.Event(m).release()
    gc.enable()
    elapsed = max_over_ranks(dist, us.value)
    timed.step_ms = step_ms
    timed.box_bytes = (box.bytes_in - box_in0) if box is not None else 0
    return elapsed, invs


def kernel_stats():
    from paper_2404_14691_b200 import _lib
    L = _lib.lib()
    out = {}
    for kind, name in enumerate(["land", "touch", "sgemm", "stencil", "spmv", "verify", "gather"]):
        n, t, b = _lib.u64(), _lib.C.c_double(), _lib.u64()
        _lib.check(L.sage_stats_get(0, kind, _lib.C.byref(n), _lib.C.byref(t), _lib.C.byref(b)), "stats_get")
        if n.value:
            out[name] = {"launches": n.value, "total_us": t.value, "work": b.value}
    return out


_BODY_KIND = {"sgemm": 1, "stencil": 2, "spmv": 3}


def body_probe(data, body: str, iters: int = 20) -> dict | None:
    """The function body `body` launched back to back on one pooled stream
    over its landed (HBM-resident) data, right after the timed region: the
    kernel's rate without other invocations sharing the GPU."""
    from paper_2404_14691_b200 import _lib
    from paper_2404_14691_b200 import device as D
    if body not in _BODY_KIND:
        return None
    name = next((n for n in sorted(data) if data[n].body == body), None)
    if name is None:
        return None
    fd = data[name]
    L = _lib.lib()
    seg = D.pool_alloc(0, fd.layout.seg_bytes, _lib.CLASS_READ_ONLY, unaccounted=True)
    inp = D.pool_alloc(0, fd.input_bytes + 256, _lib.CLASS_WRITABLE, unaccounted=True)
    out = D.pool_alloc(0, max(256, fd.out_bytes), _lib.CLASS_WRITABLE, unaccounted=True)
    slot = D.Slot(0)
    try:
        for dst, src, lay, nb in ((seg.dptr, fd.db, fd.layout, None), (inp.dptr, fd.input, None, None)):
            op = D.load(0, dst, src, lay)
            op.wait()
            op.release()
        desc = D.body_desc(_BODY_KIND[body], ro=seg.dptr, ro_bytes=fd.layout.seg_bytes, inp=inp.dptr,
                           inp_bytes=(fd.input_bytes + 15) // 16 * 16, out=out.dptr, out_bytes=max(16, fd.out_bytes),
                           args=fd.args)
        _lib.check(L.sage_stats_reset(), "stats_reset")
        evs = [slot.launch(desc) for _ in range(iters)]
        evs[-1][1].sync()
        for b, e in evs:
            b.release()
            e.release()
        return kernel_stats().get(body)
    finally:
        slot.release()
        for x in (seg, inp, out):
            x.free()


def gather_probe(data, iters: int = 20) -> dict | None:
    """The random-gather ceiling spmv's x accesses run against: the
    diagnostic GATHER body does as many hashed 4-B gathers as spmv has
    non-zeros, from an array of x's size, with no col / val streams
    (tools/gather_micro.cu sweeps the array size and cache hints: the rate
    is flat from 1 to 64 MiB, a per-SM L1TEX miss-issue limit)."""
    from paper_2404_14691_b200 import _lib
    from paper_2404_14691_b200 import device as D
    name = next((n for n in sorted(data) if data[n].body == "spmv"), None)
    if name is None:
        return None
    fd = data[name]
    rows, nnz = int(fd.args[0]), int(fd.args[1])
    elems = 1 << max(0, (rows - 1).bit_length())
    inp = D.pool_alloc(0, elems * 4, _lib.CLASS_WRITABLE, unaccounted=True)
    out = D.pool_alloc(0, 256, _lib.CLASS_WRITABLE, unaccounted=True)
    slot = D.Slot(0)
    try:
        desc = D.body_desc(_lib.BODY_GATHER, ro=0, ro_bytes=0, inp=inp.dptr, inp_bytes=elems * 4, out=out.dptr,
                           out_bytes=16, args=(nnz // 4 * 4,))
        slot.launch(desc)[1].sync()                      # warm: x in L2, module loaded
        _lib.check(_lib.lib().sage_stats_reset(), "stats_reset")
        evs = [slot.launch(desc) for _ in range(iters)]
        evs[-1][1].sync()
        for b, e in evs:
            b.release()
            e.release()
        g = kernel_stats().get("gather")
        if not g:
            return None
        us = g["total_us"] / g["launches"]
        return {"gathers_per_launch": g["work"] // g["launches"], "avg_launch_us": round(us, 2),
                "G_gathers_per_s": round(g["work"] / g["launches"] / us / 1e3, 1), "array_bytes": elems * 4,
                "launches": g["launches"]}
    finally:
        slot.release()
        for x in (inp, out):
            x.free()


def land_probe(data, iters: int = 8, gib: float = 1.0) -> dict:
    """Back-to-back lands of a 1 GiB, 8-tensor segment (8x the L2) from an
    HBM-resident record, timed live (the land kernel away from L2 effects)."""
    import numpy as np

    from paper_2404_14691_b200 import _lib
    from paper_2404_14691_b200 import device as D
    from paper_2404_14691_b200.layout import SegmentLayout
    L = _lib.lib()
    total = int(gib * (1 << 30)) // 4096 * 4096
    lay = SegmentLayout.packed([total // 8 - 37 * k for k in range(8)], align=256)
    db = np.random.default_rng(1).integers(0, 256, lay.packed_bytes, dtype=np.uint8)
    src = D.pool_alloc(0, lay.packed_bytes + 64, _lib.CLASS_WRITABLE, unaccounted=True)
    seg = D.pool_alloc(0, lay.seg_bytes, _lib.CLASS_READ_ONLY, unaccounted=True)
    try:
        up = D.load(0, src.dptr, db, None)
        up.wait()
        up.release()
        _lib.check(L.sage_device_sync(0), "device_sync")
        _lib.check(L.sage_stats_reset(), "stats_reset")
        ops = [D.load(0, seg.dptr, None, lay, device_src=src.dptr, device_src_bytes=lay.packed_bytes)
               for _ in range(iters)]
        sums = {op.wait().checksum for op in ops}
        for op in ops:
            op.release()
        if len(sums) != 1:
            raise RuntimeError("land probe: checksums differ between identical lands")
        s = kernel_stats()["land"]
        s["segment"] = f"synthetic ({lay.seg_bytes} B, {lay.n} ragged tensors, 8x L2)"
        s["d2d_GBps"] = d2d_reference(seg.dptr, src.dptr, min(lay.packed_bytes, lay.seg_bytes))
        return s
    finally:
        seg.free()
        src.free()


def d2d_reference(dst: int, src: int, nbytes: int, iters: int = 20) -> float:
    """Copy-engine D2D of the probe's packed bytes (read + write counted), the
    same-size ceiling next to the 2 GiB copy peak of MEASURED_PEAKS.json."""
    from paper_2404_14691_b200 import _lib
    from paper_2404_14691_b200 import device as D
    L = _lib.lib()
    evs = []
    for _ in range(iters + 1):
        e = _lib.H()
        _lib.check(L.sage_fanout(0, src, 0, dst, nbytes, None, 0, _lib.C.byref(e)), "fanout")
        evs.append(e.value)
    D.Event(evs[-1]).sync()
    us = _lib.C.c_double()
    _lib.check(L.sage_event_elapsed(evs[0], evs[-1], _lib.C.byref(us)), "event_elapsed")
    for e in evs:
        D.Event(e).release()
    return round(2 * nbytes * iters / us.value / 1e3, 1)


_TRAFFIC = {"spmv": "r1_spmv_traffic.json", "land": "r2_land_traffic.json", "sgemm": "r2_sgemm_traffic.json"}


def dominant_roofline(rooflines: dict, stats: dict, peaks: dict, isolated: dict | None = None,
                      gather: dict | None = None, nnz: int = 0) -> dict:
    """`roofline` of the bench contract: the kernel with the largest summed
    device time over the timed region, its achieved rate = algorithmic work
    per launch / mean launch time (CUDA events around every launch on the
    launching stream), DRAM traffic per launch from its committed ncu
    --set full capture when there is one."""
    name = max(stats, key=lambda k: stats[k]["total_us"])
    r = dict(rooflines[name])
    r["kernel"] = name
    if r["bound"] not in ("hbm", "tensor"):     # contract vocabulary; the real limiter stays recorded
        r["limiter"] = r["bound"]
        r["bound"] = "tensor" if r["unit"] == "TFLOP/s" else "hbm"
    r["how"] = (f"{r['launches']} launches inside the timed value leg, CUDA events on each launch's stream; "
                f"launches overlap other invocations' kernels, so per-launch times include contention")
    r["peak_source"] = peaks["source"]
    r["traffic"] = None
    f = ROOT / "profiles" / _TRAFFIC.get(name, "-")
    if f.exists():
        d = json.loads(f.read_text())
        r["traffic"] = d["dram_bytes_read"] + d["dram_bytes_write"]
        r["traffic_source"] = f"profiles/{f.name} (ncu --set full, one launch)"
    if isolated and isolated.get("launches"):
        us = isolated["total_us"] / isolated["launches"]
        per = isolated["work"] / isolated["launches"]
        ach = per / (us * 1e-6) / (1e12 if r["unit"] == "TFLOP/s" else 1e9)
        r["isolated"] = {"achieved": round(ach, 1), "frac": round(ach / r["peak"], 4), "avg_launch_us": round(us, 2),
                         "launches": isolated["launches"],
                         "how": "the same kernel back to back on one stream right after the timed region"}
    ser = ncu_serialized(name)
    if ser and stats[name]["launches"]:
        per = stats[name]["work"] / stats[name]["launches"]
        ach = per / (ser["mean_us"] * 1e-6) / (1e12 if r["unit"] == "TFLOP/s" else 1e9)
        r["serialized"] = {"achieved": round(ach, 1), "frac": round(ach / r["peak"], 4), **ser,
                           "how": "the same kernel's mean duration in the committed ncu launch list of this bench "
                                  "(cold-cache, serialised launches), algorithmic work per launch as above"}
    if name == "spmv" and gather and nnz:
        # the limiter's own ceiling: x gathers per second vs the pure-gather rate
        ceil = gather["G_gathers_per_s"]
        g = {"ceiling_G_gathers_per_s": ceil, "probe": gather,
             "in_burst_G_gathers_per_s": round(nnz / r["avg_launch_us"] / 1e3, 1)}
        g["in_burst_frac"] = round(g["in_burst_G_gathers_per_s"] / ceil, 4)
        if "isolated" in r:
            g["isolated_G_gathers_per_s"] = round(nnz / r["isolated"]["avg_launch_us"] / 1e3, 1)
            g["isolated_frac"] = round(g["isolated_G_gathers_per_s"] / ceil, 4)
        r["gather_roofline"] = g
    return r


_NCU_NAMES = {"spmv": "spmv4_kernel", "sgemm": "sgemm_tf32_kernel", "land": "land_kernel",
              "stencil": "stencil4_kernel"}


def ncu_serialized(name: str, path: str = "profiles/r2_bench_launches.csv") -> dict | None:
    """Mean duration and share of `name`'s launches in a committed ncu launch
    list of this bench (`ncu --metrics gpu__time_duration.sum --csv`)."""
    import csv
    import io
    f = ROOT / path
    if not f.exists() or name not in _NCU_NAMES:
        return None
    text = f.read_text()
    if '"ID"' not in text:
        return None
    rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    mine, total = [], 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1e-3)
        total += v
        if _NCU_NAMES[name] in r["Kernel Name"]:
            mine.append(v)
    if not mine:
        return None
    return {"mean_us": round(sum(mine) / len(mine), 2), "launches": len(mine),
            "share_of_kernel_time": round(sum(mine) / total, 3), "source": path}


def land_traffic(segment: str):
    """DRAM bytes per launch of the probe's land from the committed ncu --set
    full capture (profiles/r2_land_traffic.json), if it is the same segment."""
    p = ROOT / "profiles" / "r2_land_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    if d.get("segment") != segment:
        return None
    return d["dram_bytes_read"] + d["dram_bytes_write"]


def pcie_probe(gpu: int = 0, chunk_mib: int = 4, n: int = 64) -> dict:
    """The PCIe ceiling for the e2e transfer mix, measured in the same run
    (plumbing probe, torch copies from/to pinned memory): n x chunk H2D on one
    stream alone, then concurrently with n x chunk D2H on another."""
    import torch
    c = chunk_mib << 20
    h_in = torch.empty(n * c, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n * c, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n * c, dtype=torch.uint8, device=f"cuda:{gpu}")
    d_out = torch.empty(n * c, dtype=torch.uint8, device=f"cuda:{gpu}")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(both: bool) -> tuple[float, float]:
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
            if both:
                for k in range(n):
                    h_out[k * c:(k + 1) * c].copy_(d_out[k * c:(k + 1) * c], non_blocking=True)
            e2.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3, e0.elapsed_time(e2) / 1e3

    run(False)
    run(True)
    t_alone = min(run(False)[0] for _ in range(3))     # best of 3: a ceiling
    both = [run(True) for _ in range(3)]
    t_h, t_d = min(b[0] for b in both), min(b[1] for b in both)
    out = {"h2d_alone_GBps": round(n * c / t_alone / 1e9, 1),
           "h2d_with_d2h_GBps": round(n * c / t_h / 1e9, 1), "d2h_with_h2d_GBps": round(n * c / t_d / 1e9, 1),
           "how": f"{n} x {chunk_mib} MiB pinned copies per direction, torch, same process"}
    del h_in, h_out, d_in, d_out
    return out


def e2e_floor_ms(h2d: int, d2h: int, p: dict) -> float:
    """Fastest a step moving h2d / d2h bytes can be on this PCIe link: the
    D2H runs at its duplex rate while H2D shares the link, the rest of the
    H2D at the one-direction rate."""
    hd, dd, ha = p["h2d_with_d2h_GBps"] * 1e9, p["d2h_with_h2d_GBps"] * 1e9, p["h2d_alone_GBps"] * 1e9
    t_overlap = min(d2h / dd, h2d / hd)
    h_rest = max(0.0, h2d - t_overlap * hd)
    d_rest = max(0.0, d2h - t_overlap * dd)
    return round((t_overlap + h_rest / ha + d_rest / dd) * 1e3, 3)


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_reduce_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def min_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_reduce_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t.item())


def sum_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_reduce_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def ro_checksums_agree(dist, data) -> bool:
    """Every rank verified the same landed bytes for every function."""
    import torch
    mine = [data[n].ro_checksum or 0 for n in sorted(data)]
    t = torch.tensor([c - (1 << 64) if c >= (1 << 63) else c for c in mine], dtype=torch.int64,
                     device=_reduce_device(dist))
    lo, hi = t.clone(), t.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    return bool(torch.equal(lo, hi))


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


def cfg1_compare(n: int = 16) -> dict:
    """BASELINE cfg 1: 16 concurrent cold starts of one 100 MiB function,
    SAGE (parallel setup + sharing) vs FixedGSL (fresh context, serial)."""
    from paper_2404_14691_b200.parboil import synthetic_function
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation, summarize_setup
    spec, data = synthetic_function("fn100", 100, 10, 1, tensors=64)
    out = {}
    # SAGE_pinned_store: the memory daemon keeps the function's DB record in
    # pinned host memory (registered once, as SAGE's daemon caches function
    # data on the host); the others read it pageable per cold start.
    # FixedGSL rows: a fresh CUDA context per instance, on a library thread of
    # this process ("thread") or in its own OS process ("process": what a
    # container per function pays), alone (N=1) and 16 at once.  DGSF: four
    # pre-created contexts (registration time), serial data loading.
    rows = (("SAGE", "SAGE", "thread", n, 6), ("SAGE_pinned_store", "SAGE", "thread", n, 6),
            ("DGSF", "DGSF", "thread", n, 3),
            ("FixedGSL_thread_n1", "FixedGSL", "thread", 1, 3), ("FixedGSL_thread", "FixedGSL", "thread", n, 1),
            ("FixedGSL_process_n1", "FixedGSL", "process", 1, 3), ("FixedGSL_process", "FixedGSL", "process", n, 1))
    for row, pol, mode, burst, reps in rows:
        sim = Simulation(ClusterSpec(gpus=1, instance_mode=mode), policy_preset(pol), {spec.name: spec}, seed=1,
                         function_data={spec.name: data})
        if row.endswith("pinned_store"):
            sim.dataplane.pin_host_store()
        try:
            samples = []
            for rep in range(reps):
                if sim.sharing is not None:
                    for r in list(sim.sharing.residents.values()):
                        sim.sharing.evict(r)
                invs = sim.submit_many([spec.name] * burst)
                sim.drain()
                if rep >= (1 if reps > 1 else 0):   # the first burst is a warm-up
                    samples += invs
            s = summarize_setup(samples)
            s["bursts"] = reps - (1 if reps > 1 else 0)
            s["concurrent"] = burst
            out[row] = {k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()}
        finally:
            sim.close()
    sage = out["SAGE"]["setup_p50_ms"]
    out["p50_setup_ratio_fixedgsl_over_sage"] = round(out["FixedGSL_thread"]["setup_p50_ms"] / sage, 1)
    out["p50_setup_ratio_fixedgsl_process_over_sage"] = round(out["FixedGSL_process"]["setup_p50_ms"] / sage, 1)
    out["p50_setup_ratio_dgsf_over_sage"] = round(out["DGSF"]["setup_p50_ms"] / sage, 1)
    out["workload"] = f"{n} concurrent cold starts, 100 MiB RO (64 ragged tensors), 10 MiB writable, 1 MiB input"
    return out


def cpu_baseline(burst: int = 64, bursts: int = 3) -> dict:
    """The host-only serving path on this box's cores (oracle/cpu_path.py):
    the same cfg-2 burst, every invocation loaded (copy + unpack + checksum)
    and computed (fp32 torch-CPU body) on its own core, all cores busy."""
    from oracle.cpu_path import CpuServer, host_info
    from paper_2404_14691_b200.parboil import cfg2_functions
    table, data = cfg2_functions()
    names = burst_names(table, burst)
    srv = CpuServer(data, workers=min(os.cpu_count() or 1, burst))
    try:
        srv.burst(names[:srv.workers])            # warm (threads, allocator, torch kernels)
        dts = [srv.burst(names) for _ in range(bursts)]
        lp = srv.load_path_rates()
    finally:
        srv.close()
    v = burst * len(dts) / sum(dts)
    return {"value": round(v, 2), "unit": UNIT, "cores": srv.workers, "kind": "port",
            "sample": f"{len(dts)} full bursts of {burst} cfg-2 invocations, {sum(dts):.2f} s: per invocation "
                      f"host copy + unpack + checksum (C) and the fp32 body (torch-CPU, 1 thread), "
                      f"{srv.workers} invocations at a time on {srv.workers} threads",
            "host": host_info(), "load_path": lp}


def our_arm(args, rank, world, dist) -> dict:
    from paper_2404_14691_b200 import _lib
    from paper_2404_14691_b200.parboil import cfg2_functions
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation, percentile

    table, data = cfg2_functions()
    names = burst_names(table, args.burst)
    cc = args.compute_concurrency or None
    sim = Simulation(ClusterSpec(gpus=1, compute_concurrency=cc, chunk_mb=args.chunk_mb,
                                 staging_mb=args.chunk_mb * 8), policy_preset("SAGE"), table, seed=1,
                     function_data=data, copy_results=False)
    box = None
    fanout_note = None
    if world > 1 and args.fanout != "none":
        # PCIe once per box: each function's home rank loads its segment over
        # PCIe; the other ranks land it from the home's pages peer to peer
        # (p2p, default) or receive it by ncclBroadcast (nccl)
        from paper_2404_14691_b200.fanout import BoxFanout, PeerFanout
        if args.fanout == "p2p":
            job = f"{os.environ.get('MASTER_PORT', '0')}-{os.getppid()}"
            box = PeerFanout(rank, world, table, job=job, barrier=dist.barrier)
            # check the exchange end to end on this box before relying on it;
            # any rank failing -> every rank loads over its own PCIe instead
            ok = box.selftest(0) and os.environ.get("SAGE_FANOUT_SELFTEST_FAIL", "-1") != str(rank)
            if min_over_ranks(dist, 1.0 if ok else 0.0) < 1.0:
                box.close()
                box = None
                fanout_note = "peer fan-out selftest failed on a rank: every rank loaded over its own PCIe"
        else:
            box = BoxFanout(rank, world, table)
        sim.dataplane.box = box
    L = _lib.lib()
    try:
        # the e2e legs are timed without per-kernel events (they cost ~3% of a
        # PCIe-bound burst: tools/e2e_timeline.py, SAGE_TIMELINE_STATS)
        _lib.check(L.sage_stats_enable(0), "stats_enable")
        # ---- e2e: host buffers through the public API -------------------------
        # request payloads arrive in pinned host buffers (as from a NIC); the
        # functions' DB records stay pageable: cold loads pay CPU_LOAD
        from paper_2404_14691_b200 import device as D
        payloads = []
        for n in names:
            pb = D.PinnedBuffer(data[n].input_bytes)
            pb.view()[:] = data[n].input
            payloads.append(pb)
        # (a) DB records pageable: every cold load pays the CPU_LOAD memcpy
        pg_us, invs_pg = timed(sim, names, args.steps, args.warmup, dist, payloads)
        # (b) the daemon's host store pinned at registration (outside the timed
        #     region): cold loads DMA straight from it -- the headline e2e
        sim.dataplane.pin_host_store()
        clocks = ClockSampler(_my_device()).start()
        e2e_us, invs_e2e = timed(sim, names, args.steps, args.warmup, dist, payloads)
        e2e_steps = timed.step_ms
        e2e_box_bytes = timed.box_bytes
        clocks_e2e = clocks.stop()
        # per-kernel breakdown of the e2e path: one more (untimed) step with
        # CUDA events around every launch; the value leg keeps them on (its
        # dominant kernel is the contract roofline)
        _lib.check(L.sage_stats_enable(1), "stats_enable")
        _lib.check(L.sage_stats_reset(), "stats_reset")
        run_steps(sim, names, 1, payloads)
        stats_e2e = kernel_stats()
        sim.dataplane.unpin_host_store()
        for pb in payloads:
            pb.free()
        per_step = len(names)
        pcie = pcie_probe(_my_device())
        h2d = sum(i.measured.get("pcie_bytes", 0) for i in invs_e2e) / args.steps
        h2d_rank = float(h2d)        # this rank's PCIe bytes per step (N > 1: homes carry the RO segments)
        d2h = sum(data[n].out_bytes for n in names)
        setups_e2e = [i.setup_us for i in invs_e2e]
        # ---- value: HBM-resident sources ----------------------------------------
        sim.dataplane.stage_sources_in_hbm(0)
        sim.dataplane.results_in_hbm = True
        clocks = ClockSampler(_my_device()).start()
        val_us, invs_val = timed(sim, names, args.steps, args.warmup, dist)
        val_steps = timed.step_ms
        clocks_val = clocks.stop()
        stats_val = kernel_stats()
        setups_val = [i.setup_us for i in invs_val]
        gpu_launches = sum(v["launches"] for v in stats_val.values())
        probe = land_probe(data)
        dom_body = max(stats_val, key=lambda k: stats_val[k]["total_us"])
        iso = body_probe(data, dom_body)
        gceil = gather_probe(data) if dom_body == "spmv" else None
        sim.dataplane.results_in_hbm = False
        sim.dataplane.drop_hbm_sources()
        sim.check_no_leaks()
        link = None
        if box is not None and box.kind == "peer":
            # the fan-out receive step measured alone: a peer-reading land of a
            # 256 MiB segment from every other rank's pages over NVLink
            per_peer = box.link_probe(_my_device() if not _shared_gpu() else 0)
            mine = [v for v in per_peer.values() if v]
            lo = min_over_ranks(dist, min(mine) if mine else 0.0)
            hi = max_over_ranks(dist, max(mine) if mine else 0.0)
            link = {"nvlink_GBps_min": round(lo, 1), "nvlink_GBps_max": round(hi, 1),
                    "frac_of_measured_peer_copy_770": round(lo / 770.0, 3), "frac_of_nominal_900": round(lo / 900.0, 3),
                    "how": "each rank lands every peer's 256 MiB segment with the peer-reading land (checksum "
                           "fused), median of 5 per peer, device events; min / max over ranks and peers",
                    "note": ("ranks share one device (SAGE_BENCH_SHARE_GPU): an HBM rate, not NVLink"
                             if _shared_gpu() else "")}
        pcie_rank = {"h2d_bytes_per_step_min": int(min_over_ranks(dist, h2d_rank)),
                     "h2d_bytes_per_step_max": int(max_over_ranks(dist, h2d_rank))}
    finally:
        _lib.check(L.sage_stats_enable(0), "stats_enable")
        if box is not None:
            box.close()
        sim.close()

    total_inv = per_step * args.steps * world
    value = total_inv / (val_us / 1e6)
    e2e = total_inv / (e2e_us / 1e6)
    peaks = load_peaks()
    rooflines = {}
    for name, s in stats_val.items():
        avg_us = s["total_us"] / s["launches"]
        per_launch = s["work"] / s["launches"]
        if name == "sgemm":
            # 3xTF32 (FP32-accurate): three tcgen05 kind::tf32 MMAs per product;
            # the dense TF32 rate is half the measured dense BF16 rate, so the
            # bound on ALGORITHMIC fp32 FLOP/s is a third of it
            x3 = peaks["bf16_tflops"] / 2 / 3
            ach = per_launch / (avg_us * 1e-6) / 1e12
            rooflines[name] = {"bound": "tensor (3xTF32)", "achieved": round(ach, 2), "peak": round(x3, 1),
                               "unit": "TFLOP/s", "frac": round(ach / x3, 4),
                               "peak_source": "MEASURED_PEAKS bf16_tflops / 2 (TF32 MMA rate) / 3 passes",
                               "avg_launch_us": round(avg_us, 2), "launches": s["launches"],
                               "share_of_kernel_time": None}
        elif name == "spmv":
            ach = per_launch / (avg_us * 1e-6) / 1e9
            rooflines[name] = {"bound": "l2 gather", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                               "frac": round(ach / peaks["hbm_gbs"], 4), "avg_launch_us": round(avg_us, 2),
                               "launches": s["launches"], "alg_bytes_per_launch": int(per_launch),
                               "note": "one random 32-B L2 sector per non-zero for x (4 MiB, L2-resident): "
                                       "L2 sector-rate bound, not HBM (DESIGN.md §3)"}
        else:
            ach = per_launch / (avg_us * 1e-6) / 1e9
            rooflines[name] = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                               "frac": round(ach / peaks["hbm_gbs"], 4), "avg_launch_us": round(avg_us, 2),
                               "launches": s["launches"], "alg_bytes_per_launch": int(per_launch)}
    tot = sum(s["total_us"] for s in stats_val.values()) or 1.0
    for name, s in stats_val.items():
        rooflines[name]["share_of_kernel_time"] = round(s["total_us"] / tot, 3)
    # the land kernel's roofline: back-to-back lands of the largest RO segment
    # on an otherwise idle GPU (in-burst launches overlap bodies, see rooflines)
    p_us = probe["total_us"] / probe["launches"]
    p_ach = probe["work"] / probe["launches"] / (p_us * 1e-6) / 1e9
    land = {"achieved": round(p_ach, 1), "frac": round(p_ach / peaks["hbm_gbs"], 4), "avg_launch_us": round(p_us, 2),
            "alg_bytes_per_launch": probe["work"] // probe["launches"], "launches": probe["launches"],
            "segment": probe["segment"]}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(val_us / 1e3 / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32 (bodies; sgemm as 3xTF32 on tcgen05, FP32-accurate) / u8 (land)", "data": "synthetic",
        "config": workload_config(per_step, world, args.compute_concurrency),
        "setup_p50_ms": round(percentile(setups_val, 50) / 1e3, 3),
        "setup_p99_ms": round(percentile(setups_val, 99) / 1e3, 3),
        "step_ms": val_steps,
        # diagnostic only (value above is the mean over all timed steps): the
        # same throughput at the median step, so a rare host stall on a box
        # (a 20-30 ms step among ~3.5 ms ones) is visible as such
        "value_at_median_step": round(per_step * world / (statistics.median(val_steps) / 1e3), 2) if val_steps else None,
        "e2e": {"value": round(e2e, 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": round(e2e_us / 1e3 / args.steps, 3),
                "setup_p50_ms": round(percentile(setups_e2e, 50) / 1e3, 3),
                "setup_p99_ms": round(percentile(setups_e2e, 99) / 1e3, 3),
                "h2d_GBps": round(h2d * args.steps / e2e_us / 1e3, 2),
                "pcie_both_directions_GBps": round((h2d + d2h) * args.steps / e2e_us / 1e3, 2),
                "roofline": {"bound": "pcie (duplex, this box)", "floor_ms_per_step": e2e_floor_ms(h2d, d2h, pcie),
                             "ms_per_step": round(e2e_us / 1e3 / args.steps, 3),
                             "frac": round(e2e_floor_ms(h2d, d2h, pcie) / (e2e_us / 1e3 / args.steps), 4),
                             "probe": pcie},
                "step_ms": e2e_steps,
                "inputs": "request payloads in pinned host buffers; DB records in the pinned host store",
                "pageable_db": {"value": round(total_inv / (pg_us / 1e6), 2), "unit": UNIT,
                                "ms_per_step": round(pg_us / 1e3 / args.steps, 3),
                                "setup_p50_ms": round(percentile([i.setup_us for i in invs_pg], 50) / 1e3, 3),
                                "setup_p99_ms": round(percentile([i.setup_us for i in invs_pg], 99) / 1e3, 3),
                                "note": "DB records pageable: cold loads include the CPU_LOAD memcpy"}},
        # the contract's roofline: the kernel with the largest share of device
        # time in the timed value leg, timed there with CUDA events on its own
        # stream; the data plane's own kernel (land) is reported beside it
        "roofline": dominant_roofline(rooflines, stats_val, peaks, iso, gceil,
                                      next((int(data[n].args[1]) for n in sorted(data) if data[n].body == "spmv"), 0)),
        "roofline_land": {"kernel": "land", "bound": "hbm", "achieved": land["achieved"], "peak": peaks["hbm_gbs"],
                          "unit": "GB/s", "frac": land["frac"], "traffic": land_traffic(probe["segment"]),
                          "traffic_source": "profiles/r2_land_traffic.json (ncu --set full, the same 1 GiB launch)",
                          "peak_source": peaks["source"], "same_size_d2d_GBps": probe["d2d_GBps"],
                          "frac_of_same_size_d2d": round(land["achieved"] / probe["d2d_GBps"], 4),
                          "avg_launch_us": land["avg_launch_us"], "alg_bytes_per_launch": land["alg_bytes_per_launch"],
                          "launches": land["launches"],
                          "how": f"{land['launches']} back-to-back HBM-resident lands of {land['segment']}, CUDA "
                                 f"events on the land stream (in-burst launches: rooflines.land)"},
        "rooflines": rooflines,
        "kernels_e2e": stats_e2e,
        "kernels_e2e_how": "one untimed e2e step with CUDA events around every launch (the timed e2e legs run "
                           "without them)",
        "gpu_launches": gpu_launches,
        "fanout": ({"fallback": fanout_note} if fanout_note else None) if box is None else {
            "how": ("home rank loads each RO segment over PCIe; the other ranks land it from the home's pages "
                    "peer to peer (one land + checksum, interprocess event)" if box.kind == "peer" else
                    "home rank loads each RO segment over PCIe; ncclBroadcast to the other ranks, then "
                    "land+checksum from HBM there") + " (e2e / pageable legs)",
            "homes": box.homes, "rank0": box.stats(),
            "nvlink_bytes_in_all_ranks": int(sum_over_ranks(dist, box.bytes_in)),
            "nvlink_GBps_e2e": round(sum_over_ranks(dist, e2e_box_bytes) / (e2e_us / 1e6) / 1e9, 2),
            "nvlink_GBps_note": "segment bytes received by all ranks in the timed e2e steps over the e2e time "
                                "(a traffic rate, not a link benchmark)",
            "ro_checksums_agree": ro_checksums_agree(dist, data),
            "link_probe": link, "pcie_per_rank": pcie_rank},
        "clocks": clocks_val,
        "clocks_e2e": clocks_e2e,
    }
    return line


def workload_config(burst: int, world: int, cc: int = 0) -> dict:
    """The `config` both arms report (the reference arm times a bounded
    sample of the same workload, described in its cpu_baseline.sample)."""
    c = {"workload": f"cfg2: burst of {burst} concurrent invocations (sgemm/stencil/spmv uniform "
                     f"mix, shared RO segments, cold start per burst) per GPU",
         "policy": "SAGE", "burst": burst, "gpus": world,
         "l2": "inputs larger than L2 (212 MiB RO + 504 MiB inputs per step)"}
    if cc:
        c["compute_concurrency"] = cc
    return c


def reference_arm(args, rank, world) -> dict:
    """--impl reference: the reference's CPU path on this box's host cores
    (the host-only serving path of oracle/cpu_path.py; the reference itself
    is a simulator with nothing to time), rank 0 only.  One step = one full
    cfg-2 burst of `--burst` invocations, the same workload our arm serves."""
    from oracle.cpu_path import CpuServer, host_info
    from paper_2404_14691_b200.parboil import cfg2_functions
    table, data = cfg2_functions()
    names = burst_names(table, args.burst)
    srv = CpuServer(data, workers=min(os.cpu_count() or 1, args.burst))
    try:
        for _ in range(args.warmup):
            srv.burst(names)
        dts = [srv.burst(names) for _ in range(args.steps)]
        lp = srv.load_path_rates()
    finally:
        srv.close()
    total = sum(dts)
    v = args.burst * args.steps / total
    return {"metric": METRIC, "value": round(v, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total * 1e3 / args.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32 (bodies) / u8 (load)", "data": "synthetic",
            "impl": "reference", "config": workload_config(args.burst, world),
            "cpu_baseline": {"value": round(v, 2), "unit": UNIT, "cores": srv.workers, "kind": "port",
                             "sample": f"{args.steps} full bursts of {args.burst} cfg-2 invocations after "
                                       f"{args.warmup} warm-up bursts: per invocation host copy + unpack + "
                                       f"checksum (C) and the fp32 body (torch-CPU, 1 thread), {srv.workers} "
                                       f"invocations at a time on {srv.workers} threads",
                             "host": host_info(), "load_path": lp},
            "e2e": {"value": round(v, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--burst", type=int, default=64)
    ap.add_argument("--no-cfg1", action="store_true")
    ap.add_argument("--chunk-mb", type=float, default=32.0,
                    help="staged-load chunk (one H2D + one land launch each; the ring holds 8)")
    ap.add_argument("--compute-concurrency", type=int, default=0,
                    help="ComputeGate slots per GPU (functions.py:304-327; 0 = no gate)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fanout", choices=["p2p", "nccl", "none"], default="p2p",
                    help="N>1: how non-home ranks get a segment (peer land of the home's pages / ncclBroadcast / "
                         "their own PCIe load)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local = _rank_env()
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(reference_arm(args, rank, world)), flush=True)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(_my_device())
        tdist.init_process_group("gloo" if _shared_gpu() else "nccl")
        dist = tdist
    from paper_2404_14691_b200 import _lib
    _lib.lib()  # fail loudly if the native library is missing
    line = our_arm(args, rank, world, dist)
    if rank == 0 and world == 1:
        if not args.no_cfg1:
            line["cfg1_sage_vs_fixedgsl"] = cfg1_compare()
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
