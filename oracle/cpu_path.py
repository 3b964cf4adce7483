"""The host-only serving path: the CPU reference arm of bench.py.

TEST / BASELINE INFRASTRUCTURE ONLY (like everything under oracle/): only
bench.py's cpu_baseline leg and `--impl reference` run it, as the timed CPU
reference; the product never imports it.

What it times (BASELINE.md "CPU-baseline plan" items 2-3; the reference
itself, pkg/src/gslsim, is a simulator with no data-moving code):
one burst of the same invocations our arm serves, each invocation handled
like a CPU serving process would handle it on one core -- no sharing, no
GPU:
  1. CPU_LOAD   copy the function's DB record into the invocation's private
                host buffer;
  2. unpack     land the record through the segment layout and compute the
                64-bit content checksum, fused window by window (one pass
                over the landed bytes; oracle_load_into in sage_oracle.c);
  3. COMPUTE    the function body in fp32 on that core: torch-CPU sgemm
                (BLAS), the 7-point stencil, CSR spmv (torch.sparse);
and the invocations of the burst run concurrently, one per host thread, on
every core of the box.  Buffers are allocated once per worker thread,
outside the timed region, and reused.
"""
from __future__ import annotations

import os
import platform
import warnings
import subprocess
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import oracle as O


def host_info() -> dict:
    """Core count and CPU model of this box (lscpu), for the bench line."""
    info = {"cores": os.cpu_count() or 1, "machine": platform.machine()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Thread(s) per core", "Core(s) per socket", "NUMA node(s)"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    return info


class CpuServer:
    """Runs bursts of invocations of registered functions on host threads."""

    def __init__(self, data: dict, workers: int | None = None):
        import torch
        torch.set_num_threads(1)          # one invocation per core: bodies stay on their thread
        self.torch = torch
        self.data = data
        self.workers = max(1, workers or (os.cpu_count() or 1))
        self._tls = threading.local()
        self.pool = ThreadPoolExecutor(max_workers=self.workers)
        self.max_packed = max(fd.layout.packed_bytes for fd in data.values())
        self.max_seg = max(fd.layout.seg_bytes for fd in data.values())
        # spmv CSR index tensors are part of the landed segment; the torch CSR
        # object is rebuilt per invocation from its own landed copy
        list(self.pool.map(lambda _: self._buffers(), range(self.workers)))   # allocate + fault in

    def close(self) -> None:
        self.pool.shutdown()

    def _buffers(self):
        b = getattr(self._tls, "b", None)
        if b is None:
            priv = np.zeros(self.max_packed, np.uint8)
            seg = np.zeros(self.max_seg, np.uint8)
            b = self._tls.b = (priv, seg)
        return b

    def invoke(self, name: str) -> int:
        """One invocation on the calling thread; returns the landed checksum."""
        fd = self.data[name]
        lay = fd.layout
        priv, seg = self._buffers()
        seg = seg[:lay.seg_bytes]
        cs = O.load_into_c(fd.db, lay.src_off, lay.dst_off, lay.length, priv[:lay.packed_bytes], seg)
        self._body(fd, seg, fd.input)
        return cs

    def _body(self, fd, seg: np.ndarray, x: np.ndarray):
        t = self.torch
        if fd.body == "sgemm":
            m, n, k = fd.args
            A = t.from_numpy(seg[:m * k * 4].view(np.float32).reshape(m, k))
            B = t.from_numpy(x.view(np.float32).reshape(n, k))
            return t.mm(A, B.T)
        if fd.body == "stencil":
            nx, ny, nz, bits = fd.args
            beta = float(np.int32(bits).view(np.float32))
            c = t.from_numpy(seg.view(np.float32)[:nx * ny * nz].reshape(nz, ny, nx))
            g = t.from_numpy(x.view(np.float32).reshape(nz, ny, nx))
            out = g.clone()
            s = (g[1:-1, 1:-1, :-2] + g[1:-1, 1:-1, 2:] + g[1:-1, :-2, 1:-1] + g[1:-1, 2:, 1:-1]
                 + g[:-2, 1:-1, 1:-1] + g[2:, 1:-1, 1:-1])
            out[1:-1, 1:-1, 1:-1] = c[1:-1, 1:-1, 1:-1] * g[1:-1, 1:-1, 1:-1] + beta * s
            return out
        if fd.body == "spmv":
            rows, nnz, o_rp, o_col, o_val = fd.args
            rp = t.from_numpy(seg[o_rp:o_rp + 4 * (rows + 1)].view(np.int32))
            col = t.from_numpy(seg[o_col:o_col + 4 * nnz].view(np.int32))
            val = t.from_numpy(seg[o_val:o_val + 4 * nnz].view(np.float32))
            xv = t.from_numpy(x.view(np.float32))
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")   # beta-API notices
                A = t.sparse_csr_tensor(rp, col, val, size=(rows, xv.numel()), check_invariants=False)
            return A @ xv
        raise ValueError(f"no CPU body for {fd.body!r}")

    def burst(self, names) -> float:
        """Serve one burst concurrently on all workers; wall seconds."""
        t0 = time.perf_counter()
        sums = list(self.pool.map(self.invoke, names))
        dt = time.perf_counter() - t0
        if any(s == 0 for s in sums):
            raise RuntimeError("a host load produced an empty checksum")
        return dt


    def load_path_rates(self) -> dict:
        """GB/s of the host load path (copy + unpack + checksum) on one core
        and on every worker at once, next to this box's memcpy rate measured
        the same way (read + write bytes).  Algorithmic traffic per load:
        2*packed (copy) + packed + seg (unpack; the fused checksum reads the
        window from cache)."""
        fd = max(self.data.values(), key=lambda f: f.layout.seg_bytes)
        lay = fd.layout

        def one(gate):
            priv, seg = self._buffers()
            priv, seg = priv[:lay.packed_bytes], seg[:lay.seg_bytes]
            O.load_into_c(fd.db, lay.src_off, lay.dst_off, lay.length, priv, seg)   # warm
            if gate is not None:
                gate.wait()
            t0 = time.perf_counter()
            O.load_into_c(fd.db, lay.src_off, lay.dst_off, lay.length, priv, seg)
            return t0, time.perf_counter()

        b, e = self.pool.submit(one, None).result()
        gate = threading.Barrier(self.workers)
        spans = list(self.pool.map(one, [gate] * self.workers))
        wall = max(e for _, e in spans) - min(b for b, _ in spans)
        return _rates(lay, e - b, wall, self.workers)


def _rates(lay, single: float, wall: float, threads: int) -> dict:
    traffic = 3 * lay.packed_bytes + lay.seg_bytes
    mc1 = O.memcpy_rate_c(64 << 20, 1)
    mcn = O.memcpy_rate_c(64 << 20, threads)
    per_core = traffic / single / 1e9
    return {"segment": f"{lay.seg_bytes} B landed from a {lay.packed_bytes} B record",
            "per_core_GBps": round(per_core, 2), "per_core_landed_GBps": round(lay.seg_bytes / single / 1e9, 2),
            "memcpy_1core_GBps": round(mc1, 2), "frac_of_memcpy_1core": round(per_core / mc1, 3),
            "all_cores_GBps": round(traffic * threads / wall / 1e9, 2), "memcpy_all_cores_GBps": round(mcn, 2),
            "threads": threads,
            "traffic_model": "3*packed + seg bytes per load (copy read+write, unpack read+write; checksum fused)"}
