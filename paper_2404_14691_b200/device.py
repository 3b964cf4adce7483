"""Thin Python wrappers over the C-ABI (include/sage_dp.h).

These are the calls the host layer (functions / sharing / policies /
runtime) makes; each wrapper raises on a negative status and turns the
pool's SAGE_ENOMEM into the reference's `Denied` value
(resources.py:244-257).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import H, check, handles, lib


# --------------------------------------------------------------- events -----
class Event:
    """An END (or BEGIN) event of an asynchronous op.  Owned: release() once."""

    __slots__ = ("h",)

    def __init__(self, h: int):
        self.h = h

    def done(self) -> bool:
        return check(lib().sage_event_query(self.h), "sage_event_query") == _lib.SAGE_OK

    def sync(self) -> None:
        check(lib().sage_event_sync(self.h), "sage_event_sync")

    def time_us(self) -> int:
        t = C.c_int64()
        rc = check(lib().sage_event_time(self.h, C.byref(t)), "sage_event_time")
        if rc == _lib.SAGE_ENOTREADY:
            raise RuntimeError("event not complete")
        return t.value

    def release(self) -> None:
        if self.h:
            check(lib().sage_event_release(self.h), "sage_event_release")
            self.h = 0


def poll(events: Sequence[Event], timeout_us: int = 0) -> list[bool]:
    n = len(events)
    if n == 0:
        return []
    arr = (H * n)(*[e.h for e in events])
    done = (C.c_uint8 * n)()
    check(lib().sage_event_poll(arr, n, done, timeout_us), "sage_event_poll")
    return [bool(d) for d in done]


_clock = [-1, 0]   # [library generation, epoch ns]


def now_us() -> int:
    """The library clock (sage_now_us) read in Python: CLOCK_MONOTONIC minus
    the epoch sage_init set (re-read once per init)."""
    c = _clock
    if c[0] != _lib._generation:
        c[0], c[1] = _lib._generation, int(lib().sage_clock_epoch_ns())
    return (time.monotonic_ns() - c[1]) // 1000


# ---------------------------------------------------------------- pool ------
@dataclass
class Segment:
    h: int
    gpu: int
    dptr: int
    nbytes: int
    cls: int

    def free(self) -> None:
        if self.h:
            check(lib().sage_pool_free(self.h), "sage_pool_free")
            self.h = 0


class DeniedAlloc(Exception):
    def __init__(self, shortfall: int):
        super().__init__(f"pool denied: shortfall {shortfall} bytes")
        self.shortfall = shortfall


def pool_alloc(gpu: int, nbytes: int, cls: int, account_only: bool = False, unaccounted: bool = False) -> Segment:
    h, d, sf = H(), C.c_uint64(), C.c_uint64()
    flags = (_lib.ALLOC_ACCOUNT_ONLY if account_only else 0) | (0x200 if unaccounted else 0)
    rc = lib().sage_pool_alloc(gpu, nbytes, cls | flags, C.byref(h), C.byref(d), C.byref(sf))
    if rc == _lib.SAGE_ENOMEM and sf.value:
        raise DeniedAlloc(sf.value)
    check(rc, "sage_pool_alloc")
    return Segment(h.value, gpu, d.value, nbytes, cls)


def pool_configure(gpu: int, capacity: int, granularity: int) -> None:
    check(lib().sage_pool_configure(gpu, capacity, granularity), "sage_pool_configure")


def pool_effective(gpu: int, nbytes: int) -> int:
    v = C.c_uint64()
    check(lib().sage_pool_effective(gpu, nbytes, C.byref(v)), "sage_pool_effective")
    return v.value


def pool_usage(gpu: int) -> dict:
    by = (C.c_uint64 * 4)()
    tot, phys, cap = C.c_uint64(), C.c_uint64(), C.c_uint64()
    check(lib().sage_pool_usage(gpu, by, C.byref(tot), C.byref(phys), C.byref(cap)), "sage_pool_usage")
    return {"by_class": list(by), "ledger": tot.value, "physical": phys.value, "capacity": cap.value}


def pool_trim(gpu: int) -> int:
    """Unmap the pool's cached free segments and idle chunks; bytes released."""
    r = C.c_uint64()
    check(lib().sage_pool_trim(gpu, C.byref(r)), "sage_pool_trim")
    return r.value


# ------------------------------------------------------------ host buffers --
class PinnedBuffer:
    """Pinned host memory owned by the library, viewable as numpy."""

    def __init__(self, nbytes: int):
        h, p = H(), C.c_void_p()
        check(lib().sage_host_alloc(max(1, nbytes), C.byref(h), C.byref(p)), "sage_host_alloc")
        self.h, self.ptr, self.nbytes = h.value, p.value, nbytes

    def view(self, dtype=np.uint8) -> np.ndarray:
        buf = (C.c_uint8 * self.nbytes).from_address(self.ptr)
        return np.frombuffer(buf, dtype=np.uint8).view(dtype)

    def free(self) -> None:
        if self.h:
            check(lib().sage_host_free(self.h), "sage_host_free")
            self.h = 0


# ---------------------------------------------------------------- loads -----
@dataclass
class LoadResult:
    cpu_begin_us: int
    cpu_end_us: int
    gpu_begin_us: int
    gpu_end_us: int
    host_bytes: int
    link_bytes: int
    landed_bytes: int
    checksum: int
    chunks: int


class LoadOp:
    __slots__ = ("h", "end", "keepalive")

    def __init__(self, h: int, end: Event, keepalive=None):
        self.h, self.end, self.keepalive = h, end, keepalive

    def info(self) -> Optional[LoadResult]:
        li = _lib.LoadInfo()
        rc = check(lib().sage_load_info_get(self.h, C.byref(li)), "sage_load_info_get")
        if rc == _lib.SAGE_ENOTREADY:
            return None
        return LoadResult(li.cpu_begin_us, li.cpu_end_us, li.gpu_begin_us, li.gpu_end_us, li.host_bytes,
                          li.link_bytes, li.landed_bytes, li.checksum, li.chunks)

    def wait(self) -> LoadResult:
        self.end.sync()
        return self.info()

    def release(self) -> None:
        if self.h:
            check(lib().sage_load_release(self.h), "sage_load_release")
            self.h = 0
        self.end.release()
        self.keepalive = None


def _ptr(src) -> tuple[int, int, object]:
    """(address, nbytes, keepalive) of a host buffer (numpy / PinnedBuffer)."""
    if isinstance(src, PinnedBuffer):
        return src.ptr, src.nbytes, src
    a = np.ascontiguousarray(src).view(np.uint8).reshape(-1)
    return a.ctypes.data, a.size, a


def load(gpu: int, dst: int, src, layout=None, *, pinned: bool = False, device_src: int = 0,
         device_src_bytes: int = 0, peer_gpu: int = -1, wait: Sequence[Event] = (), verify: bool = True) -> LoadOp:
    """Land `src` (packed stream) into `dst` through `layout` (None = identity).
    verify=False: no checksum (a private payload; an identity load from this
    GPU's HBM or pinned memory is then a plain DMA / D2D copy)."""
    d = _lib.LoadDesc()
    d.gpu = gpu
    d.dst = dst
    d.layout = layout.handle() if layout is not None else 0
    keep = None
    if device_src:
        d.flags = _lib.LOAD_SRC_PEER if peer_gpu >= 0 else _lib.LOAD_SRC_DEVICE
        d.src = device_src
        d.src_bytes = device_src_bytes
        d.src_gpu = peer_gpu
    else:
        addr, n, keep = _ptr(src)
        d.flags = _lib.LOAD_SRC_PINNED if (pinned or isinstance(src, PinnedBuffer)) else 0
        d.src = addr
        d.src_bytes = n
    if not verify:
        d.flags |= _lib.LOAD_NO_VERIFY
    arr, nw = handles([e.h for e in wait])
    d.wait = arr
    d.n_wait = nw
    lh, eh = H(), H()
    check(lib().sage_segment_load(C.byref(d), C.byref(lh), C.byref(eh)), "sage_segment_load")
    return LoadOp(lh.value, Event(eh.value), keep)


def host_load(gpu: int, dst: "PinnedBuffer", src, wait: Sequence[Event] = ()) -> tuple[Event, Event, object]:
    """CPU_LOAD alone: memcpy src into pinned dst on the GPU's host stream."""
    addr, n, keep = _ptr(src)
    arr, nw = handles([e.h for e in wait])
    b, e = H(), H()
    check(lib().sage_host_load(gpu, dst.ptr, addr, n, arr, nw, C.byref(b), C.byref(e)), "sage_host_load")
    return Event(b.value), Event(e.value), keep


def segment_checksum(gpu: int, dptr: int, nbytes: int) -> int:
    v = C.c_uint64()
    check(lib().sage_segment_checksum(gpu, dptr, nbytes, C.byref(v)), "sage_segment_checksum")
    return v.value


def d2h(gpu: int, dptr: int, host: PinnedBuffer, nbytes: int, wait: Sequence[Event] = ()) -> Event:
    arr, nw = handles([e.h for e in wait])
    eh = H()
    check(lib().sage_d2h_cache(gpu, dptr, host.ptr, nbytes, arr, nw, C.byref(eh)), "sage_d2h_cache")
    return Event(eh.value)


def read_device(gpu: int, dptr: int, nbytes: int) -> np.ndarray:
    """Synchronous D2H copy (tests / verification)."""
    buf = PinnedBuffer(max(16, nbytes))
    try:
        ev = d2h(gpu, dptr, buf, nbytes)
        ev.sync()
        ev.release()
        return buf.view()[:nbytes].copy()
    finally:
        buf.free()


def fanout(src_gpu: int, src: int, dst_gpu: int, dst: int, nbytes: int, wait: Sequence[Event] = ()) -> Event:
    arr, nw = handles([e.h for e in wait])
    eh = H()
    check(lib().sage_fanout(src_gpu, src, dst_gpu, dst, nbytes, arr, nw, C.byref(eh)), "sage_fanout")
    return Event(eh.value)


# ---------------------------------------------------------------- slots -----
class Slot:
    """A pooled stream of the pre-created context (the GPU_CTX replacement)."""

    __slots__ = ("h", "gpu")

    def __init__(self, gpu: int):
        h = H()
        check(lib().sage_ctx_acquire(gpu, C.byref(h)), "sage_ctx_acquire")
        self.h, self.gpu = h.value, gpu

    def bind_ctx(self, ctx_dptr: int, ctx_bytes: int, wait: Sequence[Event] = ()) -> tuple[Event, Event]:
        arr, nw = handles([e.h for e in wait])
        b, e = H(), H()
        check(lib().sage_ctx_bind(self.h, ctx_dptr, ctx_bytes, arr, nw, C.byref(b), C.byref(e)), "sage_ctx_bind")
        return Event(b.value), Event(e.value)

    def wait(self, events: Sequence[Event]) -> None:
        arr, nw = handles([e.h for e in events])
        if nw:
            check(lib().sage_stream_wait(self.h, arr, nw), "sage_stream_wait")

    def record(self) -> Event:
        e = H()
        check(lib().sage_slot_record(self.h, C.byref(e)), "sage_slot_record")
        return Event(e.value)

    def launch(self, body: "_lib.BodyDesc") -> tuple[Event, Event]:
        b, e = H(), H()
        check(lib().sage_launch(self.h, C.byref(body), C.byref(b), C.byref(e)), "sage_launch")
        return Event(b.value), Event(e.value)

    def stream(self) -> int:
        s = C.c_uint64()
        check(lib().sage_slot_stream(self.h, C.byref(s)), "sage_slot_stream")
        return s.value

    def sync_wait(self, events: Sequence[Event]) -> tuple[Event, Event]:
        arr, nw = handles([e.h for e in events])
        b, e = H(), H()
        check(lib().sage_sync_wait(self.h, arr, nw, C.byref(b), C.byref(e)), "sage_sync_wait")
        return Event(b.value), Event(e.value)

    def launch_after(self, wait: Sequence[Event], body: "_lib.BodyDesc") -> tuple[Event, Event]:
        arr, nw = handles([e.h for e in wait])
        b, e = H(), H()
        check(lib().sage_launch_after(self.h, arr, nw, C.byref(body), C.byref(b), C.byref(e)), "sage_launch_after")
        return Event(b.value), Event(e.value)

    def ret_after(self, wait: Sequence[Event], src: int, dst_ptr: int, nbytes: int) -> tuple[Event, Event]:
        arr, nw = handles([e.h for e in wait])
        b, e = H(), H()
        check(lib().sage_return_after(self.h, arr, nw, src, dst_ptr, nbytes, C.byref(b), C.byref(e)),
              "sage_return_after")
        return Event(b.value), Event(e.value)

    def ret(self, src: int, host_ptr: int, nbytes: int) -> tuple[Event, Event]:
        b, e = H(), H()
        check(lib().sage_return(self.h, src, host_ptr, nbytes, C.byref(b), C.byref(e)), "sage_return")
        return Event(b.value), Event(e.value)

    def release(self) -> None:
        if self.h:
            check(lib().sage_ctx_release(self.h), "sage_ctx_release")
            self.h = 0


def body_desc(kind: int, ro: int = 0, ro_bytes: int = 0, inp: int = 0, inp_bytes: int = 0, out: int = 0,
              out_bytes: int = 0, args: Sequence[int] = ()) -> "_lib.BodyDesc":
    b = _lib.BodyDesc()
    b.body = kind
    b.ro, b.ro_bytes, b.input, b.input_bytes, b.out, b.out_bytes = ro, ro_bytes, inp, inp_bytes, out, out_bytes
    for i, a in enumerate(args):
        b.args[i] = int(a)
    return b


# ------------------------------------------------------------- FixedGSL -----
class FixedGSLJob:
    __slots__ = ("h", "end", "keepalive")

    def __init__(self, h, end, keep):
        self.h, self.end, self.keepalive = h, end, keep

    def info(self) -> Optional["_lib.FixedGSLInfo"]:
        out = _lib.FixedGSLInfo()
        rc = check(lib().sage_fixedgsl_info_get(self.h, C.byref(out)), "sage_fixedgsl_info_get")
        return None if rc == _lib.SAGE_ENOTREADY else out

    def release(self) -> None:
        self.end.release()
        if self.h:
            check(lib().sage_fixedgsl_release(self.h), "sage_fixedgsl_release")
            self.h = 0
        self.keepalive = None


def fixedgsl_submit(gpu: int, layout, ro_src, inp, alloc_bytes: int, body: "_lib.BodyDesc",
                    result: Optional[PinnedBuffer], result_bytes: int, mode: int = 0, ctx: int = 0) -> FixedGSLJob:
    """One instance-per-invocation job: mode INSTANCE_THREAD (fresh context
    on a library thread), INSTANCE_PROCESS (fresh OS process) or
    INSTANCE_POOLED (DGSF: in the pre-created context `ctx`)."""
    d = _lib.FixedGSLDesc()
    d.gpu = gpu
    d.mode = mode
    d.ctx = ctx
    d.layout = layout.handle() if layout is not None else 0
    keep = []
    if ro_src is not None:
        a, n, k = _ptr(ro_src)
        d.ro_src, d.ro_src_bytes = a, n
        keep.append(k)
    if inp is not None:
        a, n, k = _ptr(inp)
        d.input, d.input_bytes = a, n
        keep.append(k)
    d.alloc_bytes = alloc_bytes
    d.body = body
    if result is not None:
        d.result, d.result_bytes = result.ptr, result_bytes
    jh, eh = H(), H()
    check(lib().sage_fixedgsl_submit(C.byref(d), C.byref(jh), C.byref(eh)), "sage_fixedgsl_submit")
    return FixedGSLJob(jh.value, Event(eh.value), keep)


def instance_ctx_create(gpu: int, body: int) -> int:
    """A real pre-created CUDA context with `body`'s kernels loaded (DGSF)."""
    h = H()
    check(lib().sage_instance_ctx_create(gpu, body, C.byref(h)), "sage_instance_ctx_create")
    return h.value


def instance_ctx_destroy(h: int) -> None:
    check(lib().sage_instance_ctx_destroy(h), "sage_instance_ctx_destroy")


def fanout_caps() -> dict:
    """The box's one-to-many options (sage_fanout_caps): peer reachability
    per plane and whether an NVSwitch multicast object can be made."""
    c = _lib.FanoutCaps()
    check(lib().sage_fanout_caps(C.byref(c)), "sage_fanout_caps")
    return {"n_gpus": c.n_gpus, "n_devices": c.n_devices, "peer_mask": [c.peer_mask[g] for g in range(c.n_gpus)],
            "multicast_attr": bool(c.multicast_attr), "multicast": bool(c.multicast),
            "multicast_granularity": c.multicast_granularity, "why": c.why.decode(errors="replace")}


def fanout_broadcast(src_gpu: int, src_dptr: int, nbytes: int, dsts, p2p_only: bool = False,
                     wait: Sequence[Event] = ()) -> tuple[str, Event]:
    """Copy nbytes at src_dptr (on src_gpu) into every (gpu, Segment) of
    `dsts`: one NVLS multicast pass when the box allows it, else peer copies.
    Returns ("multicast" | "p2p", end event)."""
    d = _lib.BcastDesc()
    d.src_gpu, d.n_dst, d.src_dptr, d.bytes = src_gpu, len(dsts), src_dptr, nbytes
    for i, (g, seg) in enumerate(dsts):
        d.dst_gpu[i], d.dst_alloc[i] = g, seg.h
    d.flags = _lib.BCAST_P2P_ONLY if p2p_only else 0
    arr, n = _lib.handles([e.h for e in wait])
    ev = H()
    check(lib().sage_fanout_broadcast(C.byref(d), arr, n, C.byref(ev)), "sage_fanout_broadcast")
    return ("multicast" if d.path == _lib.BCAST_PATH_MULTICAST else "p2p"), Event(ev.value)
