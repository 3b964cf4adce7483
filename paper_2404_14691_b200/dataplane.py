"""The real plane: compile a stage plan into device operations.

Reference: PlanExecution (pkg/src/gslsim/functions.py:341-433) walks the
stage DAG on the event loop, charging loads to fluid channels and fixed
stages to timers.  Here `DataPlane.start` walks the same DAG ONCE, at
admission, and enqueues every node as asynchronous device work whose
dependencies are its predecessors' END events:

  CONTAINER, CPU_CTX  host-side instance state, done synchronously
  CPU_LOAD            DB record -> pinned staging (memcpy fan-out, host stream);
                      in Parallel plans it is pipelined chunk by chunk into
                      GPU_LOAD by one native load (sage_segment_load)
  GPU_CTX             bind the function context segment on a pooled stream
                      (the pre-created context: no cuCtxCreate on this path)
  GPU_LOAD            chunked H2D on the copy engine + `land` (unpack +
                      checksum) of the read-only segment (from the DB, the
                      pinned Stage-2 cache, or a peer GPU over NVLink) and of
                      the invocation input
  SYNC_WAIT           device-side wait on the leader's END events (Token)
  COMPUTE             the body kernel on the invocation's stream
  RETURN              D2H of the result into pinned memory

The host is touched again only when the RETURN END event completes (polled
by the engine), when stage times are read back and the policy releases.
FixedGSL instances (fresh_context) run as native serial jobs instead.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from . import device as D
from .functions import FunctionSpec, PlanMode, Stage, StagePlan, WarmthClass
from .layout import SegmentLayout
from .resources import AllocClass, SimulationError

_BODY = {"touch": _lib.BODY_TOUCH, "sgemm": _lib.BODY_SGEMM, "stencil": _lib.BODY_STENCIL,
         "spmv": _lib.BODY_SPMV, "spin": _lib.BODY_SPIN, "sgemm_f32": 5,
         "spmv_csb": _lib.BODY_SPMV_CSB, "resnet50_native": _lib.BODY_RESNET50}


def _a256(n: int) -> int:
    return (n + 255) // 256 * 256


def synthetic_bytes(seed: int, nbytes: int) -> np.ndarray:
    """Deterministic synthetic DB bytes (PCG64 raw draws, little endian)."""
    words = np.random.PCG64(seed).random_raw((nbytes + 7) // 8).astype(np.uint64)
    return words.view(np.uint8)[:nbytes].copy()


def _name_seed(name: str) -> int:
    h = 1469598103934665603
    for ch in name.encode():
        h = ((h ^ ch) * 1099511628211) & 0xFFFFFFFFFFFF
    return h


@dataclass
class FunctionData:
    """What a registered function loads and runs on the real plane.

    layout / db      the read-only segment: packed DB record + landing layout
                     (layout.seg_bytes must fit the spec's ro allocation)
    body / args      COMPUTE kernel (csrc/bodies.cu) and its shape arguments
    input            default per-invocation payload (pageable host bytes)
    out_bytes        bytes RETURN copies back
    """
    layout: SegmentLayout
    db: np.ndarray
    body: str = "touch"
    args: tuple = ()
    input: Optional[np.ndarray] = None
    out_bytes: int = 16
    ro_checksum: Optional[int] = None     # learnt from the first landed copy
    # HBM-resident sources (bench `value` leg: inputs already in HBM, no PCIe)
    db_dev: Optional[D.Segment] = None
    input_dev: Optional[D.Segment] = None
    # the DB record is pinned (registered host store): cold loads DMA from it
    db_pinned: bool = False
    # per-invocation device workspace after the output (the native ResNet
    # program's activations), inside the invocation's writable segment
    scratch_bytes: int = 0

    @property
    def input_bytes(self) -> int:
        return 0 if self.input is None else int(self.input.nbytes)


def synthetic_data(spec: FunctionSpec, tensors: int = 16) -> FunctionData:
    """Default data of a spec without registered data: a ragged multi-tensor
    RO record exactly filling spec.ro_bytes when landed, a synthetic input of
    spec.input_bytes, and the TOUCH body (reads RO + input, returns digests)."""
    seed = _name_seed(spec.name)
    ro = spec.ro_bytes // 16 * 16
    if ro >= 16 * 256 * tensors:
        rng = np.random.Generator(np.random.PCG64(seed))
        w = rng.uniform(0.5, 1.5, tensors)
        sizes = [int(x) // 256 * 256 for x in w / w.sum() * ro]
        sizes[-1] += ro - sum(sizes)
        # carve ragged (non-16-aligned) tensor lengths inside 256-B extents
        lens = [max(1, s - int(rng.integers(0, 200))) for s in sizes]
        src, dst, d, s0 = [], [], 0, 0
        for s, n in zip(sizes, lens):
            src.append(s0)
            dst.append(d)
            s0 += n
            d += s
        layout = SegmentLayout(tuple(src), tuple(dst), tuple(lens), s0, ro)
    elif ro > 0:
        layout = SegmentLayout.identity(ro)
    else:
        layout = SegmentLayout((), (), (), 0, 0)
    db = synthetic_bytes(seed, layout.packed_bytes)
    inp = synthetic_bytes(seed + 1, spec.input_bytes) if spec.input_bytes else None
    if spec.body == "spin":
        return FunctionData(layout, db, "spin", (int(round(spec.compute_ms * 1000)),), inp, 16)
    return FunctionData(layout, db, "touch", (), inp, 16)


class _SlabBuffer(D.PinnedBuffer):
    """A size-class slot carved from a pinned slab (no handle of its own)."""

    def __init__(self, ptr: int, cap: int):   # noqa: super().__init__ would allocate
        self.h, self.ptr, self.nbytes, self.cap = 0, ptr, cap, cap

    def free(self) -> None:
        pass


class _PinnedPool:
    """Reuse pinned host buffers.  cudaHostAlloc costs ~0.4 ms however small
    the buffer (ms per 100 MiB), so buffers up to SMALL bytes come from 64 MiB
    slabs in power-of-two size classes: the first burst of N concurrent
    invocations pays one host allocation per slab, not one per return buffer
    (cfg 5 at N = 512: the first burst's submit took ~1 s); larger ones are
    cached by exact size."""

    SMALL = 16 << 20
    SLAB = 64 << 20

    def __init__(self):
        import os
        if os.environ.get("SAGE_PINNED_SLABS") == "0":    # diagnostics: every buffer its own cudaHostAlloc
            self.SMALL = 0
        self.free: dict[int, list] = {}
        self.small: dict[int, list] = {}
        self.slabs: list = []

    @staticmethod
    def _cls(nbytes: int) -> int:
        return max(4096, 1 << (max(1, nbytes) - 1).bit_length())

    def get(self, nbytes: int) -> D.PinnedBuffer:
        if nbytes <= self.SMALL:
            c = self._cls(nbytes)
            lst = self.small.get(c)
            if not lst:
                slab = D.PinnedBuffer(self.SLAB)
                self.slabs.append(slab)
                lst = self.small.setdefault(c, [])
                lst.extend(_SlabBuffer(slab.ptr + k * c, c) for k in range(self.SLAB // c))
            buf = lst.pop()
            buf.nbytes = nbytes
            return buf
        lst = self.free.get(nbytes)
        if lst:
            return lst.pop()
        return D.PinnedBuffer(nbytes)

    def put(self, buf: D.PinnedBuffer) -> None:
        if isinstance(buf, _SlabBuffer):
            self.small.setdefault(buf.cap, []).append(buf)
        else:
            self.free.setdefault(buf.nbytes, []).append(buf)

    def close(self) -> None:
        for lst in self.free.values():
            for b in lst:
                b.free()
        self.free.clear()
        self.small.clear()
        for slab in self.slabs:
            slab.free()
        self.slabs.clear()


class _PlanFacts:
    """What the one-call path needs to know about a plan, computed once per
    plan object (plans are cached, functions.py:_plan_cached)."""

    __slots__ = ("fast", "cpu_ctx", "gpu_ctx", "gpu_load_ro", "host_ro", "sync", "timed")

    def __init__(self, plan: StagePlan):
        stages = {n.stage for n in plan.nodes}
        self.fast = Stage.CONTAINER not in stages and not (plan.mode is PlanMode.SERIAL and Stage.GPU_CTX in stages)
        self.cpu_ctx = Stage.CPU_CTX in stages
        self.gpu_ctx = Stage.GPU_CTX in stages
        g = plan.node_index(Stage.GPU_LOAD)
        self.gpu_load_ro = g is not None and plan.nodes[g].ro
        c = plan.node_index(Stage.CPU_LOAD)
        self.host_ro = c is not None and plan.nodes[c].ro
        self.sync = bool(plan.wait_ro or plan.wait_ctx)
        # stages whose device times sage_invoke reports: (index in _STAGES, stage)
        self.timed = tuple((k, st) for k, st in enumerate(_STAGES)
                           if st is not Stage.CPU_CTX and st in stages)


def _plan_facts(plan: StagePlan) -> _PlanFacts:
    pf = plan.__dict__.get("_facts")
    if pf is None:
        pf = plan.__dict__["_facts"] = _PlanFacts(plan)
    return pf


def _desc_template(fd: "FunctionData", gpu: int) -> "_lib.InvokeDesc":
    """A sage_invoke descriptor with this function's constant fields (GPU,
    body template) filled in, built once per (function, GPU); each
    invocation starts from a copy."""
    memo = fd.__dict__.setdefault("_desc_tmpl", {})
    d = memo.get(gpu)
    if d is None:
        d = memo[gpu] = _lib.InvokeDesc()
        d.gpu = gpu
        d.body = _body_template(fd)
    return d


def _body_template(fd: "FunctionData") -> "_lib.BodyDesc":
    """The function's COMPUTE descriptor without pointers, built once."""
    b = fd.__dict__.get("_body_tmpl")
    if b is None:
        if fd.body == "resnet50_native":
            from . import dnn
            dnn.native_handle(fd)       # args[0] = the registered program
        b = D.body_desc(_BODY[fd.body], ro_bytes=fd.layout.seg_bytes, inp_bytes=(fd.input_bytes + 15) // 16 * 16,
                        out_bytes=max(16, fd.out_bytes), args=fd.args)
        fd.__dict__["_body_tmpl"] = b
    return b


class _Run:
    """One invocation's device-side state."""

    __slots__ = ("inv", "plan", "gpu", "slot", "events", "loads", "marks", "hooks", "pinned", "scratch", "result",
                 "out_bytes", "job", "end", "fd", "ro_source", "t_enqueue", "invh", "keep")

    def __init__(self, inv, plan: StagePlan, gpu: int, hooks: dict, fd: Optional["FunctionData"] = None):
        self.inv, self.plan, self.gpu, self.hooks, self.fd = inv, plan, gpu, hooks, fd
        self.slot: Optional[D.Slot] = None
        self.events: list = []        # every Event to release
        self.loads: list = []         # (node idx, kind, LoadOp)
        self.marks: dict = {}         # stage -> (begin src, end src)
        self.pinned: list = []        # pinned buffers to return
        self.scratch: list = []       # unaccounted device segments
        self.result: Optional[D.PinnedBuffer] = None
        self.out_bytes = 0
        self.job: Optional[D.FixedGSLJob] = None
        self.end: Optional[D.Event] = None
        self.ro_source = ""
        self.t_enqueue = 0
        self.invh = 0                 # native invocation (sage_invoke fast path)
        self.keep = None              # host payload kept alive until completion


_STAGES = [Stage.CONTAINER, Stage.CPU_CTX, Stage.CPU_LOAD, Stage.GPU_CTX, Stage.GPU_LOAD, Stage.SYNC_WAIT,
           Stage.COMPUTE, Stage.RETURN]


def _add_reader(resident, ev_h: int) -> None:
    """A land on another GPU reads `resident`'s RO segment over NVLink: keep
    an alias of its END event so freeing the segment waits for it (finished
    readers are dropped as new ones arrive)."""
    if not ev_h:
        return
    alias = _lib.H(0)
    _lib.check(_lib.lib().sage_event_alias(ev_h, _lib.C.byref(alias)), "sage_event_alias")
    live = []
    for e in resident.readers:
        if _lib.lib().sage_event_query(e.h) == _lib.SAGE_OK:
            e.release()
        else:
            live.append(e)
    live.append(D.Event(alias.value))
    resident.readers = live


class _Borrowed(D.Event):
    """An event owned by a native invocation: released with it, never alone."""

    __slots__ = ()

    def release(self) -> None:
        self.h = 0


class _FastCompletions:
    """Engine completion source for sage_invoke runs: the library's
    completion thread queues finished invocations (already resolved), so the
    loop neither polls per-invocation events nor computes stage times."""

    def __init__(self, dp: "DataPlane", batch: int = 256):
        self.dp = dp
        self.runs: dict[int, _Run] = {}
        self._buf = (_lib.H * batch)()
        self._n = batch

    def outstanding(self) -> int:
        return len(self.runs)

    def poll(self, timeout_us: int) -> int:
        n = _lib.lib().sage_invoke_ready(self._buf, self._n, int(timeout_us))
        if n < 0:
            _lib.check(n, "sage_invoke_ready")
        if n == 0:
            return 0
        eng = self.dp.sim.engine
        eng.tick()
        fired = 0
        for k in range(n):
            run = self.runs.pop(self._buf[k], None)
            if run is not None:
                self.dp._on_done(run)
                fired += 1
        return fired


class DataPlane:
    """Device side of one Simulation (runtime.py)."""

    def __init__(self, sim):
        self.sim = sim
        self.pinned = _PinnedPool()
        self.data: dict[str, FunctionData] = {}
        self.results_in_hbm = False   # bench `value` leg: RETURN copies D2D
        self._contexts: set = set()     # DGSF pre-created CUDA contexts
        # checksum private request payloads too (shared RO segments always are);
        # off by default: a second HBM read of every input (SAGE_VERIFY_INPUTS=1)
        import os
        self.verify_inputs = os.environ.get("SAGE_VERIFY_INPUTS") == "1"
        self._free_slots: dict[int, list] = {}
        self._fast = _FastCompletions(self)
        self._scratch: dict[tuple[int, int], list] = {}
        self.box = None               # fanout.BoxFanout: PCIe once per box across processes
        self._gate_q: dict[int, deque] = {}
        self._fast_source = False
        # sage_invoke's four output handles, reused call after call (read at once)
        self._inv_out = (_lib.H(), _lib.H(), _lib.H(), _lib.H())
        self._inv_out_refs = tuple(_lib.C.byref(x) for x in self._inv_out)

    # ------------------------------------------------------- compute gate ----
    def _gate_wait(self, run: _Run) -> Optional[int]:
        """ComputeGate (functions.py:304-327, ClusterSpec.compute_concurrency):
        at most K invocations of a GPU compute at once, FIFO.  On the device
        that is a semaphore over the enqueue order: the n-th invocation's
        COMPUTE waits for the (n-K)-th to finish (its RETURN END event: the
        gate is released one stage later than in the model)."""
        gates = self.sim.compute_gates
        if not gates:
            return None
        q = self._gate_q.setdefault(run.gpu, deque())
        while q and (q[0].inv is None or q[0].inv.run is not q[0]):
            q.popleft()                              # completed and released
        if len(q) < gates[run.gpu].slots:
            return None
        pred = q[0]
        return pred.end.h if pred.end is not None and pred.end.h else None

    def _gate_push(self, run: _Run) -> None:
        gates = self.sim.compute_gates
        if not gates:
            return
        q = self._gate_q.setdefault(run.gpu, deque())
        q.append(run)
        while len(q) > gates[run.gpu].slots:
            q.popleft()

    def _scratch_get(self, gpu: int, nbytes: int) -> D.Segment:
        """Runtime scratch outside the ledger (results kept in HBM, inputs that
        do not fit the writable allocation), reused by size."""
        lst = self._scratch.get((gpu, nbytes))
        if lst:
            return lst.pop()
        return D.pool_alloc(gpu, nbytes, _lib.CLASS_WRITABLE, unaccounted=True)

    def _slot(self, gpu: int) -> D.Slot:
        """A pooled stream of the pre-created context, kept acquired across invocations."""
        lst = self._free_slots.get(gpu)
        return lst.pop() if lst else D.Slot(gpu)

    # ---------------------------------------------------------------- data ----
    def register(self, name: str, data: FunctionData) -> None:
        spec = self.sim.spec_table[name]
        if data.layout.seg_bytes > max(spec.ro_bytes, 0) and data.layout.seg_bytes:
            raise ValueError(f"function {name}: landed segment ({data.layout.seg_bytes} B) exceeds "
                             f"ro_mem_mb ({spec.ro_bytes} B)")
        if data.layout.packed_bytes != data.db.nbytes:
            raise ValueError(f"function {name}: DB record size differs from its layout")
        self.data[name] = data

    def content_key(self, spec: FunctionSpec) -> Optional[int]:
        """The checksum the function's RO record has once landed (computed
        once on the host by the library: sage_layout_checksum)."""
        fd = self.data_for(spec)
        key = fd.__dict__.get("_content_key")
        if key is None and fd.layout.seg_bytes:
            out = _lib.u64(0)
            _lib.check(_lib.lib().sage_layout_checksum(fd.layout.handle(), fd.db.ctypes.data, fd.layout.packed_bytes,
                                                       _lib.C.byref(out)), "sage_layout_checksum")
            key = fd.__dict__["_content_key"] = out.value
        return key

    def stage_sources_in_hbm(self, gpu: int = 0) -> None:
        """Copy every registered function's DB record and default input into
        HBM (runtime scratch, outside the ledger): loads then land from HBM
        with no PCIe leg -- the device-resident `value` measurement."""
        for name, fd in self.data.items():
            for attr, host in (("db_dev", fd.db), ("input_dev", fd.input)):
                if host is None or host.nbytes == 0 or getattr(fd, attr) is not None:
                    continue
                seg = D.pool_alloc(gpu, host.nbytes + 64, _lib.CLASS_WRITABLE, unaccounted=True)
                op = D.load(gpu, seg.dptr, host, None)
                op.wait()
                op.release()
                setattr(fd, attr, seg)

    def pin_host_store(self, names=None) -> None:
        """Register DB records as pinned host memory (the daemon's host
        store): cold loads then DMA straight from them, no CPU_LOAD memcpy."""
        for name in (names if names is not None else list(self.data)):
            fd = self.data[name]
            if fd.db_pinned or fd.db.nbytes == 0:
                continue
            _lib.check(_lib.lib().sage_host_register(fd.db.ctypes.data, fd.db.nbytes), "sage_host_register")
            fd.db_pinned = True

    def unpin_host_store(self) -> None:
        for fd in self.data.values():
            if fd.db_pinned:
                _lib.check(_lib.lib().sage_host_unregister(fd.db.ctypes.data), "sage_host_unregister")
                fd.db_pinned = False

    def drop_hbm_sources(self) -> None:
        for fd in self.data.values():
            for attr in ("db_dev", "input_dev"):
                seg = getattr(fd, attr)
                if seg is not None:
                    seg.free()
                    setattr(fd, attr, None)

    def data_for(self, spec: FunctionSpec) -> FunctionData:
        fd = self.data.get(spec.name)
        if fd is None:
            fd = synthetic_data(spec)
            self.data[spec.name] = fd
        return fd

    # -------------------------------------------------------- stage-2 cache ----
    def cache_segment(self, r) -> Optional[D.Event]:
        """Stage1 -> Stage2: D2H the landed segment into a pinned host cache."""
        fd = self.data_for(r.spec)
        n = fd.layout.seg_bytes
        if n == 0 or r.gpu_ro is None:
            return None
        buf = self.pinned.get(n)
        ev = D.d2h(r.gpu, r.gpu_ro.dptr, buf, n)
        r.cpu_ro_cache.segment = buf
        r.cache_event = ev
        r.cache_bytes = n
        return ev

    def drop_cache(self, r) -> None:
        buf = r.cpu_ro_cache.segment if r.cpu_ro_cache is not None else None
        if r.cache_event is not None:
            r.cache_event.sync()
            r.cache_event.release()
            r.cache_event = None
        if isinstance(buf, D.PinnedBuffer):
            self.pinned.put(buf)
            r.cpu_ro_cache.segment = None

    def precreate_context(self, gpu: int, alloc, spec: Optional[FunctionSpec] = None) -> int:
        """DGSF registration: a real CUDA context (cuCtxCreate) with the
        function's body kernels loaded; its invocations run in it."""
        body = self.data_for(spec).body if spec is not None else "touch"
        h = D.instance_ctx_create(gpu, _BODY.get(body, _lib.BODY_TOUCH))
        self._contexts.add(h)
        return h

    def release_context(self, h: int) -> None:
        if h in self._contexts:
            self._contexts.discard(h)
            D.instance_ctx_destroy(h)

    # -------------------------------------------------------------- start -----
    def start(self, inv, plan: StagePlan, wait_tokens=(), hooks=None, fresh_context: bool = False) -> None:
        spec = inv.spec
        fd = self.data_for(spec)
        run = _Run(inv, plan, inv.gpu, dict(hooks) if hooks else {}, fd)
        run.t_enqueue = self.sim.engine.tick()
        inv.run = run
        slot = getattr(inv, "ctx_slot", None)
        if fresh_context or slot is not None:
            # FixedGSL instance, or DGSF: in the slot's pre-created context (a
            # slot whose context expired re-creates one inside its own plan)
            self._start_fixedgsl(run, fd, ctx=slot.handle if slot is not None and slot.handle else 0)
            return
        try:
            if fd.body != "resnet50" and self._fast_ok(plan):
                self._enqueue_fast(run, fd, wait_tokens)
            else:
                self._enqueue(run, fd, wait_tokens)
        except Exception:
            self._release(run)
            raise
        if run.invh:
            if not self._fast_source:
                self.sim.engine.add_source(self._fast)
                self._fast_source = True
            self._fast.runs[run.invh] = run
        else:
            self.sim.engine.watch(run.end, self._on_done, run)

    # ------------------------------------------------- one-call fast path -----
    def _fast_ok(self, plan: StagePlan) -> bool:
        """Plans whose DAG is the Parallel shape (also Serial plans without a
        GPU_CTX node, e.g. DGSF's pre-created contexts): one sage_invoke call."""
        return _plan_facts(plan).fast

    def _enqueue_fast(self, run: _Run, fd: FunctionData, wait_tokens) -> None:
        inv, plan, gpu = run.inv, run.plan, run.gpu
        pf = _plan_facts(plan)
        d = _lib.InvokeDesc.from_buffer_copy(_desc_template(fd, gpu))
        flags = 0
        if pf.cpu_ctx:
            t = self.sim.engine.tick()
            run.marks[Stage.CPU_CTX] = (t, t)     # host-side, synchronous
        in_dst, out_dst = self._input_dst(run, fd)
        grant = inv.grant
        resident = grant.resident if grant is not None else None
        if pf.gpu_ctx:
            flags |= _lib.INV_CTX
            d.ctx_dptr, d.ctx_bytes = self._ctx_dst(run)
        box = self.box
        publish = False
        peer = None
        ro = 0
        if fd.layout.seg_bytes:
            if resident is not None and resident.gpu_ro is not None:
                ro = resident.gpu_ro.dptr
            else:
                try:
                    ro = self._ro_dst(run)
                except SimulationError:
                    ro = 0
        if pf.gpu_load_ro and fd.layout.seg_bytes and resident is not None and resident.shares is not None:
            run.ro_source = "dedup"   # identical content already landed on this GPU: mapped, not loaded
        elif pf.gpu_load_ro and fd.layout.seg_bytes:
            if not ro:
                raise SimulationError(f"{inv}: no read-only segment to land into")
            flags |= _lib.INV_RO
            d.ro_dst = ro
            cache = resident.cpu_ro_cache.segment if (resident is not None and resident.cpu_ro_cache is not None) else None
            peer = self._peer_source(run) if pf.host_ro else None
            if not pf.host_ro and isinstance(cache, D.PinnedBuffer):
                # Stage2 / Stage3 rejoin: the pinned cache holds the landed bytes
                d.ro_kind, d.ro_src, d.ro_src_bytes = _lib.SRC_PINNED, cache.ptr, cache.nbytes
                if resident.cache_event is not None:
                    d.ro_wait[0] = resident.cache_event.h
                    d.n_ro_wait = 1
                run.ro_source = "cache"
            elif peer is not None:
                # PCIe once per box: land the resident peer copy over NVLink
                d.ro_kind, d.ro_src_gpu = _lib.SRC_PEER, peer.gpu
                d.ro_src, d.ro_src_bytes = peer.gpu_ro.dptr, fd.layout.seg_bytes
                if not peer.ro_token.ready and peer.ro_token.event is not None:
                    d.ro_wait[0] = peer.ro_token.event.h
                    d.n_ro_wait = 1
                run.ro_source = "nvlink"
            elif fd.db_dev is not None:
                d.ro_kind, d.ro_layout = _lib.SRC_HBM, fd.layout.handle()
                d.ro_src, d.ro_src_bytes = fd.db_dev.dptr, fd.layout.packed_bytes
                run.ro_source = "hbm"
            elif box is not None and grant is not None and grant.leader_ro and not box.is_home(inv.spec.name):
                # PCIe once per box (multi-process): the segment comes from its
                # home rank over NVLink; GPU_LOAD lands and verifies it locally
                nb = fd.layout.seg_bytes

                def scratch(n, run=run, gpu=gpu):
                    seg = self._scratch_get(gpu, n)
                    run.scratch.append(seg)
                    return seg
                how, src, ev = box.fetch(gpu, inv.spec.name, nb, scratch)
                run.events.append(ev)
                if how == "peer":   # one land reads the home's pages peer to peer
                    d.ro_kind, d.ro_src_gpu, d.ro_layout = _lib.SRC_PEER, gpu, 0
                    d.ro_src, d.ro_src_bytes = src, nb
                    run.ro_source = "nvlink"
                else:               # the bytes were copied into a local buffer
                    d.ro_kind, d.ro_layout, d.ro_src, d.ro_src_bytes = _lib.SRC_HBM, 0, src.dptr, nb
                    run.ro_source = "nccl"
                d.ro_wait[0] = ev.h
                d.n_ro_wait = 1
            else:
                d.ro_kind = _lib.SRC_PINNED if fd.db_pinned else _lib.SRC_HOST
                d.ro_layout = fd.layout.handle()
                d.ro_src, d.ro_src_bytes = fd.db.ctypes.data, fd.layout.packed_bytes
                run.ro_source = "pcie"
                publish = box is not None and grant is not None and grant.leader_ro
        if fd.input_bytes:
            flags |= _lib.INV_INPUT | (_lib.INV_VERIFY_INPUT if self.verify_inputs else 0)
            d.in_dst, d.in_bytes = in_dst, fd.input_bytes
            payload = inv.payload
            if payload is None and fd.input_dev is not None:
                d.in_kind, d.in_src = _lib.SRC_HBM, fd.input_dev.dptr
            else:
                p = self._payload(inv, fd)
                if isinstance(p, D.PinnedBuffer):
                    d.in_kind, d.in_src = _lib.SRC_PINNED, p.ptr
                else:
                    d.in_kind, d.in_src = _lib.SRC_HOST, p.ctypes.data
                run.keep = p
        n = 0
        if pf.sync:
            flags |= _lib.INV_SYNC
            for t in wait_tokens:
                if n < 2 and not t.ready and t.event is not None:
                    d.wait[n] = t.event.h
                    n += 1
        gate = self._gate_wait(run)
        if gate is not None:
            d.wait[n] = gate
            n += 1
        d.n_wait = n
        # COMPUTE: the function's body template (in the desc template) + this
        # invocation's pointers
        body = d.body
        body.ro, body.input, body.out = ro, in_dst, out_dst
        run.out_bytes = fd.out_bytes
        d.ret_src, d.ret_bytes = out_dst, fd.out_bytes
        if self.results_in_hbm:
            seg = self._scratch_get(gpu, max(256, fd.out_bytes))
            run.scratch.append(seg)
            d.ret_dst = seg.dptr
        else:
            run.result = self.pinned.get(max(16, fd.out_bytes))
            d.ret_dst = run.result.ptr
            flags |= _lib.INV_RET_HOST
        d.flags = flags
        h, done, ro_end, ctx_end = self._inv_out
        _lib.check(_lib.lib().sage_invoke(_lib.C.byref(d), *self._inv_out_refs), "sage_invoke")
        run.invh = h.value
        run.end = _Borrowed(done.value)
        self._gate_push(run)
        if run.ro_source == "nvlink" and peer is not None:
            _add_reader(peer, ro_end.value or done.value)
        if publish:
            # home rank: send the landed segment to the other ranks; eviction
            # waits for the send (sharing._evict)
            ev = box.publish(gpu, ro, fd.layout.seg_bytes, _Borrowed(ro_end.value),
                             seg_handle=resident.gpu_ro.segment.h, name=inv.spec.name)
            if resident.ro_busy is not None:
                resident.ro_busy.release()
            resident.ro_busy = ev
        if run.hooks:
            tok = run.hooks.get(Stage.GPU_LOAD)
            if tok is not None:
                tok.attach(_Borrowed(ro_end.value or done.value))
            tok = run.hooks.get(Stage.GPU_CTX)
            if tok is not None:
                tok.attach(_Borrowed(ctx_end.value or done.value))

    def _collect_fast(self, run: _Run) -> None:
        inv = run.inv
        info = _lib.InvokeInfo()
        rc = _lib.check(_lib.lib().sage_invoke_collect(run.invh, _lib.C.byref(info)), "sage_invoke_collect")
        if rc == _lib.SAGE_ENOTREADY:
            raise SimulationError(f"{inv}: collected before completion")
        to_eng = self.sim.engine.to_engine_time
        t = info.t
        stages = inv.stages
        for k, st in _plan_facts(run.plan).timed:
            if t[2 * k] >= 0:
                stages[st] = [to_eng(t[2 * k]), to_eng(t[2 * k + 1])]
        for st, (b, e) in run.marks.items():
            stages[st] = [self._t(b), self._t(e)]
        m = inv.measured
        m["host_bytes"] = info.host_bytes
        if run.ro_source == "nccl":             # RO bytes came over NVLink, landed from HBM
            m["nvlink_bytes"] = run.fd.layout.seg_bytes
            m["pcie_bytes"] = info.link_bytes
        elif run.ro_source == "nvlink":
            m["nvlink_bytes"] = run.fd.layout.seg_bytes
            m["pcie_bytes"] = info.link_bytes - run.fd.layout.seg_bytes
        else:
            m["pcie_bytes"] = info.link_bytes
        if info.ro_landed_us >= 0:
            self._verify_ro(run, info.ro_checksum)
            inv.ro_landed_us = to_eng(info.ro_landed_us)
        if run.fd.input_bytes:
            inv.input_checksum = info.in_checksum
        inv.ro_source = run.ro_source
        if isinstance(run.result, D.PinnedBuffer) and run.out_bytes:
            inv.result = run.result.view()[:run.out_bytes]

    def _input_dst(self, run: _Run, fd: FunctionData) -> tuple[int, int]:
        """(input dptr, out dptr) inside the private writable allocation, or an
        unaccounted scratch segment when writable is too small."""
        inv = run.inv
        need = _a256(fd.input_bytes + 16) + _a256(fd.out_bytes) + fd.scratch_bytes
        wr = inv.private.get(AllocClass.WRITABLE) if inv.private else None
        if wr is None:
            wr = next((a for a in inv.allocations if a.cls is AllocClass.WRITABLE), None)
        if wr is not None and wr.requested >= need and wr.dptr:
            base = wr.dptr
        else:
            seg = self._scratch_get(run.gpu, need)
            run.scratch.append(seg)
            base = seg.dptr
        return base, base + _a256(fd.input_bytes + 16)

    def _ro_dst(self, run: _Run) -> int:
        inv = run.inv
        grant = getattr(inv, "grant", None)
        if grant is not None and grant.resident.gpu_ro is not None:
            return grant.resident.gpu_ro.dptr          # the shared segment (leader or follower)
        for a in inv.allocations:                      # private RO (SAGE-NR, DGSF)
            if a.cls is AllocClass.READ_ONLY:
                return a.dptr
        raise SimulationError(f"{inv}: no read-only segment to land into")

    def _ctx_dst(self, run: _Run) -> tuple[int, int]:
        inv = run.inv
        grant = getattr(inv, "grant", None)
        if grant is not None and grant.leader_ctx:
            a = grant.resident.gpu_ctx
            return a.dptr, a.requested
        for a in inv.allocations:
            if a.cls is AllocClass.CONTEXT:
                return a.dptr, a.requested
        slot = getattr(inv, "ctx_slot", None)
        if slot is not None and slot.seg is not None:
            return slot.seg.dptr, slot.seg.requested
        return 0, 0

    def _peer_source(self, run: _Run):
        """A resident, landed copy of this function's RO on another GPU."""
        sim = self.sim
        if sim.gpu_count < 2 or not sim.policy_cfg.fanout or sim.sharing is None:
            return None
        name = run.inv.spec.name
        best = None
        for (n, g), r in sim.sharing.residents.items():
            if n == name and g != run.gpu and r.gpu_ro is not None and r.ro_token is not None:
                if best is None or r.ro_token.ready:
                    best = r
        return best

    def _enqueue(self, run: _Run, fd: FunctionData, wait_tokens) -> None:
        inv, plan, gpu = run.inv, run.plan, run.gpu
        nodes = plan.nodes
        ends: list[list] = [[] for _ in nodes]
        run.slot = self._slot(gpu)
        ev = run.events
        in_dst, out_dst = self._input_dst(run, fd)
        grant = getattr(inv, "grant", None)
        resident = grant.resident if grant is not None else None
        serial = plan.mode is PlanMode.SERIAL
        i_cpu = plan.node_index(Stage.CPU_LOAD)
        i_gpu = plan.node_index(Stage.GPU_LOAD)
        staged_ro = staged_in = None   # serial: pinned copies made by CPU_LOAD
        for i, node in enumerate(nodes):
            deps = [e for p in node.preds for e in ends[p]]
            st = node.stage
            if st in (Stage.CONTAINER, Stage.CPU_CTX):
                t = self.sim.engine.tick()
                run.marks[st] = (t, t)           # host-side, synchronous
            elif st is Stage.CPU_LOAD:
                if not serial:
                    continue                     # fused into the GPU_LOAD pipeline
                ops = []
                if node.ro and fd.layout.packed_bytes:
                    staged_ro = self.pinned.get(fd.layout.packed_bytes)
                    run.pinned.append(staged_ro)
                    b, e, _ = D.host_load(gpu, staged_ro, fd.db, deps)
                    ops += [b, e]
                    ends[i].append(e)
                if fd.input_bytes:
                    staged_in = self.pinned.get(fd.input_bytes)
                    run.pinned.append(staged_in)
                    b, e, _ = D.host_load(gpu, staged_in, self._payload(inv, fd), deps)
                    ops += [b, e]
                    ends[i].append(e)
                ev.extend(ops)
                run.marks[st] = (ops[0], ops[-1]) if ops else (self.sim.engine.tick(),) * 2
            elif st is Stage.GPU_CTX:
                dptr, nb = self._ctx_dst(run)
                b, e = run.slot.bind_ctx(dptr, nb, deps)
                ev += [b, e]
                ends[i].append(e)
                run.marks[st] = (b, e)
                tok = run.hooks.get(Stage.GPU_CTX)
                if tok is not None:
                    tok.attach(e)
            elif st is Stage.GPU_LOAD:
                cpu_deps = [e for p in nodes[i_cpu].preds for e in ends[p]] if (i_cpu is not None and not serial) else []
                wait = deps + cpu_deps
                ro_end = None
                borrowed = resident is not None and resident.shares is not None
                if node.ro and fd.layout.seg_bytes and not borrowed:
                    ro_end = self._load_ro(run, fd, resident, wait, staged_ro)
                    ends[i].append(ro_end)
                elif borrowed:
                    run.ro_source = "dedup"      # identical content already landed: mapped, not loaded
                if fd.input_bytes:
                    if fd.input_dev is not None and getattr(inv, "payload", None) is None:
                        op = D.load(gpu, in_dst, None, None, device_src=fd.input_dev.dptr,
                                    device_src_bytes=fd.input_bytes, wait=wait)
                    else:
                        src = staged_in if staged_in is not None else self._payload(inv, fd)
                        op = D.load(gpu, in_dst, src, None, pinned=staged_in is not None, wait=wait)
                    run.loads.append(("input", op))
                    ends[i].append(op.end)
                if not ends[i]:
                    e = run.slot.record()
                    ev.append(e)
                    ends[i].append(e)
                tok = run.hooks.get(Stage.GPU_LOAD)
                if tok is not None:
                    tok.attach(ro_end if ro_end is not None else ends[i][0])
            elif st is Stage.SYNC_WAIT:
                tok_evs = [t.event for t in wait_tokens if not t.ready and t.event is not None]
                b, e = run.slot.sync_wait(deps + tok_evs)
                ev += [b, e]
                ends[i].append(e)
                run.marks[st] = (b, e)
            elif st is Stage.COMPUTE:
                gate = self._gate_wait(run)
                if gate is not None:
                    deps = list(deps) + [_Borrowed(gate)]
                if fd.body == "resnet50":
                    # DNN body: PyTorch on the invocation's stream, weights read in
                    # place from the landed (shared) segment
                    from . import dnn
                    run.slot.wait(deps)
                    b = run.slot.record()
                    dnn.run_resnet50(fd, self._ro_dst(run), in_dst, out_dst, run.slot.stream(),
                                     _lib.gpu_device(gpu), plane=gpu)
                    e = run.slot.record()
                else:
                    body = self._body(run, fd, resident, in_dst, out_dst)
                    b, e = run.slot.launch_after(deps, body)
                ev += [b, e]
                ends[i].append(e)
                run.marks[st] = (b, e)
            elif st is Stage.RETURN:
                run.out_bytes = fd.out_bytes
                if self.results_in_hbm:
                    # device-resident measurement: results stay in HBM (D2D)
                    seg = D.pool_alloc(gpu, max(256, fd.out_bytes), _lib.CLASS_WRITABLE, unaccounted=True)
                    run.scratch.append(seg)
                    b, e = run.slot.ret_after(deps, out_dst, seg.dptr, fd.out_bytes)
                else:
                    run.result = self.pinned.get(max(16, fd.out_bytes))
                    b, e = run.slot.ret_after(deps, out_dst, run.result.ptr, fd.out_bytes)
                ev += [b, e]
                ends[i].append(e)
                run.marks[st] = (b, e)
                run.end = e
        if run.end is None:
            raise SimulationError("plan has no RETURN node")
        self._gate_push(run)

    def _payload(self, inv, fd: FunctionData):
        p = getattr(inv, "payload", None)
        if p is None:
            return fd.input
        if p.nbytes != fd.input_bytes:
            raise ValueError(f"{inv}: payload of {p.nbytes} B, function expects {fd.input_bytes} B")
        return p

    def _load_ro(self, run: _Run, fd: FunctionData, resident, wait, staged_ro) -> D.Event:
        gpu = run.gpu
        dst = self._ro_dst(run)
        plan = run.plan
        i_cpu = plan.node_index(Stage.CPU_LOAD)
        host_ro = i_cpu is not None and plan.nodes[i_cpu].ro
        if staged_ro is not None:                                   # serial: from pinned staging
            op = D.load(gpu, dst, staged_ro, fd.layout, wait=wait)
            run.ro_source = "pcie"
        elif not host_ro and resident is not None and resident.cpu_ro_cache is not None \
                and isinstance(resident.cpu_ro_cache.segment, D.PinnedBuffer):
            # Stage2 / Stage3 rejoin: re-land the cached (already unpacked) segment
            w = list(wait) + ([resident.cache_event] if resident.cache_event is not None else [])
            op = D.load(gpu, dst, resident.cpu_ro_cache.segment, None, wait=w)
            run.ro_source = "cache"
        else:
            peer = self._peer_source(run) if host_ro else None
            if peer is not None:
                # PCIe once per box: land from the resident peer copy over NVLink
                w = list(wait) + ([peer.ro_token.event] if (not peer.ro_token.ready and peer.ro_token.event) else [])
                op = D.load(gpu, dst, None, None, device_src=peer.gpu_ro.dptr,
                            device_src_bytes=fd.layout.seg_bytes, peer_gpu=peer.gpu, wait=w)
                run.ro_source = "nvlink"
                _add_reader(peer, op.end.h)
            elif fd.db_dev is not None:
                op = D.load(gpu, dst, None, fd.layout, device_src=fd.db_dev.dptr,
                            device_src_bytes=fd.layout.packed_bytes, wait=wait)
                run.ro_source = "hbm"
            else:
                op = D.load(gpu, dst, fd.db, fd.layout, pinned=fd.db_pinned, wait=wait)
                run.ro_source = "pcie"
        run.loads.append(("ro", op))
        return op.end

    def _body(self, run: _Run, fd: FunctionData, resident, in_dst: int, out_dst: int):
        inv = run.inv
        ro = 0
        if fd.layout.seg_bytes:
            try:
                ro = self._ro_dst(run)
            except SimulationError:
                ro = 0
        in_bytes = (fd.input_bytes + 15) // 16 * 16
        return D.body_desc(_BODY[fd.body], ro=ro, ro_bytes=fd.layout.seg_bytes, inp=in_dst, inp_bytes=in_bytes,
                           out=out_dst, out_bytes=max(16, fd.out_bytes), args=fd.args)

    # ----------------------------------------------------------- FixedGSL -----
    def _start_fixedgsl(self, run: _Run, fd: FunctionData, ctx: int = 0) -> None:
        """An instance job: FixedGSL (a fresh context, on a library thread or
        -- ClusterSpec.instance_mode "process" -- in its own OS process), or
        DGSF in a pre-created context `ctx` (data reserved per invocation)."""
        inv = run.inv
        spec = inv.spec
        run.result = self.pinned.get(max(16, fd.out_bytes))
        run.out_bytes = fd.out_bytes
        if ctx:
            mode, reserve = _lib.INSTANCE_POOLED, sum(a.effective for a in inv.allocations)
        else:
            mode = _lib.INSTANCE_PROCESS if self.sim.cluster.instance_mode == "process" else _lib.INSTANCE_THREAD
            alloc = inv.allocations[0].effective if inv.allocations else 0
            reserve = max(0, alloc - spec.context_bytes)
        body = D.body_desc(_BODY[fd.body], out_bytes=max(16, fd.out_bytes), args=fd.args)
        run.job = D.fixedgsl_submit(run.gpu, fd.layout if fd.layout.n else None,
                                    fd.db if fd.layout.packed_bytes else None, self._payload(inv, fd),
                                    reserve, body, run.result, fd.out_bytes, mode=mode, ctx=ctx)
        run.end = run.job.end
        run.ro_source = "pcie"
        self.sim.engine.watch(run.end, self._on_done, run)

    # ---------------------------------------------------------- completion ----
    def _t(self, x) -> Optional[int]:
        if x is None:
            return None
        if isinstance(x, int):
            return x
        return self.sim.engine.to_engine_time(x.time_us())

    def _on_done(self, run: _Run) -> None:
        inv = run.inv
        eng = self.sim.engine
        try:
            self._collect(run)
            for tok in run.hooks.values():
                tok.set_ready(eng.now)
            # listeners see inv.result as a zero-copy view of the returned bytes
            self.sim._on_invocation_done(inv, eng.now)
            if inv.result is not None:
                inv.result = inv.result.copy() if self.sim.copy_results else None
        finally:
            for tok in run.hooks.values():
                tok.set_ready(eng.now)
            self._release(run)

    def _collect(self, run: _Run) -> None:
        inv = run.inv
        if run.invh:
            self._collect_fast(run)
            return
        if run.job is not None:
            info = run.job.info()
            if info is None or info.status != 0:
                raise SimulationError(f"{inv}: FixedGSL instance failed ({info.status if info else '?'}): "
                                      f"{_lib.last_error()}")
            for k, stage in enumerate([Stage.CONTAINER, Stage.CPU_CTX, Stage.CPU_LOAD, Stage.GPU_CTX,
                                       Stage.GPU_LOAD, Stage.SYNC_WAIT, Stage.COMPUTE, Stage.RETURN]):
                b, e = info.t[2 * k], info.t[2 * k + 1]
                if b >= 0:
                    inv.stages[stage] = [self.sim.engine.to_engine_time(b), self.sim.engine.to_engine_time(e)]
            inv.ro_checksum = info.checksum
            inv.teardown_us = info.teardown_us
            inv.measured["pcie_bytes"] = run.fd.layout.packed_bytes + run.fd.input_bytes
            inv.measured["host_bytes"] = run.fd.layout.packed_bytes
        else:
            for st, (b, e) in run.marks.items():
                inv.stages[st] = [self._t(b), self._t(e)]
            cpu_b = cpu_e = gpu_b = gpu_e = None
            hb = lb = 0
            for kind, op in run.loads:
                li = op.info()
                if li is None:
                    raise SimulationError(f"{inv}: load not complete at RETURN")
                if li.cpu_begin_us >= 0:
                    cpu_b = li.cpu_begin_us if cpu_b is None else min(cpu_b, li.cpu_begin_us)
                    cpu_e = li.cpu_end_us if cpu_e is None else max(cpu_e, li.cpu_end_us)
                gpu_b = li.gpu_begin_us if gpu_b is None else min(gpu_b, li.gpu_begin_us)
                gpu_e = li.gpu_end_us if gpu_e is None else max(gpu_e, li.gpu_end_us)
                hb += li.host_bytes
                lb += li.link_bytes
                if kind == "ro":
                    self._verify_ro(run, li.checksum)
                    inv.ro_landed_us = self.sim.engine.to_engine_time(li.gpu_end_us)
                else:
                    inv.input_checksum = li.checksum
            inv.measured["host_bytes"] = hb
            inv.measured[run.ro_source + "_bytes" if run.ro_source == "nvlink" else "pcie_bytes"] = lb
            eng = self.sim.engine
            if Stage.GPU_LOAD not in run.marks and gpu_b is not None:
                inv.stages[Stage.GPU_LOAD] = [eng.to_engine_time(gpu_b), eng.to_engine_time(gpu_e)]
            elif Stage.GPU_LOAD not in run.marks:
                t = self._t(run.t_enqueue)
                inv.stages[Stage.GPU_LOAD] = [t, t]
            if run.plan.node_index(Stage.CPU_LOAD) is not None and Stage.CPU_LOAD not in run.marks:
                if cpu_b is not None:
                    inv.stages[Stage.CPU_LOAD] = [eng.to_engine_time(cpu_b), eng.to_engine_time(cpu_e)]
                else:
                    t = run.t_enqueue
                    inv.stages[Stage.CPU_LOAD] = [t, t]
        inv.ro_source = run.ro_source
        if isinstance(run.result, D.PinnedBuffer) and run.out_bytes:
            inv.result = run.result.view()[:run.out_bytes]

    def _verify_ro(self, run: _Run, checksum: int) -> None:
        inv = run.inv
        inv.ro_checksum = checksum
        fd = run.fd
        grant = getattr(inv, "grant", None)
        r = grant.resident if grant is not None else None
        if fd.ro_checksum is None:
            fd.ro_checksum = checksum
        elif fd.ro_checksum != checksum:
            raise SimulationError(f"{inv}: landed read-only segment checksum {checksum:016x} != "
                                  f"{fd.ro_checksum:016x} (source {run.ro_source})")
        if r is not None and grant.leader_ro and r.gpu_ro is not None and r.ro_checksum is None:
            self.sim.sharing.record_checksum(r, checksum)    # the content index of the native table

    def _release(self, run: _Run) -> None:
        if run.invh:
            _lib.check(_lib.lib().sage_invoke_release(run.invh), "sage_invoke_release")
            run.invh = 0
            run.keep = None
        for _, op in run.loads:
            op.release()
        run.loads.clear()
        for e in run.events:
            e.release()
        run.events.clear()
        if run.slot is not None:
            self._free_slots.setdefault(run.slot.gpu, []).append(run.slot)   # back to the pool
            run.slot = None
        for b in run.pinned:
            self.pinned.put(b)
        run.pinned.clear()
        if run.result is not None:
            self.pinned.put(run.result)
            run.result = None
        for s in run.scratch:     # device work on them is complete: back to the pool
            self._scratch.setdefault((s.gpu, s.nbytes), []).append(s)
        run.scratch.clear()
        if run.job is not None:
            run.job.release()
            run.job = None
        if run.inv is not None and run.inv.run is run:
            run.inv.run = None   # break inv <-> run: finished records free by refcount

    def close(self) -> None:
        self.unpin_host_store()
        self.drop_hbm_sources()
        for lst in self._scratch.values():
            for seg in lst:
                seg.free()
        self._scratch.clear()
        for lst in self._free_slots.values():
            for s in lst:
                s.release()
        self._free_slots.clear()
        for h in list(self._contexts):
            self.release_context(h)
        self.pinned.close()
