"""The invocation API on real B200s.

Drop-in for gslsim.simulation (pkg/src/gslsim/simulation.py): `ClusterSpec`
(:23-37), the `Invocation` record with stage timestamps and per-channel bytes
(:40-93), and `Simulation` with `submit` (:163-170), `start_invocation`
(:174-187), `fail_invocation` (:189-192), `_on_invocation_done` (:194-200),
`completion_listeners` (:151), `run` (:227-232) and `check_no_leaks`
(:237-254).  The class keeps the reference's name so callers switch by
import; it is not a simulation: stages run on the GPU, times are the wall
clock (engine.py), and `Invocation.stages` are measured.

Reported per invocation (reference semantics, metrics.py:184-213):
  setup_us = compute_begin - arrival       (the headline latency)
  host_bytes_umb / pcie_bytes_umb          PLANNED bytes, reference units
  measured{host,pcie,nvlink}_bytes         bytes the hardware moved
"""
from __future__ import annotations

import gc
import itertools
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .dataplane import DataPlane, FunctionData
from .engine import DISPATCH_STREAM, Engine, EventKind, rng_stream, s_to_us
from .functions import ComputeGate, FunctionSpec, Stage, StagePlan, WarmthClass
from .policies import PolicyConfig, PoolPolicy, SharingPolicy, build_policy
from .resources import DevicePool, MemoryLedger, SimulationError
from .sharing import SharingManager

OUTCOME_COMPLETED = "completed"
OUTCOME_FAILED = "failed"
OUTCOME_PENDING = "pending"
B200_BUDGET_MB = 171_661          # 180 GB (= 171,661 MiB) pool budget per GPU (BASELINE cfg 4)


@dataclass(frozen=True)
class ClusterSpec:
    """Reference fields (simulation.py:23-37) + the real plane's sizing.
    pcie_bw_mbps / host_bw_mbps are kept for config compatibility only: the
    hardware sets the bandwidth now."""
    gpus: int = 1
    gpu_mem_mb: float = B200_BUDGET_MB
    pcie_bw_mbps: float = 5051.0
    host_bw_mbps: float = 1631.0
    cpu_mem_mb: Optional[float] = None
    compute_concurrency: Optional[int] = None
    pre_warmed_containers: bool = True
    # admission window: at most this many started, unfinished invocations per
    # GPU; later arrivals wait in the dispatcher's FIFO (None: unlimited, the
    # reference's rule -- admission is bounded by memory only).  A window keeps
    # a backlog above capacity on the host instead of growing device-side
    # state for it (streams, segments, pinned buffers)
    admission_window: Optional[int] = None
    chunk_mb: float = 32.0     # staged-load chunk: one H2D + one land launch each (8 / 16 / 32 MiB: e2e 3,616 / 3,706 / 3,728 inv/s)
    staging_mb: float = 256.0  # 8 ring slots
    host_threads: Optional[int] = None
    # FixedGSL instances: "thread" (a fresh context on a library thread) or
    # "process" (a fresh OS process per instance, the container-per-function shape)
    instance_mode: str = "thread"

    def __post_init__(self):
        if self.gpus < 1:
            raise ValueError("cluster needs at least one GPU")
        if self.instance_mode not in ("thread", "process"):
            raise ValueError(f"instance_mode must be 'thread' or 'process', not {self.instance_mode!r}")
        if self.gpu_mem_mb <= 0 or self.pcie_bw_mbps <= 0 or self.host_bw_mbps <= 0:
            raise ValueError("cluster capacities and bandwidths must be positive")


class Invocation:
    __slots__ = ("id", "spec", "arrival_us", "gpu", "start_us", "completion_us", "warmth", "outcome", "stages",
                 "host_bytes_umb", "pcie_bytes_umb", "allocations", "grant", "ctx_slot", "was_queued",
                 "fail_reason", "private", "run", "payload", "result", "measured", "ro_checksum",
                 "input_checksum", "ro_source", "teardown_us", "ro_landed_us")

    def __init__(self, iid: int, spec: FunctionSpec, arrival_us: int, payload=None):
        self.id = iid
        self.spec = spec
        self.arrival_us = arrival_us
        self.gpu: Optional[int] = None
        self.start_us: Optional[int] = None
        self.completion_us: Optional[int] = None
        self.warmth: Optional[WarmthClass] = None
        self.outcome = OUTCOME_PENDING
        self.stages: dict = {}
        self.host_bytes_umb = 0
        self.pcie_bytes_umb = 0
        self.allocations: list = []
        self.grant = None
        self.ctx_slot = None
        self.was_queued = False
        self.fail_reason: Optional[str] = None
        self.private: dict = {}
        self.run = None
        self.payload = payload
        self.result: Optional[np.ndarray] = None
        self.measured: dict = {"host_bytes": 0, "pcie_bytes": 0, "nvlink_bytes": 0}
        self.ro_checksum: Optional[int] = None
        self.input_checksum: Optional[int] = None
        self.ro_source = ""
        self.teardown_us = None
        self.ro_landed_us: Optional[int] = None   # when this invocation's RO load landed

    def mark_queued(self) -> None:
        self.was_queued = True

    @property
    def latency_us(self) -> Optional[int]:
        return None if self.completion_us is None else self.completion_us - self.arrival_us

    @property
    def queued_us(self) -> Optional[int]:
        return None if self.start_us is None else self.start_us - self.arrival_us

    @property
    def setup_us(self) -> Optional[int]:
        """compute_begin - arrival (the headline setup latency)."""
        c = self.stages.get(Stage.COMPUTE)
        return None if c is None else c[0] - self.arrival_us

    def __repr__(self):
        return f"Invocation({self.id}, {self.spec.name}, t={self.arrival_us})"


class _quiet_gc:
    """No cyclic-GC pass while the wall-clock loop serves invocations: a
    generation-2 collection over the run's invocation records stalls the
    loop for tens of ms (measured: cfg-2 Poisson probes at 100/s with a p99
    of 35-64 ms in the last quarter), which an open-loop arrival stream turns
    into a backlog.  Reference counting still frees every finished record;
    the collector runs again after the loop (a serving process tunes its
    collector the same way)."""

    def __enter__(self):
        import gc
        self._was = gc.isenabled()
        gc.disable()

    def __exit__(self, *exc):
        import gc
        if self._was:
            gc.enable()
        return False


class Simulation:
    """One runtime instance of one policy on the local GPUs (the drop-in)."""

    def __init__(self, cluster: ClusterSpec, policy_cfg: PolicyConfig, spec_table: dict, source=None, seed: int = 0,
                 duration_us: int = 0, log_events: bool = False, register_functions=None,
                 function_data: Optional[dict] = None, init_device: bool = True, copy_results: bool = True):
        self.cluster = cluster
        self.policy_cfg = policy_cfg
        self.spec_table = spec_table
        self.seed = seed
        self.duration_us = duration_us
        self.gpu_count = cluster.gpus
        self.pre_warmed = cluster.pre_warmed_containers
        self._owns_device = False
        if init_device and not _lib.is_up():
            flags = _lib.SAGE_INIT_PEER_ACCESS if cluster.gpus > 1 else 0
            if cluster.gpus > _lib.device_count():
                # more logical GPUs than devices: independent planes share a
                # device (tests the multi-GPU control plane on one GPU)
                flags |= _lib.SAGE_INIT_SHARE_DEVICE
            per_gpu = int(cluster.gpu_mem_mb * (1 << 20)) + (8 << 30)
            _lib.init(n_gpus=cluster.gpus, pool_bytes=per_gpu, staging_bytes=int(cluster.staging_mb * (1 << 20)),
                      chunk_bytes=int(cluster.chunk_mb * (1 << 20)), flags=flags, host_threads=cluster.host_threads)
            self._owns_device = True
        self.engine = Engine(log_events=log_events)
        self.dispatcher_rng = rng_stream(seed, DISPATCH_STREAM)
        gran = policy_cfg.granularity_bytes
        cap = int(round(cluster.gpu_mem_mb * (1 << 20)))
        self.gpu_ledgers = [MemoryLedger(f"gpu{g}", cap, gran, backend=DevicePool(g)) for g in range(cluster.gpus)]
        cpu_cap = None if cluster.cpu_mem_mb is None else int(round(cluster.cpu_mem_mb * (1 << 20)))
        self.cpu_ledger = MemoryLedger("cpu", cpu_cap)
        self.compute_gates = None
        if cluster.compute_concurrency is not None:
            self.compute_gates = [ComputeGate(cluster.compute_concurrency) for _ in range(cluster.gpus)]
        self.dataplane = DataPlane(self)
        for name, data in (function_data or {}).items():
            self.dataplane.register(name, data)
        self.sharing: Optional[SharingManager] = None
        self.policy = build_policy(self, policy_cfg)
        if isinstance(self.policy, SharingPolicy):
            intervals = policy_cfg.stage_interval_s
            if not isinstance(intervals, (list, tuple)):
                intervals = (intervals,) * 4
            self.sharing = SharingManager(self.engine, self.gpu_ledgers, self.cpu_ledger,
                                          ro_sharing=policy_cfg.ro_sharing, ctx_sharing=policy_cfg.ctx_sharing,
                                          multi_stage_exit=policy_cfg.multi_stage_exit,
                                          keep_alive_s=policy_cfg.keep_alive_s, stage_intervals_s=intervals,
                                          on_gpu_freed=self.policy.on_memory_freed, dataplane=self.dataplane)
        if isinstance(self.policy, PoolPolicy):
            names = register_functions if register_functions is not None else sorted(spec_table)
            for name in names:
                self.policy.register(self.spec_table[name])
        # copy_results=False: inv.result is only valid inside completion
        # listeners (zero-copy view of the pinned return buffer)
        self.copy_results = copy_results
        self.invocations: list[Invocation] = []
        self.completion_listeners = []
        self._ids = itertools.count()
        self._in_flight = 0
        self._in_flight_gpu = [0] * cluster.gpus
        self._window = cluster.admission_window
        self.source = source
        # a serving process: move everything allocated so far (torch, function
        # data) out of the cyclic collector's reach so a full collection
        # during a burst stays short (measured: ~7 ms hiccups otherwise)
        gc.collect()
        gc.freeze()
        if source is not None:
            source.attach(self)

    # -- registration (extension: the bytes a function loads) ------------------------
    def register_data(self, name: str, data: FunctionData) -> None:
        if name not in self.spec_table:
            raise SimulationError(f"unknown function {name!r}")
        self.dataplane.register(name, data)

    def prepare(self, names=None) -> None:
        """Registration-time work for `names` (default: every function):
        materialise the data, upload the landing plans.  Keeps first-
        invocation setup free of one-off costs, as a deployed function is."""
        for name in (names if names is not None else sorted(self.spec_table)):
            fd = self.dataplane.data_for(self.spec_table[name])
            if fd.layout.n:
                fd.layout.handle()
            if fd.body == "resnet50":
                from . import dnn
                for dev in sorted({_lib.gpu_device(g) for g in range(self.gpu_count)}):
                    dnn.prewarm(fd, dev)
            elif fd.body == "resnet50_native":
                from . import dnn
                dnn.native_handle(fd)

    def prewarm(self, concurrency: int, names=None) -> None:
        """Deployment-time warm-up: one burst of `concurrency` invocations
        (round robin over `names`, default every function) per GPU, drained,
        then every resident evicted and the burst forgotten.  The plane's
        lazily grown resources -- pooled streams, writable segments (pool
        chunks), pinned return buffers, events -- then exist for that many
        concurrent invocations, so an open-loop arrival stream that first
        reaches that concurrency does not stall on their creation (a stall
        under Poisson arrivals builds a backlog that needs still more of
        them)."""
        names = list(names if names is not None else sorted(self.spec_table))
        if concurrency <= 0 or not names:
            return
        first = len(self.invocations)
        self.submit_many([names[k % len(names)] for k in range(concurrency * self.gpu_count)])
        self.drain()
        if self.sharing is not None:
            for r in list(self.sharing.residents.values()):
                self.sharing.evict(r)
        del self.invocations[first:]

    # -- workload entry points ----------------------------------------------------------
    def submit(self, fn_name: str, arrival_us: Optional[int] = None, payload=None) -> Invocation:
        if fn_name not in self.spec_table:
            raise SimulationError(f"unknown function {fn_name!r}")
        now = self.engine.tick()
        inv = Invocation(next(self._ids), self.spec_table[fn_name], now if arrival_us is None else arrival_us,
                         payload)
        self.invocations.append(inv)
        self.policy.on_arrival(inv)
        return inv

    def submit_many(self, fn_names, payloads=None) -> list[Invocation]:
        """A burst arriving at one instant (the BASELINE concurrent configs)."""
        now = self.engine.tick()
        out = []
        for k, name in enumerate(fn_names):
            out.append(self.submit(name, arrival_us=now, payload=None if payloads is None else payloads[k]))
        return out

    # -- policy callbacks ----------------------------------------------------------------
    def start_invocation(self, inv: Invocation, warmth: WarmthClass, plan: StagePlan, wait_tokens=(),
                         stage_hooks=None, fresh_context: bool = False) -> None:
        inv.start_us = self.engine.tick()
        inv.warmth = warmth
        moved = plan.__dict__.get("_moved")
        if moved is None:   # (host, PCIe) bytes the plan moves, once per (immutable) plan
            moved = plan.__dict__["_moved"] = (
                sum(n.bytes_umb for n in plan.nodes if n.stage is Stage.CPU_LOAD),
                sum(n.bytes_umb for n in plan.nodes if n.stage is Stage.GPU_LOAD))
        inv.host_bytes_umb += moved[0]
        inv.pcie_bytes_umb += moved[1]
        self._in_flight += 1
        self._in_flight_gpu[inv.gpu] += 1
        self.dataplane.start(inv, plan, wait_tokens, stage_hooks, fresh_context=fresh_context)

    def fail_invocation(self, inv: Invocation, reason: str) -> None:
        inv.outcome = OUTCOME_FAILED
        inv.fail_reason = reason
        inv.completion_us = self.engine.now

    def _on_invocation_done(self, inv: Invocation, now: int) -> None:
        inv.outcome = OUTCOME_COMPLETED
        inv.completion_us = now
        self._in_flight -= 1
        self._in_flight_gpu[inv.gpu] -= 1
        self.policy.complete(inv)
        if self._window is not None:
            self.policy.on_memory_freed(inv.gpu)   # a window slot opened: start the next waiting
        for cb in self.completion_listeners:
            cb(inv, now)

    def window_open(self, gpu: int) -> bool:
        """Room in GPU `gpu`'s admission window (ClusterSpec.admission_window)."""
        return self._window is None or self._in_flight_gpu[gpu] < self._window

    # -- run -------------------------------------------------------------------------------
    @property
    def in_flight(self) -> int:
        return self._in_flight

    def idle(self) -> bool:
        src_done = self.source is None or getattr(self.source, "exhausted", True)
        return self._in_flight == 0 and self.policy.queued_count() == 0 and src_done

    def run(self, until: Optional[int] = None) -> "Simulation":
        """With `until` (engine µs): run the wall clock to it, like the
        reference's fixed-duration run.  Without: until every submitted
        invocation completed (decay timers stay armed)."""
        if until is None:
            until = self.duration_us or None
        with _quiet_gc():
            if until is None:
                self.engine.run(idle=self.idle)
            else:
                self.engine.run(until=until)
        return self

    def drain(self) -> "Simulation":
        with _quiet_gc():
            self.engine.run(idle=self.idle)
        return self

    def queued_at_end(self) -> int:
        return self.policy.queued_count()

    def check_no_leaks(self) -> None:
        persistent = 0
        if self.sharing is not None:
            persistent += self.sharing.held_bytes()
        if isinstance(self.policy, PoolPolicy):
            for pool in self.policy.pools.values():
                for slot in pool.contexts:
                    if slot.seg is not None:
                        persistent += slot.seg.effective
        actual = sum(l.usage for l in self.gpu_ledgers)
        if actual != persistent:
            raise SimulationError(f"GPU memory leak: {actual} B held vs {persistent} B persistent")
        for l in self.gpu_ledgers:
            l.check_native()

    def close(self) -> None:
        """Free everything and shut the device plane down."""
        if self.sharing is not None:
            self.sharing.close()
        if isinstance(self.policy, PoolPolicy):
            for (name, gpu), pool in self.policy.pools.items():
                for slot in pool.contexts:
                    if slot.seg is not None:
                        self.gpu_ledgers[gpu].free(slot.seg)
                        slot.seg = None
        self.dataplane.close()
        if self._owns_device:
            _lib.shutdown()
            self._owns_device = False

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ------------------------------------------------------------------ metrics ---
def percentile(samples, p) -> float:
    """Nearest-rank percentile (reference metrics.py:29-37)."""
    import math
    from fractions import Fraction
    if not 0 <= p <= 100:
        raise ValueError(f"percentile p must be in [0, 100], got {p}")
    n = len(samples)
    if n == 0:
        raise ValueError("percentile of empty sample set")
    rank = max(1, math.ceil(Fraction(p) * n / 100))
    return sorted(samples)[rank - 1]


def summarize_setup(invocations) -> dict:
    done = [i for i in invocations if i.outcome == OUTCOME_COMPLETED]
    setups = [i.setup_us for i in done if i.setup_us is not None]
    lats = [i.latency_us for i in done]
    out = {"completed": len(done), "failed": sum(i.outcome == OUTCOME_FAILED for i in invocations)}
    if setups:
        out.update(setup_p50_ms=percentile(setups, 50) / 1e3, setup_p99_ms=percentile(setups, 99) / 1e3,
                   setup_mean_ms=sum(setups) / len(setups) / 1e3)
    if lats:
        out.update(latency_p50_ms=percentile(lats, 50) / 1e3, latency_p99_ms=percentile(lats, 99) / 1e3)
    return out


# ----------------------------------------------------------------- workload ---
class SequenceSource:
    """Explicit (engine µs, function) arrivals replayed on the wall clock
    (reference OpenLoopSource over a SequenceSpec, workload.py:116-140)."""

    def __init__(self, arrivals):
        self.arrivals = sorted(arrivals, key=lambda a: a[0])
        self._idx = 0
        self._sim = None

    @property
    def exhausted(self) -> bool:
        return self._idx >= len(self.arrivals)

    def attach(self, sim) -> None:
        self._sim = sim
        self._schedule_next()

    def _schedule_next(self) -> None:
        if self._idx >= len(self.arrivals):
            return
        t, _ = self.arrivals[self._idx]
        self._sim.engine.schedule(max(t, self._sim.engine.now), EventKind.ARRIVAL, self._on_arrival, self._idx)

    def _on_arrival(self, idx) -> None:
        t, name = self.arrivals[idx]
        self._idx += 1
        self._schedule_next()
        self._sim.submit(name, arrival_us=t)
