"""GPU memory ledgers over the VMM segment pool.

Drop-in for gslsim.resources.MemoryLedger / Denied / AllocClass
(pkg/src/gslsim/resources.py:237-337): capacity-checked allocation with the
reference's rounding (round_up_umb, :36-40: 1024 MB for FixedGSL, exact
otherwise), a `Denied` VALUE carrying the shortfall (:244-257, :309-315) and
SimulationError on a double or unknown free (:324-326).

Differences on the real plane:
  * sizes are bytes (1 MB := 1 MiB), not µMB;
  * every READ_ONLY / CONTEXT / WRITABLE allocation is a real cuMemCreate
    segment of the native pool (its device pointer is `Allocation.dptr`);
    INSTANCE_FIXED (FixedGSL) is charged here but mapped by the instance's
    own fresh context (account-only);
  * the ledger counts are mirrored in C (sage_pool_usage) and must agree.

The Channel model (resources.py:82-234) has no counterpart: contention on
the host path and on PCIe is real hardware behaviour now.
"""
from __future__ import annotations

import itertools
from enum import Enum
from typing import Callable, Optional


class SimulationError(RuntimeError):
    """A broken invariant (always a logic bug) -- reference engine.py:25-26."""


class AllocClass(Enum):
    CONTEXT = 0
    READ_ONLY = 1
    WRITABLE = 2
    INSTANCE_FIXED = 3

    __hash__ = object.__hash__   # members are singletons: identity hash (hot dict keys)


def round_up(size: int, granularity: int) -> int:
    """Least multiple of the granularity >= size (0 = exact)."""
    if granularity <= 0:
        return size
    return -((-size) // granularity) * granularity


class Denied:
    """Allocation refusal carrying the shortfall; a value, not an error."""

    __slots__ = ("shortfall",)

    def __init__(self, shortfall: int):
        self.shortfall = shortfall

    @property
    def shortfall_mb(self) -> float:
        return self.shortfall / (1 << 20)

    def __repr__(self):
        return f"Denied(shortfall={self.shortfall_mb:.3f} MiB)"


class Allocation:
    __slots__ = ("id", "requested", "effective", "cls", "owner", "segment")

    def __init__(self, aid, requested, effective, cls, owner, segment=None):
        self.id = aid
        self.requested = requested
        self.effective = effective
        self.cls = cls
        self.owner = owner
        self.segment = segment

    @property
    def dptr(self) -> int:
        return self.segment.dptr if self.segment is not None else 0


class DevicePool:
    """Backend: the native VMM pool of one GPU (libsagedp)."""

    def __init__(self, gpu: int):
        from . import device
        self._d = device
        self.gpu = gpu

    def configure(self, capacity: int, granularity: int) -> None:
        self._d.pool_configure(self.gpu, capacity, granularity)

    def alloc(self, nbytes: int, cls: AllocClass, account_only: bool):
        try:
            return self._d.pool_alloc(self.gpu, nbytes, cls.value, account_only=account_only)
        except self._d.DeniedAlloc as exc:
            raise MemoryError(exc.shortfall) from exc

    def free(self, seg, after=None) -> None:
        """`after`: a device Event or a list of them (the pages outlive the
        ledger entry until every one completed)."""
        evs = [e.h for e in (after if isinstance(after, (list, tuple)) else [after]) if e is not None and e.h]
        if evs:
            from . import _lib
            _lib.check(_lib.lib().sage_pool_free_after_n(seg.h, (_lib.H * len(evs))(*evs), len(evs)),
                       "sage_pool_free_after_n")
            seg.h = 0
        else:
            seg.free()

    def usage(self) -> dict:
        return self._d.pool_usage(self.gpu)


class MemoryLedger:
    """Capacity-checked allocation table for one GPU (or the host side).

    capacity=None means unlimited (the host RO cache ledger).  Requested sizes
    are rounded up to `granularity`; usage is in effective bytes.
    """

    def __init__(self, name: str, capacity: Optional[int] = None, granularity: int = 0,
                 backend=None, on_change: Optional[Callable[[], None]] = None):
        self.name = name
        self.capacity = capacity
        self.granularity = granularity
        self.backend = backend
        self.on_change = on_change
        self._allocs: dict[int, Allocation] = {}
        self._ids = itertools.count()
        self._usage = 0
        self._by_class = {c: 0 for c in AllocClass}
        if backend is not None and capacity is not None:
            backend.configure(capacity, granularity)

    @property
    def usage(self) -> int:
        return self._usage

    @property
    def free_bytes(self) -> Optional[int]:
        return None if self.capacity is None else self.capacity - self._usage

    def effective(self, size: int) -> int:
        return round_up(size, self.granularity)

    def fits(self, size: int) -> bool:
        if self.capacity is None:
            return True
        return self.effective(size) <= self.capacity - self._usage

    def try_alloc(self, size: int, cls: AllocClass, owner=None, account_only: bool = False):
        """Allocate (and map) or return Denied carrying the shortfall."""
        if size <= 0:
            raise SimulationError(f"ledger {self.name}: allocation size must be > 0")
        eff = self.effective(size)
        if self.capacity is not None and eff > self.capacity - self._usage:
            return Denied(eff - (self.capacity - self._usage))
        seg = None
        if self.backend is not None:
            try:
                seg = self.backend.alloc(size, cls, account_only or cls is AllocClass.INSTANCE_FIXED)
            except MemoryError as exc:  # the native pool disagrees: physical exhaustion
                return Denied(int(exc.args[0]) if exc.args else eff)
        alloc = Allocation(next(self._ids), size, eff, cls, owner, seg)
        self._allocs[alloc.id] = alloc
        self._usage += eff
        self._by_class[cls] += eff
        if self.on_change:
            self.on_change()
        return alloc

    def free(self, alloc: Allocation, after=None) -> None:
        """Release now; with `after` (a device Event, or a list) the physical
        pages are returned only once it completes (a D2H or a peer land may
        still read them)."""
        if self._allocs.get(alloc.id) is not alloc:
            raise SimulationError(f"ledger {self.name}: double or unknown free (id={alloc.id})")
        del self._allocs[alloc.id]
        self._usage -= alloc.effective
        self._by_class[alloc.cls] -= alloc.effective
        if self.backend is not None and alloc.segment is not None:
            self.backend.free(alloc.segment, after)
        if self.on_change:
            self.on_change()

    def usage_by_class(self) -> dict[AllocClass, int]:
        return dict(self._by_class)

    def allocations(self) -> list[Allocation]:
        return list(self._allocs.values())

    def check_native(self) -> None:
        """The C pool's ledger must equal this mirror exactly."""
        if self.backend is None:
            return
        u = self.backend.usage()
        want = [self._by_class[c] for c in AllocClass]
        if u["ledger"] != self._usage or u["by_class"] != want:
            raise SimulationError(f"ledger {self.name}: native {u} != python {self._usage} {want}")
