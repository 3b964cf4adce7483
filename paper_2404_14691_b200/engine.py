"""Wall-clock event loop of the real plane.

Keeps the timer / callback API of gslsim.engine.Engine
(pkg/src/gslsim/engine.py:74-155: `now`, `schedule`, `cancel`, `step`,
`run(until)`, `pending`, `event_log`) and the named PCG64 streams
(`rng_stream`, :46-52) so placements replay exactly as in the reference.
What changes: time is the library clock (µs since sage_init, the same clock
device event times are converted onto), and besides timers the loop polls
device completions (`watch`) -- completions are polled, never called back
from CUDA threads (include/sage_dp.h conventions).
"""
from __future__ import annotations

import heapq
import time
from enum import Enum
from typing import Any, Callable, Optional

from numpy.random import Generator, PCG64, SeedSequence

from .resources import SimulationError

US_PER_MS = 1_000
US_PER_S = 1_000_000
WORKLOAD_STREAM = 0
DISPATCH_STREAM = 1


class EventKind(Enum):
    ARRIVAL = "Arrival"
    TRANSFER_COMPLETE = "TransferComplete"
    STAGE_COMPLETE = "StageComplete"
    EXIT_TIMER = "ExitTimer"
    GENERATOR_TICK = "GeneratorTick"
    MEASUREMENT_TICK = "MeasurementTick"
    DEVICE_COMPLETE = "DeviceComplete"

    __hash__ = object.__hash__   # members are singletons: identity hash (hot dict keys)


def ms_to_us(ms: float) -> int:
    return int(round(ms * US_PER_MS))


def s_to_us(s: float) -> int:
    return int(round(s * US_PER_S))


def rng_stream(seed: int, stream_id: int) -> Generator:
    """Same (seed, stream) -> same draws as the reference (engine.py:46-52)."""
    return Generator(PCG64(SeedSequence(entropy=seed, spawn_key=(stream_id,))))


class Event:
    __slots__ = ("time", "seq", "kind", "payload", "callback", "cancelled", "dispatched", "engine")

    def __init__(self, time_us, seq, kind, callback, payload, engine):
        self.time = time_us
        self.seq = seq
        self.kind = kind
        self.payload = payload
        self.callback = callback
        self.cancelled = False
        self.dispatched = False
        self.engine = engine

    def __repr__(self):
        return f"Event(t={self.time}, seq={self.seq}, kind={self.kind.value})"


class _Watch:
    __slots__ = ("ev", "cb", "payload")

    def __init__(self, ev, cb, payload):
        self.ev, self.cb, self.payload = ev, cb, payload


class Engine:
    """Single-threaded loop: timers in (time, seq) order + polled device events.

    `clock` returns µs; by default the native library clock, so event times
    read back from the device are on the same axis.
    """

    def __init__(self, log_events: bool = False, clock: Optional[Callable[[], int]] = None,
                 poll: Optional[Callable] = None):
        if clock is None:
            from . import device
            clock = device.now_us
            poll = poll or device.poll
        self._clock = clock
        self._poll = poll
        self._t0 = clock()
        self._now = 0
        self._seq = 0
        self._heap: list = []
        self._live = 0
        self._watches: list[_Watch] = []
        self._sources: list = []   # completion sources: .outstanding() / .poll(timeout_us)
        self._log = [] if log_events else None

    # time ---------------------------------------------------------------------
    def wall_us(self) -> int:
        return self._clock() - self._t0

    @property
    def now(self) -> int:
        return self._now

    def tick(self) -> int:
        """Advance `now` to the wall clock (monotone)."""
        w = self.wall_us()
        if w > self._now:
            self._now = w
        return self._now

    def to_engine_time(self, lib_us: int) -> int:
        """Library-clock µs (device event times) -> engine time."""
        return lib_us - self._t0

    # timers ---------------------------------------------------------------------
    def schedule(self, time_us: int, kind: EventKind, callback: Callable[[Any], None], payload: Any = None) -> Event:
        if time_us < self._now:
            raise SimulationError(f"schedule into the past: t={time_us} < now={self._now} ({kind.value})")
        ev = Event(time_us, self._seq, kind, callback, payload, self)
        self._seq += 1
        heapq.heappush(self._heap, (ev.time, ev.seq, ev))
        self._live += 1
        return ev

    def cancel(self, handle: Event) -> bool:
        if not isinstance(handle, Event) or handle.engine is not self:
            raise SimulationError(f"cancel of unknown event handle: {handle!r}")
        if handle.dispatched or handle.cancelled:
            return False
        handle.cancelled = True
        self._live -= 1
        return True

    # device completions ---------------------------------------------------------
    def watch(self, device_event, callback: Callable[[Any], None], payload: Any = None) -> None:
        """Call callback(payload) from the loop once device_event completes."""
        self._watches.append(_Watch(device_event, callback, payload))

    def add_source(self, source) -> None:
        """A completion source the loop drains besides watched events: an
        object with outstanding() -> int and poll(timeout_us) -> callbacks run
        (the data plane's native completion queue)."""
        self._sources.append(source)

    def _outstanding(self) -> int:
        return sum(s.outstanding() for s in self._sources)

    def _poll_sources(self, timeout_us: int) -> int:
        n = 0
        for s in self._sources:
            if s.outstanding():
                n += s.poll(timeout_us)
                timeout_us = 0
        return n

    def watching(self) -> int:
        return len(self._watches) + self._outstanding()

    def _poll_watches(self, timeout_us: int) -> int:
        if not self._watches:
            return 0
        done = self._poll([w.ev for w in self._watches], timeout_us)
        fired = [w for w, d in zip(self._watches, done) if d]
        if not fired:
            return 0
        self._watches = [w for w, d in zip(self._watches, done) if not d]
        self.tick()
        for w in fired:
            if self._log is not None:
                self._log.append(f"{self._now} - {EventKind.DEVICE_COMPLETE.value}")
            w.cb(w.payload)
        return len(fired)

    # loop -------------------------------------------------------------------------
    def _pop_due(self) -> Optional[Event]:
        while self._heap:
            t, _, ev = self._heap[0]
            if ev.cancelled:
                heapq.heappop(self._heap)
                continue
            if t <= self._now:
                heapq.heappop(self._heap)
                return ev
            return None
        return None

    def _dispatch(self, ev: Event) -> None:
        ev.dispatched = True
        self._live -= 1
        if self._log is not None:
            self._log.append(f"{ev.time} {ev.seq} {ev.kind.value}")
        ev.callback(ev.payload)

    def _next_timer(self) -> Optional[int]:
        while self._heap and self._heap[0][2].cancelled:
            heapq.heappop(self._heap)
        return self._heap[0][0] if self._heap else None

    def step(self) -> int:
        """Dispatch everything due now plus completed device work; returns count.

        A timer runs with `now` = its scheduled instant (as in the reference),
        so chained timers (the four decay stages) never accumulate lateness."""
        wall = max(self.wall_us(), self._now)
        n = 0
        while self._heap:
            t, _, ev = self._heap[0]
            if ev.cancelled:
                heapq.heappop(self._heap)
                continue
            if t > wall:
                break
            heapq.heappop(self._heap)
            self._now = max(self._now, t)
            self._dispatch(ev)
            n += 1
        self._now = max(self._now, wall)
        n += self._poll_watches(0)
        if self._sources:
            n += self._poll_sources(0)
        return n

    def run(self, until: Optional[int] = None, idle: Optional[Callable[[], bool]] = None) -> int:
        """Run until engine time `until` (wall clock), or -- with until=None --
        until no timer and no device watch is pending.  `idle()` returning
        True also ends the loop (used to stop once all invocations drained
        while far-future decay timers stay armed)."""
        dispatched = 0
        while True:
            dispatched += self.step()
            if idle is not None and idle():
                break
            nt = self._next_timer()
            if until is not None and self._now >= until:
                break
            outstanding = self._outstanding() if self._sources else 0
            if nt is None and not self._watches and not outstanding:
                if until is None:
                    break
                time.sleep(max(0, until - self.wall_us()) / 1e6)
                self.tick()
                continue
            horizon = nt if nt is not None else (until if until is not None else self._now + 1000)
            if until is not None:
                horizon = min(horizon, until)
            wait = max(0, horizon - self.wall_us())
            if self._watches:
                dispatched += self._poll_watches(0 if outstanding else min(wait, 200))
            if outstanding:
                # blocks in the library (GIL released) until a completion
                dispatched += self._poll_sources(min(wait, 50 if self._watches else 200))
            elif not self._watches and wait > 0:
                time.sleep(min(wait, 2000) / 1e6)
        return dispatched

    def pending(self) -> int:
        return self._live + len(self._watches) + self._outstanding()

    @property
    def event_log(self) -> list[str]:
        if self._log is None:
            raise SimulationError("event log not enabled for this engine")
        return self._log
