"""Arrival streams for the real plane.

`generate_arrivals` restates the reference's open-loop generator
(pkg/src/gslsim/workload.py:75-113): the same PCG64 stream
(rng_stream(seed, WORKLOAD_STREAM), engine.py:46-52), the same block-wise
exponential gaps + weighted choice over the sorted mix, the same rounding to
integer microseconds -- so a stream drives the reference model and the B200
plane identically (as `compare_policies` does, experiments.py:86-93).
`OpenLoopSource` replays a stream on the wall clock (reference:
workload.py:116-140), optionally time-scaled.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .engine import US_PER_MS, US_PER_S, WORKLOAD_STREAM, EventKind, rng_stream


@dataclass(frozen=True)
class ArrivalRecord:
    timestamp_us: int
    function: str

    @property
    def timestamp_ms(self) -> float:
        return self.timestamp_us / US_PER_MS


@dataclass(frozen=True)
class PoissonOpenSpec:
    rate_per_s: float
    duration_s: float
    mix: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.rate_per_s < 0 or self.duration_s <= 0:
            raise ValueError("Poisson source needs rate >= 0 and duration > 0")


@dataclass(frozen=True)
class SequenceSpec:
    arrivals: tuple


def _normalize_mix(mix: dict) -> list:
    if not mix:
        raise ValueError("function mix must not be empty")
    total = sum(mix.values())
    if total <= 0 or any(w <= 0 for w in mix.values()):
        raise ValueError("function mix weights must be positive")
    return [(name, w / total) for name, w in sorted(mix.items())]


def generate_arrivals(spec, seed: int) -> list[ArrivalRecord]:
    if isinstance(spec, PoissonOpenSpec):
        rng = rng_stream(seed, WORKLOAD_STREAM)
        mix = _normalize_mix(spec.mix)
        names = [n for n, _ in mix]
        weights = [w for _, w in mix]
        if spec.rate_per_s == 0:
            return []
        out, t = [], 0.0
        end = spec.duration_s * US_PER_S
        mean_us = US_PER_S / spec.rate_per_s
        done = False
        while not done:
            gaps = rng.exponential(mean_us, size=1024)
            picks = rng.choice(len(names), size=1024, p=weights)
            for gap, pick in zip(gaps, picks):
                t += gap
                if t >= end:
                    done = True
                    break
                out.append(ArrivalRecord(int(round(t)), names[pick]))
        return out
    if isinstance(spec, SequenceSpec):
        return [ArrivalRecord(int(round(ms * US_PER_MS)), name) for ms, name in spec.arrivals]
    raise TypeError(f"not an open-loop source spec: {spec!r}")


class OpenLoopSource:
    """Replays a pre-generated stream on the engine's wall clock, starting at
    attach time; `time_scale` < 1 compresses it (e.g. tests)."""

    def __init__(self, arrivals: list, time_scale: float = 1.0):
        self.arrivals = list(arrivals)
        self.functions = sorted({a.function for a in self.arrivals})
        self.time_scale = time_scale
        self._idx = 0
        self._sim = None
        self._t0 = 0

    @property
    def exhausted(self) -> bool:
        return self._idx >= len(self.arrivals)

    def attach(self, sim) -> None:
        self._sim = sim
        self._t0 = sim.engine.tick()
        self._schedule_next()

    def _at(self, i: int) -> int:
        return self._t0 + int(round(self.arrivals[i].timestamp_us * self.time_scale))

    def _schedule_next(self) -> None:
        if self._idx >= len(self.arrivals):
            return
        self._sim.engine.schedule(max(self._at(self._idx), self._sim.engine.now), EventKind.ARRIVAL,
                                  self._on_arrival, self._idx)

    def _on_arrival(self, i: int) -> None:
        self._idx += 1
        self._schedule_next()
        self._sim.submit(self.arrivals[i].function, arrival_us=self._at(i))

