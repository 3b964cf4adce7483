"""Trace replay and peak-throughput search on the real plane (SURVEY.md
§8f-3).

The reference drives its model from flat trace CSVs (`timestamp_ms,function`,
pkg/src/gslsim/workload.py:178-212), from Azure Functions per-minute counts
flattened into that format (:215-253), and searches for the largest stable
offered rate by doubling then bisecting (:256-354).  The same file formats,
error messages and stability rule are kept here; the probes run on the GPU
plane in wall-clock time.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass

from .engine import US_PER_MS, EventKind
from .workload import ArrivalRecord, OpenLoopSource


class TraceParseError(ValueError):
    """A malformed trace / MAF file; the message names the file and line."""


@dataclass(frozen=True)
class TraceSpec:
    path: str
    time_scale: float = 1.0


def _data_rows(reader, first_line: int):
    for line, row in enumerate(reader, start=first_line):
        if row and not (len(row) == 1 and not row[0].strip()):
            yield line, row


def parse_trace(path, known_functions=None) -> list[ArrivalRecord]:
    """Arrivals of a flat trace, ordered by (time, function)."""
    with open(path, "r", encoding="utf-8", newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None:                      # an empty file is an empty trace
            return []
        if [c.strip() for c in header] != ["timestamp_ms", "function"]:
            raise TraceParseError(f"{path}: line 1: expected header 'timestamp_ms,function'")
        recs = []
        for line, row in _data_rows(reader, 2):
            where = f"{path}: line {line}"
            if len(row) != 2:
                raise TraceParseError(f"{where}: expected 2 columns, got {len(row)}")
            try:
                t_ms = float(row[0])
            except ValueError:
                raise TraceParseError(f"{where}: bad timestamp {row[0]!r}") from None
            if t_ms < 0:
                raise TraceParseError(f"{where}: negative timestamp")
            name = row[1].strip()
            if known_functions is not None and name not in known_functions:
                raise TraceParseError(f"{where}: unknown function {name!r}")
            recs.append(ArrivalRecord(int(round(t_ms * US_PER_MS)), name))
    return sorted(recs, key=lambda r: (r.timestamp_us, r.function))


def trace_arrivals(spec: TraceSpec, known_functions=None) -> list[ArrivalRecord]:
    return [ArrivalRecord(int(round(r.timestamp_us * spec.time_scale)), r.function)
            for r in parse_trace(spec.path, known_functions)]


def trace_totals(records) -> dict[str, int]:
    counts: dict[str, int] = {}
    for r in records:
        counts[r.function] = counts.get(r.function, 0) + 1
    return {k: counts[k] for k in sorted(counts)}


def flatten_maf(input_path, output_path) -> int:
    """MAF rows (function id + 1440 per-minute counts) -> flat trace: count k
    in minute m becomes arrivals at m*60000 + i*60000//k ms, i < k."""
    arrivals = []
    with open(input_path, "r", encoding="utf-8", newline="") as fh:
        reader = csv.reader(fh)
        if next(reader, None) is None:
            raise TraceParseError(f"{input_path}: empty input")
        for line, row in _data_rows(reader, 2):
            where = f"{input_path}: line {line}"
            if len(row) != 1 + 1440:
                raise TraceParseError(f"{where}: expected 1441 columns, got {len(row)}")
            fn = row[0].strip()
            for minute, cell in enumerate(row[1:]):
                try:
                    k = int(cell or 0)
                except ValueError:
                    raise TraceParseError(f"{where}: bad count {cell!r} at minute {minute}") from None
                if k < 0:
                    raise TraceParseError(f"{where}: negative count at minute {minute}")
                base = minute * 60_000
                arrivals += [(base + (60_000 * i) // k, fn) for i in range(k)]
    arrivals.sort()
    with open(output_path, "w", encoding="utf-8", newline="") as fh:
        out = csv.writer(fh, lineterminator="\n")
        out.writerow(["timestamp_ms", "function"])
        out.writerows(arrivals)
    return len(arrivals)


# ------------------------------------------------------------- peak search ---
@dataclass
class StabilityStats:
    queue_early: int
    queue_end: int
    p99_first_quartile_ms: float | None
    p99_last_quartile_ms: float | None
    completed_first_quartile: int
    completed_last_quartile: int


def is_stable(s: StabilityStats, p99_growth_limit: float = 2.0, queue_slack: int = 0,
              p99_slack_ms: float = 0.0) -> bool:
    """No backlog growth over the probe, and late arrivals' p99 latency within
    `p99_growth_limit` x that of early arrivals (idle probes are stable; a
    probe that stopped completing is not).  The slacks (0 = the reference's
    rule) absorb the jitter of real hardware: a backlog of in-flight work that
    wanders by a few invocations, millisecond-scale p99s that double by
    chance."""
    grew = s.queue_end > s.queue_early + queue_slack
    idle = s.completed_first_quartile == 0 and s.completed_last_quartile == 0
    if grew or (not idle and s.completed_last_quartile == 0):
        return False
    if idle or not s.p99_first_quartile_ms:
        return True
    return s.p99_last_quartile_ms <= max(p99_growth_limit * s.p99_first_quartile_ms,
                                         s.p99_first_quartile_ms + p99_slack_ms)


@dataclass
class PeakSearchResult:
    rate_per_s: float
    hit_ceiling: bool
    trajectory: list            # (rate, stable) in probe order
    diagnostic: str = ""


def find_peak_throughput(probe, *, rate_min: float = 0.5, rate_ceiling: float = 4096.0, resolution: float = 0.01,
                         p99_growth_limit: float = 2.0, queue_slack: int = 0, p99_slack_ms: float = 0.0
                         ) -> PeakSearchResult:
    """Largest stable rate: probe rate_min, double until a probe is unstable
    (or the ceiling is stable), then bisect the bracket to `resolution`."""
    res = PeakSearchResult(0.0, False, [])

    def stable(rate: float) -> bool:
        verdict = is_stable(probe(rate), p99_growth_limit, queue_slack, p99_slack_ms)
        res.trajectory.append((rate, verdict))
        return verdict

    if not stable(rate_min):
        res.diagnostic = f"no stable rate at minimum probe {rate_min}/s"
        return res
    good, bad = rate_min, None
    while bad is None:
        nxt = min(2 * good, rate_ceiling)
        if not stable(nxt):
            bad = nxt
        elif nxt >= rate_ceiling:
            res.rate_per_s, res.hit_ceiling = rate_ceiling, True
            res.diagnostic = "stable at the configured rate ceiling"
            return res
        else:
            good = nxt
    while bad - good > resolution * good:
        mid = 0.5 * (good + bad)
        good, bad = (mid, bad) if stable(mid) else (good, mid)
    res.rate_per_s = good
    return res


class BacklogSampler:
    """Backlog (admitted or queued, not completed) of a running Simulation,
    sampled on its engine every `period_us` (the reference samples its
    admission queue, simulation.py:214-220)."""

    def __init__(self, sim, period_us: int = 100_000):
        self.sim, self.period = sim, period_us
        self.samples: dict[int, int] = {}
        self._stopped = False

    def start(self) -> "BacklogSampler":
        self._tick(None)
        return self

    def backlog(self) -> int:
        return self.sim.in_flight + self.sim.policy.queued_count()

    def _tick(self, _payload) -> None:
        if self._stopped:
            return
        now = self.sim.engine.now
        self.samples[now] = self.backlog()
        self.sim.engine.schedule(now + self.period, EventKind.MEASUREMENT_TICK, self._tick, None)

    def stop(self) -> None:
        self._stopped = True


def probe_stats(invocations, t0_us: int, duration_us: int, queue_early: int, queue_end: int) -> StabilityStats:
    """Stability signals of a finished probe: p99 latency of the first and
    last arrival quartiles of [t0, t0 + duration) and the backlog early / at
    the end of the arrival window."""
    from .runtime import percentile
    q1, q4 = t0_us + duration_us // 4, t0_us + duration_us - duration_us // 4
    early = [i.latency_us / US_PER_MS for i in invocations if i.arrival_us <= q1 and i.outcome == "completed"]
    late = [i.latency_us / US_PER_MS for i in invocations if i.arrival_us >= q4 and i.outcome == "completed"]
    return StabilityStats(queue_early, queue_end, percentile(early, 99) if early else None,
                          percentile(late, 99) if late else None, len(early), len(late))


def run_probe(sim, arrivals, duration_us: int) -> StabilityStats:
    """Replay `arrivals` (one probe) on a live Simulation and judge it.

    Backlog signal: the reference compares its admission queue early and at
    the end (SAGE admits at once, so on the real plane overload shows as
    in-flight work piling up on the device instead).  Here queue_early is the
    LARGEST backlog sampled in the first half of the window and queue_end the
    backlog when arrivals stop: under overload the backlog grows past
    anything seen early; under a sustainable rate it fluctuates below it."""
    src = OpenLoopSource(arrivals)
    t0 = sim.engine.tick()
    sampler = BacklogSampler(sim).start()
    first = len(sim.invocations)
    src.attach(sim)
    sim.source = src
    sim.run(until=t0 + duration_us)
    queue_end = sampler.backlog()
    sampler.stop()
    sim.drain()
    early = [b for t, b in sampler.samples.items() if t0 <= t <= t0 + duration_us // 2]
    queue_early = max(early) if early else 0
    return probe_stats(sim.invocations[first:], t0, duration_us, queue_early, queue_end)
