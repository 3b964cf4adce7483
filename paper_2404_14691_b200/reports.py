"""Run reports in the reference's artifact schema.

The reference writes `summary.json`, `invocations.csv` and
`memory_timeline.csv` for every run (pkg/src/gslsim/metrics.py:90-233,
experiments.py:50-55).  The same file names, columns, keys and number
formats are produced here for runs of the real plane, so a reference user's
tooling reads them unchanged:

  invocations.csv      one row per invocation, reference columns; the
                       host / PCIe byte columns are the PLANNED bytes in
                       reference MB (umb / 10^6), the stage columns measured
                       device times (engine ms)
  memory_timeline.csv  per-GPU ledger usage by allocation class at every
                       ledger change (MB := MiB on the real plane)
  summary.json         the reference's summary keys + `extensions` (setup
                       p50/p99, measured bytes) that the reference lacks
"""
from __future__ import annotations

import csv
import json

from .engine import US_PER_MS, US_PER_S
from .functions import STAGE_ORDER
from .resources import AllocClass
from .runtime import OUTCOME_COMPLETED, OUTCOME_FAILED, OUTCOME_PENDING, percentile

MIB = 1 << 20
UMB_PER_MB = 1_000_000

INVOCATION_COLUMNS = (["id", "function", "gpu", "arrival_ms", "start_ms", "completion_ms", "end_to_end_ms",
                       "queued_ms", "warmth", "outcome", "host_bytes_mb", "pcie_bytes_mb"]
                      + [f"{st.value}_{edge}_ms" for st in STAGE_ORDER for edge in ("begin", "end")])
TIMELINE_COLUMNS = ["t_ms", "gpu", "context_mb", "read_only_mb", "writable_mb", "instance_mb", "total_mb"]
_CLASSES = (AllocClass.CONTEXT, AllocClass.READ_ONLY, AllocClass.WRITABLE, AllocClass.INSTANCE_FIXED)


def _ms(us) -> str:
    return "" if us is None else f"{us / US_PER_MS:.3f}"


def _mb(umb: int) -> str:
    return f"{umb / UMB_PER_MB:.6f}"


def write_invocations_csv(path, invocations) -> None:
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(INVOCATION_COLUMNS)
        for inv in sorted(invocations, key=lambda i: i.id):
            done = inv.outcome == OUTCOME_COMPLETED
            row = [inv.id, inv.spec.name, "" if inv.gpu is None else inv.gpu, _ms(inv.arrival_us), _ms(inv.start_us),
                   _ms(inv.completion_us), _ms(inv.latency_us if done else None),
                   _ms(inv.queued_us if inv.start_us is not None else None),
                   "" if inv.warmth is None else inv.warmth.label(), inv.outcome,
                   _mb(inv.host_bytes_umb), _mb(inv.pcie_bytes_umb)]
            for st in STAGE_ORDER:
                span = inv.stages.get(st)
                row += [_ms(span[0] if span else None), _ms(span[1] if span and span[1] is not None else None)]
            w.writerow(row)


class MemoryTimeline:
    """Ledger usage of one GPU by class, one entry per change (entries at the
    same instant collapse to the last state), with the exact time integral
    and peak of the total for summary.json's gpu_memory."""

    def __init__(self, gpu: int, ledger, clock):
        self.gpu, self.ledger, self.clock = gpu, ledger, clock
        self.entries: list[tuple] = []
        self._area = 0          # byte-µs
        self._t_last = None
        self._u_last = 0
        self._peak = 0
        self._t_first = None
        ledger.on_change = self.record
        self.record()

    def record(self) -> None:
        t = self.clock()
        by = self.ledger.usage_by_class()
        entry = (t,) + tuple(by[c] for c in _CLASSES)
        total = sum(entry[1:])
        if self._t_last is not None:
            self._area += self._u_last * (t - self._t_last)
        else:
            self._t_first = t
        self._t_last, self._u_last = t, total
        self._peak = max(self._peak, total)
        if self.entries and self.entries[-1][0] == t:
            self.entries[-1] = entry
        else:
            self.entries.append(entry)

    def close(self) -> None:
        self.record()
        if self.ledger.on_change == self.record:
            self.ledger.on_change = None

    def average_bytes(self, t_end=None) -> float:
        t_end = self.clock() if t_end is None else t_end
        if self._t_first is None or t_end <= self._t_first:
            return float(self._u_last)
        area = self._area + self._u_last * (t_end - self._t_last)
        return area / (t_end - self._t_first)

    def peak_bytes(self) -> int:
        return self._peak


def write_timeline_csv(path, timelines) -> None:
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(TIMELINE_COLUMNS)
        for tl in timelines:
            for t, *parts in tl.entries:
                w.writerow([f"{t / US_PER_MS:.3f}", tl.gpu] + [f"{p / MIB:.6f}" for p in parts]
                           + [f"{sum(parts) / MIB:.6f}"])


def summarize(invocations, duration_us: int, spec_table, timelines=()) -> dict:
    """The reference RunSummary (metrics.py:124-181) for a real-plane run:
    throughput over the run period, per-function latency stats, Eq. 1
    theoretical throughput and normalised performance, GPU memory average /
    peak; `channel_utilization` stays empty (the hardware has no modelled
    channels -- measured bytes are under extensions)."""
    period_ms = duration_us / US_PER_MS
    done = [i for i in invocations if i.outcome == OUTCOME_COMPLETED]
    by_fn: dict[str, list] = {}
    for i in done:
        by_fn.setdefault(i.spec.name, []).append(i.latency_us)
    per_fn = {name: {"count": len(l), "mean_ms": sum(l) / len(l) / US_PER_MS, "p50_ms": percentile(l, 50) / US_PER_MS,
                     "p99_ms": percentile(l, 99) / US_PER_MS, "max_ms": max(l) / US_PER_MS}
              for name, l in sorted(by_fn.items())}
    theo = {name: period_ms / spec.compute_ms for name, spec in sorted(spec_table.items())}
    norm = {name: (len(by_fn.get(name, ())) / t if t > 0 else 0.0) for name, t in theo.items()}
    lats = [i.latency_us for i in done]
    setups = [i.setup_us for i in done if i.setup_us is not None]
    measured = {k: sum(i.measured.get(k, 0) for i in done) for k in ("host_bytes", "pcie_bytes", "nvlink_bytes")}
    # the reference's summary.json layout (RunSummary.to_dict, metrics.py:104-116)
    return {
        "duration_ms": period_ms,
        "counts": {"arrivals": len(invocations), "completed": len(done),
                   "failed": sum(i.outcome == OUTCOME_FAILED for i in invocations),
                   "pending": sum(i.outcome == OUTCOME_PENDING for i in invocations)},
        "throughput_per_s": len(done) / (duration_us / US_PER_S) if duration_us else 0.0,
        "latency_ms": {"mean": sum(lats) / len(lats) / US_PER_MS if lats else None,
                       "p99": percentile(lats, 99) / US_PER_MS if lats else None},
        "per_function": per_fn,
        "theoretical_throughput": theo,
        "normalized_performance": norm,
        "channel_utilization": {},
        "gpu_memory_mb": {f"gpu{tl.gpu}": {"avg_mb": tl.average_bytes() / MIB, "peak_mb": tl.peak_bytes() / MIB}
                          for tl in timelines},
        "extensions": {
            "setup_p50_ms": percentile(setups, 50) / US_PER_MS if setups else None,
            "setup_p99_ms": percentile(setups, 99) / US_PER_MS if setups else None,
            "measured_bytes": measured,
        },
    }


def write_summary_json(path, summary: dict) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(summary, indent=2, sort_keys=True) + "\n")


def write_artifacts(out_dir, sim, duration_us: int, timelines=()) -> dict:
    """summary.json + invocations.csv (+ memory_timeline.csv) into out_dir."""
    from pathlib import Path
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    summary = summarize(sim.invocations, duration_us, sim.spec_table, timelines)
    write_summary_json(out / "summary.json", summary)
    write_invocations_csv(out / "invocations.csv", sim.invocations)
    if timelines:
        write_timeline_csv(out / "memory_timeline.csv", timelines)
    return summary
