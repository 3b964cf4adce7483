"""Run reports in the reference's artifact schema and the trace / MAF / peak
search drivers, on CPU.

Schema and the cfg-1 burst's invocations.csv rows come from the reference
itself (tests/golden/report_schema.json, tests/golden/make_report_golden.py);
the trace, MAF and peak-search cases restate the reference's own tests
(pkg/tests/test_workload.py:48-154)."""
import csv
import json
from pathlib import Path

import pytest

from paper_2404_14691_b200 import reports as R
from paper_2404_14691_b200.functions import load_spec_table
from paper_2404_14691_b200.replay import (StabilityStats, TraceParseError, TraceSpec, find_peak_throughput,
                                          flatten_maf, is_stable, parse_trace, trace_arrivals, trace_totals)
from paper_2404_14691_b200.resources import AllocClass, MemoryLedger

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "report_schema.json").read_text())


def test_artifact_schema_is_the_references():
    assert list(R.INVOCATION_COLUMNS) == GOLD["invocation_columns"]
    assert R.TIMELINE_COLUMNS == GOLD["timeline_columns"]


def test_burst16_invocations_csv_matches_reference(tmp_path):
    from test_host_logic import FakeSim
    table = load_spec_table({"fn100": {"ro_mem_mb": 100, "writable_mem_mb": 10, "compute_ms": 1,
                                       "input_bytes_host_mb": 1, "input_bytes_pcie_mb": 1}})
    sim = FakeSim("SAGE", table)
    for _ in range(16):
        sim.submit("fn100")
    for inv in sim.running:
        inv.completion_us = sim.engine.now
    sim.complete_all()
    path = tmp_path / "invocations.csv"
    R.write_invocations_csv(path, sim.invocations)
    rows = list(csv.reader(path.open()))
    assert rows[0] == GOLD["invocation_columns"]
    keep = [rows[0].index(c) for c in GOLD["burst16_SAGE"]["columns"]]
    assert [[r[i] for i in keep] for r in rows[1:]] == GOLD["burst16_SAGE"]["rows"]
    summary = R.summarize(sim.invocations, 30_000_000, table)
    assert set(GOLD["summary_keys"]) <= set(summary)
    assert summary["counts"] == {"arrivals": 16, "completed": 16, "failed": 0, "pending": 0}
    assert sorted(summary["per_function"]["fn100"]) == GOLD["per_function_keys"]


def test_memory_timeline_integral_and_peak(tmp_path):
    t = [0]
    led = MemoryLedger("gpu0", 1 << 30)
    tl = R.MemoryTimeline(0, led, clock=lambda: t[0])
    t[0] = 1_000
    a = led.try_alloc(100 << 20, AllocClass.READ_ONLY)
    t[0] = 3_000
    b = led.try_alloc(50 << 20, AllocClass.WRITABLE)
    t[0] = 4_000
    led.free(a)
    t[0] = 5_000
    led.free(b)
    # usage: 0 for 1 ms, 100 MiB for 2 ms, 150 MiB for 1 ms, 50 MiB for 1 ms
    assert tl.peak_bytes() == 150 << 20
    assert tl.average_bytes(5_000) == pytest.approx(((100 << 20) * 2 + (150 << 20) + (50 << 20)) / 5)
    R.write_timeline_csv(tmp_path / "tl.csv", [tl])
    rows = list(csv.reader((tmp_path / "tl.csv").open()))
    assert rows[0] == GOLD["timeline_columns"]
    assert [r[0] for r in rows[1:]] == ["0.000", "1.000", "3.000", "4.000", "5.000"]
    assert rows[3][2:] == ["0.000000", "100.000000", "50.000000", "0.000000", "150.000000"]
    tl.close()
    assert led.on_change is None


# ---- traces (reference tests/test_workload.py:48-114) ------------------------
def test_trace_sorted_counted_scaled(tmp_path):
    p = tmp_path / "t.csv"
    p.write_text("timestamp_ms,function\n50,b\n10,a\n30,a\n", encoding="utf-8")
    recs = parse_trace(str(p))
    assert [r.timestamp_us for r in recs] == [10_000, 30_000, 50_000]
    assert trace_totals(recs) == {"a": 2, "b": 1}
    p.write_text("timestamp_ms,function\n7200000,a\n", encoding="utf-8")
    assert trace_arrivals(TraceSpec(str(p), time_scale=0.01))[0].timestamp_us == 72_000_000


def test_trace_empty_and_header_only(tmp_path):
    (tmp_path / "e.csv").write_text("", encoding="utf-8")
    (tmp_path / "h.csv").write_text("timestamp_ms,function\n", encoding="utf-8")
    assert parse_trace(str(tmp_path / "e.csv")) == [] == parse_trace(str(tmp_path / "h.csv"))


def test_trace_errors_name_the_row(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("timestamp_ms,function\n5,a\n-3,b\n", encoding="utf-8")
    with pytest.raises(TraceParseError, match="line 3"):
        parse_trace(str(p))
    p.write_text("timestamp_ms,function\n5,ghost\n", encoding="utf-8")
    with pytest.raises(TraceParseError, match="ghost"):
        parse_trace(str(p), known_functions={"a"})
    p.write_text("time,fn\n5,a\n", encoding="utf-8")
    with pytest.raises(TraceParseError, match="line 1"):
        parse_trace(str(p))


def _maf(tmp_path, body):
    src = tmp_path / "maf.csv"
    src.write_text(",".join(["HashFunction"] + [str(i) for i in range(1, 1441)]) + "\n" + body, encoding="utf-8")
    return src


def test_flatten_maf_spreads_minute_counts(tmp_path):
    src = _maf(tmp_path, ",".join(["fn1", "3", "0", "2"] + ["0"] * 1437) + "\n")
    out = tmp_path / "flat.csv"
    assert flatten_maf(str(src), str(out)) == 5
    assert out.read_text().splitlines() == ["timestamp_ms,function", "0,fn1", "20000,fn1", "40000,fn1",
                                            "120000,fn1", "150000,fn1"]


def test_flatten_maf_empty_and_malformed(tmp_path):
    src = _maf(tmp_path, ",".join(["fn1"] + ["0"] * 1440) + "\n")
    out = tmp_path / "o.csv"
    assert flatten_maf(str(src), str(out)) == 0
    assert out.read_text().splitlines() == ["timestamp_ms,function"]
    bad = tmp_path / "bad.csv"
    bad.write_text("h\nfn1,1,2,3\n", encoding="utf-8")
    with pytest.raises(TraceParseError, match="line 2"):
        flatten_maf(str(bad), str(out))


# ---- peak search (reference tests/test_workload.py:120-154) -------------------
def _stats(queue_early=0, queue_end=0, p99_first=10.0, p99_last=10.0, done_first=100, done_last=100):
    return StabilityStats(queue_early, queue_end, p99_first, p99_last, done_first, done_last)


def test_stability_rule():
    assert is_stable(_stats())
    assert not is_stable(_stats(queue_end=5))
    assert not is_stable(_stats(p99_last=25.0))
    assert is_stable(_stats(p99_last=19.9))
    assert not is_stable(_stats(done_last=0, p99_last=None))
    assert is_stable(_stats(done_first=0, done_last=0, p99_first=None, p99_last=None))


@pytest.mark.parametrize("true_peak", [37.0, 0.9, 1000.0])
def test_peak_search_converges(true_peak):
    res = find_peak_throughput(lambda r: _stats() if r <= true_peak else _stats(queue_end=100), rate_min=0.5)
    assert not res.hit_ceiling and res.rate_per_s <= true_peak
    assert (true_peak - res.rate_per_s) / true_peak < 0.02
    assert all(ok == (r <= true_peak) for r, ok in res.trajectory)


def test_peak_search_floor_and_ceiling():
    res = find_peak_throughput(lambda r: _stats(queue_end=10), rate_min=0.5)
    assert res.rate_per_s == 0.0 and "minimum probe" in res.diagnostic
    res = find_peak_throughput(lambda r: _stats(), rate_min=1, rate_ceiling=64)
    assert res.hit_ceiling and res.rate_per_s == 64


def test_stability_slack_absorbs_hardware_jitter():
    jitter = _stats(queue_early=1, queue_end=2, p99_first=2.0, p99_last=4.5)
    assert not is_stable(jitter)                                  # the reference rule
    assert is_stable(jitter, queue_slack=4, p99_slack_ms=5.0)
    overload = _stats(queue_early=60, queue_end=250, p99_first=50.0, p99_last=200.0)
    assert not is_stable(overload, queue_slack=16, p99_slack_ms=5.0)
