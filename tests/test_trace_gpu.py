"""Trace replay on the real plane writes the reference's artifacts
(summary.json, invocations.csv, memory_timeline.csv), and the peak search
runs its probes on the plane."""
import csv
import json

import pytest

pytestmark = pytest.mark.gpu


def test_trace_replay_writes_reference_artifacts(built, tmp_path):
    from conftest import gpu_available
    from paper_2404_14691_b200 import reports
    from paper_2404_14691_b200.parboil import cfg2_functions
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.replay import TraceSpec, trace_arrivals
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
    from paper_2404_14691_b200.workload import OpenLoopSource
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    table, data = cfg2_functions(scale=8)
    names = sorted(table)
    tr = tmp_path / "trace.csv"
    tr.write_text("timestamp_ms,function\n" + "".join(f"{2.5 * k},{names[k % 3]}\n" for k in range(24)))
    arrivals = trace_arrivals(TraceSpec(str(tr)), known_functions=set(table))
    with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data) as sim:
        tls = [reports.MemoryTimeline(g, l, lambda: sim.engine.now) for g, l in enumerate(sim.gpu_ledgers)]
        t0 = sim.engine.tick()
        src = OpenLoopSource(arrivals)
        src.attach(sim)
        sim.source = src
        sim.drain()
        dur = sim.engine.tick() - t0
        for tl in tls:
            tl.close()
        summary = reports.write_artifacts(tmp_path / "out", sim, dur, tls)
        rows = list(csv.reader((tmp_path / "out" / "invocations.csv").open()))
        assert len(rows) == 25 and rows[0] == list(reports.INVOCATION_COLUMNS)
        col = {c: rows[0].index(c) for c in ("function", "warmth", "outcome", "compute_begin_ms")}
        for r, inv in zip(rows[1:], sorted(sim.invocations, key=lambda i: i.id)):
            assert r[col["function"]] == inv.spec.name and r[col["outcome"]] == "completed"
            assert r[col["warmth"]] == inv.warmth.label() and r[col["compute_begin_ms"]] != ""
        assert [r[col["warmth"]] for r in rows[1:4]] == ["Cold"] * 3
        on_disk = json.loads((tmp_path / "out" / "summary.json").read_text())
        assert on_disk["counts"]["completed"] == 24 == summary["counts"]["completed"]
        ro = sum(data[n].layout.seg_bytes for n in names)
        assert on_disk["gpu_memory_mb"]["gpu0"]["peak_mb"] * (1 << 20) >= ro
        tl_rows = list(csv.reader((tmp_path / "out" / "memory_timeline.csv").open()))
        assert tl_rows[0] == reports.TIMELINE_COLUMNS and len(tl_rows) > 4


def test_peak_search_probes_the_plane(built):
    from conftest import gpu_available
    from paper_2404_14691_b200.parboil import cfg2_functions
    from paper_2404_14691_b200.policies import policy_preset
    from paper_2404_14691_b200.replay import find_peak_throughput, run_probe
    from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
    from paper_2404_14691_b200.workload import PoissonOpenSpec, generate_arrivals
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    table, data = cfg2_functions(scale=8)
    with Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data) as sim:
        seen = []

        def probe(rate):
            arr = generate_arrivals(PoissonOpenSpec(rate, 0.25, {n: 1.0 for n in table}), 1)
            st = run_probe(sim, arr, 250_000)
            seen.append((rate, st.completed_first_quartile + st.completed_last_quartile))
            return st

        res = find_peak_throughput(probe, rate_min=100, rate_ceiling=400, resolution=0.5)
        assert res.trajectory and len(seen) == len(res.trajectory)
        assert all(done > 0 for _, done in seen)
        assert sim.in_flight == 0
