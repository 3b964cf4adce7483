"""BASELINE.json configs on the real plane (reference drivers:
pkg/src/gslsim/experiments.py:37-193 -- run / compare on one pre-generated
stream / peak).  Each runner returns a JSON-able dict.

  cfg1  16 concurrent cold starts of one 100 MiB function: SAGE vs FixedGSL
  cfg2  the Parboil burst (bench.py)
  cfg3  ResNet-50 inference function under Poisson arrivals; PCIe-once +
        peer-land fan-out across G (logical on a 1-GPU pool) GPUs
  cfg4  ten functions with RO log-spaced 10 MiB .. 2 GiB, Poisson mix under
        the 180 GB budget: resident density and time-averaged memory
  cfg5  N = 1..512 simultaneous cold starts of a 100 MiB function: SAGE vs
        the host-only loading path (every invocation pulls its own copy)

    python -m paper_2404_14691_b200.experiments cfg1 cfg3 cfg4 cfg5 --out profiles/
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

from .functions import FunctionSpec, Stage
from .parboil import synthetic_function
from .policies import policy_preset
from .runtime import ClusterSpec, Simulation, percentile, summarize_setup
from .workload import OpenLoopSource, PoissonOpenSpec, generate_arrivals


def _evict_all(sim) -> None:
    if sim.sharing is not None:
        for r in list(sim.sharing.residents.values()):
            sim.sharing.evict(r)


def _round(d):
    return {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items()}


def cfg1(n: int = 16, reps: int = 5) -> dict:
    """BASELINE cfg 1: n concurrent cold starts of one 100 MiB function.
    SAGE vs DGSF (4 pre-created contexts) vs FixedGSL with a fresh context per
    instance -- on a library thread, or in its own OS process -- alone (N=1)
    and n at once."""
    spec, data = synthetic_function("fn100", 100, 10, 1, tensors=64)
    out = {}
    rows = (("SAGE", "SAGE", "thread", n, reps + 1), ("DGSF", "DGSF", "thread", n, 3),
            ("FixedGSL_thread_n1", "FixedGSL", "thread", 1, 4), ("FixedGSL", "FixedGSL", "thread", n, 2),
            ("FixedGSL_process_n1", "FixedGSL", "process", 1, 4), ("FixedGSL_process", "FixedGSL", "process", n, 2))
    for row, pol, mode, burst, r in rows:
        sim = Simulation(ClusterSpec(gpus=1, instance_mode=mode), policy_preset(pol), {spec.name: spec}, seed=1,
                         function_data={spec.name: data})
        try:
            sim.prepare()
            samples = []
            for rep in range(r):
                _evict_all(sim)
                invs = sim.submit_many([spec.name] * burst)
                sim.drain()
                if rep >= (1 if r > 1 else 0):     # the first burst warms the process
                    samples += invs
            s = summarize_setup(samples)
            s["bursts"] = r - (1 if r > 1 else 0)
            s["concurrent"] = burst
            if pol == "FixedGSL":
                ctx = [i.stages[Stage.GPU_CTX][1] - i.stages[Stage.GPU_CTX][0] for i in samples]
                s["fresh_context_ms_p50"] = percentile(ctx, 50) / 1e3
            out[row] = _round(s)
        finally:
            sim.close()
    sage = out["SAGE"]["setup_p50_ms"]
    out["p50_setup_ratio"] = round(out["FixedGSL"]["setup_p50_ms"] / sage, 1)
    out["p50_setup_ratio_process"] = round(out["FixedGSL_process"]["setup_p50_ms"] / sage, 1)
    out["p50_setup_ratio_dgsf"] = round(out["DGSF"]["setup_p50_ms"] / sage, 1)
    out["workload"] = f"{n} concurrent cold starts, 100 MiB RO (64 ragged tensors), 10 MiB writable, 1 MiB input"
    return out


def cfg3(rate: float = 300.0, duration_s: float = 4.0, gpus_list=(1, 2, 4), seed: int = 1, dtype: str = "fp32",
         engine: str | None = None, prewarm: int = 64, window: int | None = None) -> dict:
    from .dnn import resnet50
    spec, data = resnet50(dtype=dtype, engine=engine)
    arrivals = generate_arrivals(PoissonOpenSpec(rate, duration_s, {spec.name: 1.0}), seed)
    out = {"engine": data.body, "workload": f"ResNet-50 (random init, {data.layout.seg_bytes} B {dtype} weights, batch 8) "
                       f"Poisson {rate:g}/s for {duration_s:g} s ({len(arrivals)} arrivals), plane pre-warmed with a "
                       f"{prewarm}-invocation burst" + (f", admission window {window} per GPU" if window else "")}
    for g in gpus_list:
        sim = Simulation(ClusterSpec(gpus=g, admission_window=window), policy_preset("SAGE"), {spec.name: spec},
                         seed=seed, function_data={spec.name: data}, copy_results=False)
        try:
            sim.prepare()
            # deployment warm-up: graph instances of the program, streams, pool
            # chunks and pinned buffers exist before the first arrival
            sim.prewarm(prewarm)
            src = OpenLoopSource(arrivals)
            t0 = time.perf_counter()
            src.attach(sim)
            sim.source = src
            sim.drain()
            wall = time.perf_counter() - t0
            invs = [i for i in sim.invocations if i.outcome == "completed"]
            srcs = {}
            for i in invs:
                if i.ro_source:
                    srcs[i.ro_source] = srcs.get(i.ro_source, 0) + 1
            s = summarize_setup(invs)
            from . import dnn
            s.update(graph_captures=dict(dnn.CAPTURES))
            s.update(gpus=g, throughput_per_s=len(invs) / wall, wall_s=wall, ro_loads=srcs,
                     pcie_ro_bytes=sum(i.measured["pcie_bytes"] for i in invs),
                     nvlink_bytes=sum(i.measured.get("nvlink_bytes", 0) for i in invs),
                     note="logical GPUs share the one physical B200 of this pool" if g > 1 else "")
            out[f"G{g}"] = _round(s)
            sim.check_no_leaks()
        finally:
            sim.close()
    return out


def cfg4(rate: float = 10.0, duration_s: float = 6.0, seed: int = 1, include_fixedgsl: bool = True) -> dict:
    ro = [10 * (2048 / 10) ** (k / 9) for k in range(10)]          # log-spaced 10 .. 2048 MiB
    table, data = {}, {}
    for k, r in enumerate(ro):
        spec, fd = synthetic_function(f"f{k}", round(r, 1), round(0.05 * r, 1), round(0.01 * r, 2), tensors=32)
        table[spec.name] = spec
        data[spec.name] = fd
    arrivals = generate_arrivals(PoissonOpenSpec(rate, duration_s, {n: 1.0 for n in table}), seed)
    out = {"workload": f"10 functions, RO {', '.join(f'{r:.1f}' for r in ro)} MiB; Poisson {rate:g}/s for "
                       f"{duration_s:g} s ({len(arrivals)} arrivals); 180 GB budget"}
    for pol in (("SAGE", "FixedGSL") if include_fixedgsl else ("SAGE",)):
        sim = Simulation(ClusterSpec(gpus=1), policy_preset(pol), table, seed=seed, function_data=data,
                         copy_results=False)
        try:
            sim.prepare()
            samples = []
            peak_res = 0
            peak_mem = 0
            area = 0.0
            last = [time.perf_counter(), 0]

            def tick(*_):
                nonlocal peak_res, peak_mem, area
                now = time.perf_counter()
                used = sim.gpu_ledgers[0].usage
                area += last[1] * (now - last[0])
                last[0], last[1] = now, used
                peak_mem = max(peak_mem, used)
                if sim.sharing is not None:
                    peak_res = max(peak_res, sum(1 for r in sim.sharing.residents.values() if r.gpu_ro or r.gpu_ctx))
                samples.append(used)

            sim.completion_listeners.append(lambda inv, now: tick())
            src = OpenLoopSource(arrivals)
            t0 = time.perf_counter()
            last[0] = t0
            src.attach(sim)
            sim.source = src
            sim.drain()
            tick()
            wall = time.perf_counter() - t0
            invs = [i for i in sim.invocations if i.outcome == "completed"]
            s = summarize_setup(invs)
            s.update(throughput_per_s=len(invs) / wall, wall_s=wall, peak_resident_functions=peak_res,
                     peak_gpu_mem_gb=peak_mem / 1e9, avg_gpu_mem_gb=area / max(1e-9, wall) / 1e9)
            out[pol] = _round(s)
            print(json.dumps({"cfg4_partial": pol, **out[pol]}), file=sys.stderr, flush=True)
        finally:
            sim.close()
    return out


def cfg5(ns=(1, 2, 4, 8, 16, 32, 64, 128, 256, 512), reps: int = 3, gpus_list=(1,)) -> dict:
    """N simultaneous cold starts of one 100 MiB function on G GPUs: SAGE
    (PCIe once per box + NVLink peer lands, shared) vs the host-only loading
    path (SAGE-NR: every invocation lands its own copy over PCIe).  G > 1
    runs logical GPUs on this pool's one device: placement, sharing and the
    PCIe-once invariant are real, the NVLink bandwidth is not."""
    spec, data = synthetic_function("fn100", 100, 10, 1, tensors=64)
    out = {"workload": "N simultaneous cold starts of one 100 MiB function: SAGE (PCIe once, shared, NVLink "
                       "fan-out) vs host-only loading (SAGE-NR: every invocation lands its own copy)"}
    for g in gpus_list:
        for pol in ("SAGE", "SAGE_NR"):
            sim = Simulation(ClusterSpec(gpus=g), policy_preset(pol), {spec.name: spec}, seed=1,
                             function_data={spec.name: data}, copy_results=False)
            try:
                sim.prepare()
                _evict_all(sim)
                sim.submit_many([spec.name] * 4 * g)         # warm the process
                sim.drain()
                rows = {}
                for n in ns:
                    setups, walls, pcie, nvl = [], [], 0, 0
                    for _ in range(reps):
                        _evict_all(sim)
                        t0 = time.perf_counter()
                        invs = sim.submit_many([spec.name] * n)
                        sim.drain()
                        walls.append(time.perf_counter() - t0)
                        setups += [i.setup_us for i in invs]
                        pcie = sum(i.measured["pcie_bytes"] for i in invs)
                        nvl = sum(i.measured.get("nvlink_bytes", 0) for i in invs)
                    rows[str(n)] = {"setup_p50_ms": round(percentile(setups, 50) / 1e3, 3),
                                    "setup_p99_ms": round(percentile(setups, 99) / 1e3, 3),
                                    "burst_ms": round(1e3 * min(walls), 3), "pcie_bytes": pcie,
                                    "nvlink_bytes": nvl}
                out[pol if g == 1 else f"{pol}_G{g}"] = rows
            finally:
                sim.close()
    return out


def _workload(kind: str):
    """(spec table, function data) of a named workload."""
    if kind in ("cfg3", "cfg3_bf16"):
        from .dnn import resnet50
        spec, data = resnet50(dtype="bf16" if kind == "cfg3_bf16" else "fp32")
        return {spec.name: spec}, {spec.name: data}
    from .parboil import cfg2_functions
    return cfg2_functions()


def trace(path: str, workload: str = "cfg2", policy: str = "SAGE", time_scale: float = 1.0, seed: int = 1,
          out_dir=None) -> dict:
    """Replay a flat trace CSV (reference format) on the real plane and write
    the reference's artifacts (summary.json, invocations.csv,
    memory_timeline.csv) -- reference `gslsim run` with a trace workload."""
    from . import reports
    from .replay import TraceSpec, trace_arrivals
    table, data = _workload(workload)
    arrivals = trace_arrivals(TraceSpec(path, time_scale), known_functions=set(table))
    sim = Simulation(ClusterSpec(gpus=1), policy_preset(policy), table, seed=seed, function_data=data,
                     copy_results=False)
    try:
        sim.prepare()
        tls = [reports.MemoryTimeline(g, l, lambda: sim.engine.now) for g, l in enumerate(sim.gpu_ledgers)]
        src = OpenLoopSource(arrivals)
        t0 = sim.engine.tick()
        src.attach(sim)
        sim.source = src
        sim.drain()
        duration = max(1, sim.engine.tick() - t0)
        for tl in tls:
            tl.close()
        summary = reports.summarize(sim.invocations, duration, table, tls)
        if out_dir:
            reports.write_artifacts(out_dir, sim, duration, tls)
        summary["workload"] = f"trace {path} ({len(arrivals)} arrivals, time scale {time_scale:g}) over {workload}"
        return summary
    finally:
        sim.close()


def peak(workload: str = "cfg2", probe_s: float = 2.0, rate_min: float = 50.0, rate_ceiling: float = 65536.0,
         resolution: float = 0.05, seed: int = 1, prewarm: int = 256) -> dict:
    """Largest stable Poisson rate of a workload on one B200 (reference
    `gslsim peak`, experiments.py:128-155): doubling + bisection over
    `probe_s`-second probes on one warm plane."""
    from .replay import find_peak_throughput, run_probe
    table, data = _workload(workload)
    sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=seed, function_data=data,
                     copy_results=False)
    probes = []
    try:
        sim.prepare()
        sim.prewarm(prewarm)
        dur = int(probe_s * 1e6)

        def probe(rate: float):
            arr = generate_arrivals(PoissonOpenSpec(rate, probe_s, {n: 1.0 for n in table}), seed)
            n0 = len(sim.invocations)
            loads0 = dict(sim.sharing.ro_loads_performed) if sim.sharing is not None else {}
            st = run_probe(sim, arr, dur)
            warmth: dict = {}
            for i in sim.invocations[n0:]:
                w = i.warmth.name if i.warmth is not None else "none"
                warmth[w] = warmth.get(w, 0) + 1
            loads = ({k[0]: v - loads0.get(k, 0) for k, v in sim.sharing.ro_loads_performed.items()}
                     if sim.sharing is not None else {})
            probes.append({"rate_per_s": rate, "arrivals": len(arr), "queue_early": st.queue_early,
                           "queue_end": st.queue_end, "p99_first_ms": st.p99_first_quartile_ms,
                           "p99_last_ms": st.p99_last_quartile_ms, "warmth": warmth, "ro_loads": loads})
            return st

        res = find_peak_throughput(probe, rate_min=rate_min, rate_ceiling=rate_ceiling, resolution=resolution,
                                   queue_slack=16, p99_slack_ms=5.0)
        return {"workload": f"{workload} Poisson probes of {probe_s:g} s, SAGE, 1 GPU, plane pre-warmed with a "
                            f"{prewarm}-invocation burst",
                "stability": "reference rule (replay.is_stable) + slack: backlog +16 invocations, p99 +5 ms",
                "peak_rate_per_s": res.rate_per_s, "hit_ceiling": res.hit_ceiling, "diagnostic": res.diagnostic,
                "trajectory": [[r, ok] for r, ok in res.trajectory], "probes": probes}
    finally:
        sim.close()


RUNNERS = {"cfg1": cfg1, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5, "peak": peak}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", choices=sorted(RUNNERS))
    ap.add_argument("--out", default=None)
    ap.add_argument("--rate", type=float, default=None, help="cfg3: Poisson rate (/s)")
    ap.add_argument("--window", type=int, default=None, help="cfg3: admission window per GPU (default none)")
    ap.add_argument("--gpus", default=None, help="cfg3: comma-separated logical GPU counts")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg3", "cfg3_bf16"],
                    help="peak / trace: function set")
    ap.add_argument("--trace", default=None, help="trace: flat trace CSV (timestamp_ms,function)")
    ap.add_argument("--time-scale", type=float, default=1.0)
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "bf16"], help="cfg3: ResNet-50 weights / input")
    ap.add_argument("--engine", default=None, choices=["native", "torch"],
                    help="cfg3: ResNet-50 body (default: native for bf16, torch for fp32)")
    args = ap.parse_args(argv)
    if args.trace:
        res = trace(args.trace, args.workload, time_scale=args.time_scale, out_dir=args.out)
        print(json.dumps({"trace": res}), flush=True)
        return
    for c in args.configs:
        t0 = time.perf_counter()
        kw = {}
        if c == "peak":
            kw["workload"] = args.workload
        if c == "cfg5" and args.gpus:
            kw["gpus_list"] = tuple(int(g) for g in args.gpus.split(","))
        if c == "cfg3":
            if args.rate is not None:
                kw["rate"] = args.rate
            if args.gpus:
                kw["gpus_list"] = tuple(int(g) for g in args.gpus.split(","))
            kw["dtype"] = args.dtype
            kw["engine"] = args.engine
            kw["window"] = args.window
        res = RUNNERS[c](**kw)
        res["elapsed_s"] = round(time.perf_counter() - t0, 1)
        line = json.dumps({c: res})
        print(line, flush=True)
        if args.out:
            Path(args.out).mkdir(parents=True, exist_ok=True)
            (Path(args.out) / f"{c}.json").write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
