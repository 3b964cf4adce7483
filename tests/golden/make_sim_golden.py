"""Generate tests/golden/sim_parity.json from the reference simulator itself.

Imports gslsim from /root/reference/pkg/src (present only in the build
container; the JSON travels with the repo, the reference does not) and
records, per scenario, what the reference decides for each invocation:
warmth class, whether it waits on a leader, planned host/PCIe bytes (µMB),
read-only load counts and GPU ledger usage by class.  The real plane must
reproduce every one of these exactly (after MB := MiB unit conversion);
tests/test_runtime_gpu.py replays the same arrival lists on a B200 and
tests/test_host_logic.py replays the admission logic on CPU.

Timing-sensitive scenarios use arrival gaps centred in the 30 s decay
windows, so a replay with every time scaled by 1/100 (0.3 s windows, ms
invocations) classifies identically.

    python tests/golden/make_sim_golden.py
"""
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from gslsim.config import parse_config  # noqa: E402
from gslsim.experiments import run_experiment  # noqa: E402
from gslsim.functions import Stage, builtin_spec_table  # noqa: E402
from gslsim.resources import AllocClass  # noqa: E402


def cfg(policy, arrivals, duration_s, functions="builtin", cluster=None, **abl):
    data = {"cluster": cluster or {"gpus": 1}, "functions": functions, "policy": policy, "seed": 1,
            "duration_s": duration_s, "workload": {"kind": "sequence", "arrivals": arrivals}}
    data.update(abl)
    return parse_config(data)


def record(sim):
    out = []
    for inv in sorted(sim.invocations, key=lambda i: i.id):
        out.append({
            "id": inv.id, "function": inv.spec.name, "gpu": inv.gpu, "outcome": inv.outcome,
            "warmth": inv.warmth.label() if inv.warmth is not None else None,
            "sync_wait": Stage.SYNC_WAIT in inv.stages,
            "has_gpu_ctx": Stage.GPU_CTX in inv.stages,
            "host_bytes_umb": inv.host_bytes_umb, "pcie_bytes_umb": inv.pcie_bytes_umb,
        })
    return out


def usage_at_zero(c):
    """Ledger usage by class right after every t=0 admission."""
    from gslsim.config import build_simulation
    sim = build_simulation(c)
    sim.engine.run(until=0)
    led = sim.gpu_ledgers[0]
    allocs = sorted([a.cls.value, a.requested_umb, a.effective_umb] for a in led.allocations())
    return {cl.value: v for cl, v in led.usage_by_class().items()} | {"total": led.usage_umb, "allocs": allocs}


def main():
    fixture = {"units": "umb (1 MB = 10^6 umb); replay converts MB := MiB", "scenarios": {}}
    S = fixture["scenarios"]
    table = {"fn100": {"ro_mem_mb": 100, "writable_mem_mb": 10, "compute_ms": 1,
                       "input_bytes_host_mb": 1, "input_bytes_pcie_mb": 1}}

    # burst of 16 cold starts of one 100 MB function (BASELINE cfg 1)
    for pol in ("SAGE", "SAGE_NR", "FixedGSL", "FixedGSLF", "DGSF"):
        c = cfg(pol, [[0, "fn100"]] * 16, 30, functions=table)
        res = run_experiment(c)
        sc = {"arrivals_ms": [[0, "fn100"]] * 16, "functions": table, "policy": pol,
              "invocations": record(res.sim), "usage_t0": usage_at_zero(c)}
        if res.sim.sharing is not None:
            sc["ro_loads"] = {f"{k[0]}@{k[1]}": v for k, v in res.sim.sharing.ro_loads_performed.items()}
        S[f"burst16_{pol}"] = sc

    # staged warm-state probe (validate_table5 arrivals): Cold, Stage1Hot,
    # Stage2, Stage3, Stage4, Cold
    arr = [[0, "resnet50"], [15500, "resnet50"], [60600, "resnet50"], [135800, "resnet50"],
           [241200, "resnet50"], [366700, "resnet50"]]
    res = run_experiment(cfg("SAGE", arr, 400))
    S["table5_SAGE"] = {"arrivals_ms": arr, "functions": "builtin", "policy": "SAGE", "invocations": record(res.sim),
                        "ro_loads": {f"{k[0]}@{k[1]}": v for k, v in res.sim.sharing.ro_loads_performed.items()}}

    # byte conservation over a run (test_simulation.py:171-182): ro_loads == 3
    arr = [[0, "resnet50"], [0, "resnet50"], [100, "resnet50"], [40000, "resnet50"], [200000, "resnet50"]]
    res = run_experiment(cfg("SAGE", arr, 220))
    S["conservation_SAGE"] = {"arrivals_ms": arr, "functions": "builtin", "policy": "SAGE",
                              "invocations": record(res.sim),
                              "ro_loads": {f"{k[0]}@{k[1]}": v for k, v in res.sim.sharing.ro_loads_performed.items()}}

    # allocation closed forms for every builtin function (test_policies.py:134-146)
    alloc = {}
    for name in sorted(builtin_spec_table()):
        a = {}
        for pol in ("FixedGSL", "SAGE", "SAGE_NR", "FixedGSLF"):
            a[pol] = usage_at_zero(cfg(pol, [[0, name]], 5))
        alloc[name] = a
    S["alloc_builtin"] = alloc

    # two concurrent resnet50 under SAGE: only writable is new (test_policies.py:116-121)
    S["sage_two_resnet_t0"] = usage_at_zero(cfg("SAGE", [[0, "resnet50"], [0, "resnet50"]], 10))

    # mixed burst on 2 GPUs: placement from the dispatcher stream
    arr = [[0, "resnet50"]] * 6 + [[0, "vgg11"]] * 6
    res = run_experiment(cfg("SAGE", arr, 10, cluster={"gpus": 2}))
    S["mixed_2gpu_SAGE"] = {"arrivals_ms": arr, "functions": "builtin", "policy": "SAGE", "gpus": 2,
                            "invocations": record(res.sim),
                            "ro_loads": {f"{k[0]}@{k[1]}": v for k, v in res.sim.sharing.ro_loads_performed.items()}}

    # the reference's open-loop Poisson streams (workload.py:75-113)
    from gslsim.workload import PoissonOpenSpec, generate_arrivals
    arr = {}
    for seed, rate, dur, mix in ((1, 50.0, 2.0, {"resnet50": 1.0}),
                                 (7, 400.0, 1.0, {"a": 1.0, "b": 2.0, "c": 0.5}),
                                 (3, 20.0, 30.0, {f"f{i}": 1.0 for i in range(10)})):
        recs = generate_arrivals(PoissonOpenSpec(rate_per_s=rate, duration_s=dur, mix=mix), seed)
        arr[f"seed{seed}_rate{rate:g}"] = {"seed": seed, "rate_per_s": rate, "duration_s": dur, "mix": mix,
                                           "arrivals": [[r.timestamp_us, r.function] for r in recs]}
    S["poisson_arrivals"] = arr

    path = Path(__file__).with_name("sim_parity.json")
    path.write_text(json.dumps(fixture, indent=1, sort_keys=True) + "\n")
    print(f"wrote {path} ({len(S)} scenarios)")


if __name__ == "__main__":
    main()
