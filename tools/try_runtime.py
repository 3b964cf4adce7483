"""Quick end-to-end run of the runtime (cfg-1 shape): SAGE vs FixedGSL."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200.functions import spec_from_dict  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation, summarize_setup  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
pols = sys.argv[2].split(",") if len(sys.argv) > 2 else ["SAGE", "FixedGSL"]
table = {"fn100": spec_from_dict("fn100", {"ro_mem_mb": 100, "writable_mem_mb": 10, "compute_ms": 1,
                                           "input_bytes_host_mb": 1, "input_bytes_pcie_mb": 1})}
out = {}


def rel(inv):
    return {k.value: [v[0] - inv.arrival_us, v[1] - inv.arrival_us] for k, v in inv.stages.items()}


for pol in pols:
    sim = Simulation(ClusterSpec(gpus=1), policy_preset(pol), table, seed=1)
    try:
        for rep in range(3 if pol == "SAGE" else 1):
            t0 = time.perf_counter()
            invs = sim.submit_many(["fn100"] * n)
            t1 = time.perf_counter()
            sim.drain()
            t2 = time.perf_counter()
            s = summarize_setup(invs)
            s["submit_ms"] = (t1 - t0) * 1e3
            s["wall_ms"] = (t2 - t0) * 1e3
            s["warmth"] = sorted({i.warmth.label() for i in invs})
            s["ro_sources"] = sorted({i.ro_source for i in invs})
            s["checksums"] = len({i.ro_checksum for i in invs if i.ro_checksum})
            s["inv0"] = rel(invs[0])
            s["inv_last"] = rel(invs[-1])
            out[f"{pol}_rep{rep}"] = s
            if sim.sharing is not None:   # force a cold start next rep
                for r in list(sim.sharing.residents.values()):
                    sim.sharing.evict(r)
        sim.check_no_leaks()
    finally:
        sim.close()
print(json.dumps(out, indent=1, default=str))
