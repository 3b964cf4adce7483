"""cfg-5 tail probe: N simultaneous cold starts of the 100 MiB function, rep
by rep -- setup p50 / p99 / max per rep and the slowest invocation's stages.
python tools/probe_cfg5.py [N] [reps]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200.experiments import _evict_all, synthetic_function  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation, percentile  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec, data = synthetic_function("fn100", 100, 10, 1, tensors=64)
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=1,
                 function_data={spec.name: data}, copy_results=False)
sim.prepare()
_evict_all(sim)
sim.submit_many([spec.name] * 4)
sim.drain()
for r in range(reps):
    _evict_all(sim)
    t0 = time.perf_counter()
    invs = sim.submit_many([spec.name] * n)
    t_sub = time.perf_counter() - t0
    sim.drain()
    wall = time.perf_counter() - t0
    s = [i.setup_us for i in invs]
    worst = max(invs, key=lambda i: i.setup_us)
    a = worst.arrival_us
    print(json.dumps({"rep": r, "submit_ms": round(t_sub * 1e3, 2), "wall_ms": round(wall * 1e3, 2),
                      "p50_ms": round(percentile(s, 50) / 1e3, 2), "p99_ms": round(percentile(s, 99) / 1e3, 2),
                      "max_ms": round(max(s) / 1e3, 2), "worst_id": worst.id, "worst_warmth": worst.warmth.name,
                      "worst_stages": {k.name: [round((b - a) / 1e3, 2), round((e - a) / 1e3, 2)]
                                       for k, (b, e) in worst.stages.items()}}))
sim.close()
