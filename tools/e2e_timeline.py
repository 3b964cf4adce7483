"""Per-invocation stage timeline of one e2e cfg-2 burst (pinned host store +
pinned request payloads, results D2H): where does the 64-burst spend its
time?  Prints one JSON object per invocation (µs relative to the arrival) and
a summary of when the PCIe directions were busy."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.functions import Stage  # noqa: E402
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402

table, data = cfg2_functions()
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data, copy_results=False)
names = [sorted(table)[k % 3] for k in range(64)]
pls = []
for n in names:
    pb = D.PinnedBuffer(data[n].input_bytes)
    pb.view()[:] = data[n].input
    pls.append(pb)
sim.dataplane.pin_host_store()
import os  # noqa: E402
from paper_2404_14691_b200 import _lib  # noqa: E402
_lib.check(_lib.lib().sage_stats_enable(int(os.environ.get("SAGE_TIMELINE_STATS", "0"))), "stats_enable")
out = []
spans = []                                     # (first H2D begin, last return end) per burst
walls = []
import time  # noqa: E402
REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 6
for rep in range(REPS):
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
    t_sub = time.perf_counter()
    invs = sim.submit_many(names, payloads=pls)
    t_done = time.perf_counter()
    sim.drain()
    t_drained = time.perf_counter()
    walls.append([round((t_done - t_sub) * 1e6), round((t_drained - t_sub) * 1e6)])
    spans.append([min(i.stages[Stage.GPU_LOAD][0] for i in invs), max(i.stages[Stage.RETURN][1] for i in invs)])
    if rep == REPS - 1:
        t0 = min(i.arrival_us for i in invs)
        for i in invs:
            st = {s.name.lower(): [b - t0, e - t0] for s, (b, e) in i.stages.items()}
            out.append({"id": i.id, "fn": i.spec.name, "warmth": i.warmth.name, "setup": i.setup_us,
                        "lat": i.latency_us, "stages": st})
for o in out:
    print(json.dumps(o))
end = max(o["stages"]["return"][1] for o in out)
print(json.dumps({"bursts_us": [round(b - a) for a, b in spans],
                  "gaps_between_bursts_us": [round(spans[k + 1][0] - spans[k][1]) for k in range(len(spans) - 1)],
                  "submit_and_drain_wall_us": walls}))
print(json.dumps({"burst_us": end,
                  "last_gpu_load_end": max(o["stages"]["gpu_load"][1] for o in out),
                  "first_return_begin": min(o["stages"]["return"][0] for o in out),
                  "last_compute_end": max(o["stages"]["compute"][1] for o in out)}))
sim.dataplane.unpin_host_store()
sim.close()
