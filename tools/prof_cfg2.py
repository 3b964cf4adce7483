"""Where does a cfg-2 burst spend its time? host submit vs device drain, + cProfile."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402

table, data = cfg2_functions()
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data, copy_results=False)
names = [sorted(table)[k % 3] for k in range(64)]
payloads = []
for n in names:
    pb = D.PinnedBuffer(data[n].input_bytes)
    pb.view()[:] = data[n].input
    payloads.append(pb)
mode = sys.argv[1] if len(sys.argv) > 1 else "e2e"
if mode == "value":
    sim.dataplane.stage_sources_in_hbm(0)
    sim.dataplane.results_in_hbm = True
    payloads = None
elif mode == "e2e":
    sim.dataplane.pin_host_store()


def burst():
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
    t0 = time.perf_counter()
    invs = sim.submit_many(names, payloads=payloads)
    t1 = time.perf_counter()
    sim.drain()
    t2 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t0) * 1e3, invs


for _ in range(3):
    burst()
rows = [burst() for _ in range(5)]
print(mode, "submit_ms", [round(r[0], 2) for r in rows], "total_ms", [round(r[1], 2) for r in rows])
invs = rows[-1][2]
last = max(invs, key=lambda i: i.completion_us)
t0 = min(i.arrival_us for i in invs)
print("timeline (ms from arrival): name warmth | gpu_load | compute | return")
for i in sorted(invs, key=lambda i: i.stages[next(iter(i.stages))][0]):
    cols = []
    for k, v in i.stages.items():
        if k.value in ("gpu_load", "compute", "return", "sync_wait"):
            cols.append(f"{k.value[:4]} {(v[0] - t0) / 1e3:6.2f}-{(v[1] - t0) / 1e3:6.2f}")
    print(f"{i.id:5d} {i.spec.name:8s} {i.warmth.label():8s} {i.ro_source or '-':6s} | " + " | ".join(cols))
pr = cProfile.Profile()
pr.enable()
burst()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
sim.close()
