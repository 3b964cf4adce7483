"""Distribution of cfg-2 value-leg burst times (HBM sources, D2D results):
per burst host wall of submit_many and of drain, 40 bursts."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402

table, data = cfg2_functions()
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data, copy_results=False)
names = [sorted(table)[k % 3] for k in range(64)]
if "pre" in sys.argv:   # the bench order: e2e bursts (pinned payloads / store) first
    from paper_2404_14691_b200 import device as D
    pls = []
    for n in names:
        pb = D.PinnedBuffer(data[n].input_bytes)
        pb.view()[:] = data[n].input
        pls.append(pb)
    for pin in (False, True):
        if pin:
            sim.dataplane.pin_host_store()
        for rep in range(13):
            for r in list(sim.sharing.residents.values()):
                sim.sharing.evict(r)
            sim.submit_many(names, payloads=pls)
            sim.drain()
    sim.dataplane.unpin_host_store()
    for pb in pls:
        pb.free()
sim.dataplane.stage_sources_in_hbm(0)
sim.dataplane.results_in_hbm = True
_lib.lib().sage_stats_enable(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
rows = []
for rep in range(45):
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
    t0 = time.perf_counter()
    sim.submit_many(names)
    t1 = time.perf_counter()
    sim.drain()
    t2 = time.perf_counter()
    rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t2 - t0) * 1e3))
rows = rows[5:]
for k in range(3):
    col = sorted(r[k] for r in rows)
    print(["submit", "drain", "total"][k], "min %.2f p50 %.2f p90 %.2f max %.2f" % (col[0], statistics.median(col), col[int(0.9 * len(col))], col[-1]))
print("totals", [round(r[2], 2) for r in rows])
sim.close()
