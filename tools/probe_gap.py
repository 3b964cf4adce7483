"""Host time between e2e bursts: drain return -> residents evicted -> the
next burst's first invocation submitted (the device sits idle meanwhile)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402

table, data = cfg2_functions()
names = bench.burst_names(table, 64)
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data, copy_results=False)
pls = []
for n in names:
    pb = D.PinnedBuffer(data[n].input_bytes)
    pb.view()[:] = data[n].input
    pls.append(pb)
sim.dataplane.pin_host_store()
ev, sub1, sub_all, drain = [], [], [], []
try:
    for k in range(25):
        t0 = time.perf_counter()
        for r in list(sim.sharing.residents.values()):
            sim.sharing.evict(r)
        t1 = time.perf_counter()
        first = sim.submit_many(names[:1], payloads=pls[:1])
        t2 = time.perf_counter()
        rest = sim.submit_many(names[1:], payloads=pls[1:])
        t3 = time.perf_counter()
        sim.drain()
        t4 = time.perf_counter()
        if k >= 5:
            ev.append((t1 - t0) * 1e6); sub1.append((t2 - t1) * 1e6); sub_all.append((t3 - t1) * 1e6)
            drain.append((t4 - t3) * 1e6)
    med = lambda v: round(sorted(v)[len(v) // 2], 1)
    print(json.dumps({"evict_us": med(ev), "first_submit_us": med(sub1), "submit_all_us": med(sub_all),
                      "drain_after_submit_us": med(drain)}))
finally:
    sim.dataplane.unpin_host_store()
    sim.close()
