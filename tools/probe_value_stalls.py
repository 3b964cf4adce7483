"""Where do the rare 20+ ms value-leg steps go?  Runs the bench's value leg
(HBM-resident sources, results in HBM, per-kernel events on) for N steps with
per-phase wall times, and a sampler thread that snapshots the main thread's
Python stack every 1 ms; for every slow step, prints the phases and the
most-sampled stack lines.  python tools/probe_value_stalls.py [steps] [stats] [nvml]"""
import collections
import gc
import sys
import threading
import time
import traceback
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
stats = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nvml = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # 1: the bench's NVML clock sampler runs alongside
table, data = cfg2_functions()
names = bench.burst_names(table, 64)
sim = Simulation(ClusterSpec(gpus=1, chunk_mb=32, staging_mb=256), policy_preset("SAGE"), table, seed=1,
                 function_data=data, copy_results=False)
L = _lib.lib()
_lib.check(L.sage_stats_enable(stats), "stats")
sim.dataplane.stage_sources_in_hbm(0)
sim.dataplane.results_in_hbm = True
bench.run_steps(sim, names, 3)
main_id = threading.get_ident()
samples = []
sampling = threading.Event()
stop = False


def sampler():
    while not stop:
        if sampling.is_set():
            f = sys._current_frames().get(main_id)
            if f is not None:
                st = traceback.extract_stack(f)
                samples.append(" <- ".join(f"{Path(x.filename).name}:{x.lineno}:{x.name}" for x in st[-4:][::-1]))
        time.sleep(0.001)


th = threading.Thread(target=sampler, daemon=True)
th.start()
clocks = bench.ClockSampler(0).start() if nvml else None
gc.collect()
gc.disable()
rows = []
for k in range(steps):
    samples.clear()
    sampling.set()
    t0 = time.perf_counter()
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
    t1 = time.perf_counter()
    invs = sim.submit_many(names)
    t2 = time.perf_counter()
    sim.drain()
    t3 = time.perf_counter()
    _lib.check(L.sage_device_sync(0), "sync")
    t4 = time.perf_counter()
    sampling.clear()
    ph = [round((b - a) * 1e3, 2) for a, b in ((t0, t1), (t1, t2), (t2, t3), (t3, t4))]
    tot = round((t4 - t0) * 1e3, 2)
    rows.append(tot)
    if tot > 8.0:
        top = collections.Counter(samples).most_common(4)
        print(f"step {k}: {tot} ms  evict/submit/drain/sync {ph}")
        for s, c in top:
            print(f"    {c:4d}  {s}")
stop = True
gc.enable()
if clocks is not None:
    print("clocks", clocks.stop())
rows.sort()
print("steps", len(rows), "p50", rows[len(rows) // 2], "p90", rows[int(len(rows) * 0.9)], "max", rows[-1],
      "over 8 ms:", sum(r > 8 for r in rows))
