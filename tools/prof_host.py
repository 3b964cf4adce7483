"""Wall-clock split of the host path per invocation in the value leg (HBM
sources, D2D results): admission (policy/sharing/ledger), the data-plane
enqueue (descriptor build + sage_invoke), completion (collect / release /
policy.complete) -- by wrapping the methods with perf_counter timers."""
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200 import dataplane as DP  # noqa: E402
from paper_2404_14691_b200 import policies as P  # noqa: E402
from paper_2404_14691_b200 import runtime as R  # noqa: E402
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402

acc = defaultdict(float)
cnt = defaultdict(int)


def wrap(cls, name, label):
    orig = getattr(cls, name)

    def f(*a, **k):
        t = time.perf_counter()
        try:
            return orig(*a, **k)
        finally:
            acc[label] += time.perf_counter() - t
            cnt[label] += 1
    setattr(cls, name, f)


wrap(R.Simulation, "submit", "submit (total)")
wrap(P.SharingPolicy, "_try_start", "  _try_start (admission+start)")
wrap(DP.DataPlane, "start", "    dataplane.start")
wrap(DP.DataPlane, "_enqueue_fast", "      _enqueue_fast")
wrap(DP.DataPlane, "_on_done", "_on_done (completion total)")
wrap(DP.DataPlane, "_collect_fast", "  _collect_fast")
wrap(DP.DataPlane, "_release", "  _release")
wrap(P.SharingPolicy, "complete", "  policy.complete")
wrap(DP._FastCompletions, "poll", "poll (incl. waits)")

table, data = cfg2_functions()
sim = R.Simulation(R.ClusterSpec(gpus=1), P.policy_preset("SAGE"), table, seed=1, function_data=data,
                   copy_results=False)
names = [sorted(table)[k % 3] for k in range(64)]
sim.dataplane.stage_sources_in_hbm(0)
sim.dataplane.results_in_hbm = True
for rep in range(25):
    if rep == 5:
        acc.clear()
        cnt.clear()
        t0 = time.perf_counter()
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
    sim.submit_many(names)
    sim.drain()
wall = time.perf_counter() - t0
n = 20 * 64
print(f"{n} invocations, {wall * 1e6 / n:.1f} us wall per invocation")
for k, v in acc.items():
    print(f"{k:38s} {v * 1e6 / n:8.1f} us/inv   ({cnt[k]} calls)")
sim.close()
