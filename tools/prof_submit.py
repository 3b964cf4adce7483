"""Split per-invocation submit time: policy/sharing (Python) vs sage_invoke (native)."""
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
sim.dataplane.stage_sources_in_hbm(0)
sim.dataplane.results_in_hbm = True
L = _lib.lib()
acc = {"invoke": 0.0, "n": 0}
orig = L.sage_invoke


def timed_invoke(*a):
    t = time.perf_counter()
    r = orig(*a)
    acc["invoke"] += time.perf_counter() - t
    acc["n"] += 1
    return r


L.sage_invoke = timed_invoke


def wrap(obj, name, key):
    orig_fn = getattr(obj, name)

    def w(*a, **k):
        t = time.perf_counter()
        r = orig_fn(*a, **k)
        acc[key] = acc.get(key, 0.0) + time.perf_counter() - t
        return r
    setattr(obj, name, w)


wrap(sim.policy, "_try_start", "try_start")
wrap(sim, "start_invocation", "start_inv")
wrap(sim.dataplane, "_enqueue_fast", "enqueue_fast")
wrap(sim.sharing, "preview", "preview")
wrap(sim.sharing, "admit", "admit")
for stats in (0, 1):
    L.sage_stats_enable(stats)
    for rep in range(8):
        for r in list(sim.sharing.residents.values()):
            sim.sharing.evict(r)
        for k in list(acc):
            acc[k] = 0.0 if k != "n" else 0
        t0 = time.perf_counter()
        sim.submit_many(names)
        t1 = time.perf_counter()
        sim.drain()
        t2 = time.perf_counter()
    print(f"stats={stats}: submit {1e6*(t1-t0)/64:.1f} us/inv, of which sage_invoke {1e6*acc['invoke']/acc['n']:.1f} us; "
          f"burst total {1e3*(t2-t0):.2f} ms; per inv: " +
          ", ".join(f"{k} {1e6*v/64:.1f}" for k, v in acc.items() if k not in ("n", "invoke")))
sim.close()

# ---- where the host time goes (cProfile over 4 bursts, stats off) ----------
import cProfile  # noqa: E402
import pstats  # noqa: E402

sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data, copy_results=False)
sim.dataplane.stage_sources_in_hbm(0)
sim.dataplane.results_in_hbm = True
L.sage_stats_enable(0)
for rep in range(3):
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
    sim.submit_many(names)
    sim.drain()
pr = cProfile.Profile()
for rep in range(4):
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
    pr.enable()
    sim.submit_many(names)
    sim.drain()
    pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(40)
st.sort_stats("cumulative").print_stats(40)
sim.close()
