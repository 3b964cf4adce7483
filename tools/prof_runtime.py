"""cProfile of the SAGE submit path (control-plane overhead per invocation)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200.functions import spec_from_dict  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation, summarize_setup  # noqa: E402

table = {"fn100": spec_from_dict("fn100", {"ro_mem_mb": 100, "writable_mem_mb": 10, "compute_ms": 1,
                                           "input_bytes_host_mb": 1, "input_bytes_pcie_mb": 1})}
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1)
for rep in range(3):
    invs = sim.submit_many(["fn100"] * 64)
    sim.drain()
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
pr = cProfile.Profile()
pr.enable()
for rep in range(5):
    invs = sim.submit_many(["fn100"] * 64)
    sim.drain()
    for r in list(sim.sharing.residents.values()):
        sim.sharing.evict(r)
pr.disable()
print(summarize_setup(invs))
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
sim.close()
