"""Diagnose stage-time conversion: arrival vs device-event stage times in
bench's leg order (e2e with stats, then HBM-resident value leg)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2404_14691_b200 import _lib  # noqa: E402
from paper_2404_14691_b200 import device as D  # noqa: E402
from paper_2404_14691_b200.functions import Stage  # noqa: E402
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402

table, data = cfg2_functions()
names = bench.burst_names(table, 64)
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data, copy_results=False)
L = _lib.lib()
L.sage_stats_enable(int(sys.argv[1]) if len(sys.argv) > 1 else 1)


def show(tag, invs):
    s = sorted(i.setup_us for i in invs)
    i = invs[0]
    print(tag, "setup min/med/max us", s[0], s[len(s) // 2], s[-1], "arr", i.arrival_us,
          {k.value: v for k, v in i.stages.items()})


for leg in ("e2e", "value"):
    if leg == "value":
        sim.dataplane.stage_sources_in_hbm(0)
        sim.dataplane.results_in_hbm = True
    for step in range(6):
        invs = bench.run_steps(sim, names, 1)
        show(f"{leg}{step}", invs)
    e = sim.engine
    print("engine now", e.now, "wall", e.wall_us(), "lib", D.now_us())
sim.close()
