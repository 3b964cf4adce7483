import sys, time
sys.path.insert(0, ".")
from paper_2404_14691_b200.parboil import cfg2_functions
from paper_2404_14691_b200.policies import policy_preset
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation
table, data = cfg2_functions()
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data, copy_results=False)
sim.submit_many([sorted(table)[k % 3] for k in range(64)])
sim.drain()
print("drained; exiting without close", flush=True)
if len(sys.argv) > 1:
    raise SystemExit(0)
