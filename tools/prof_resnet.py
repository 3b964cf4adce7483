"""Host cost of ResNet-50 invocations (CUDA-graph bodies): bursts of 64 on a
warm plane, wall time per invocation + cProfile of one burst."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200.dnn import resnet50  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
spec, data = resnet50(dtype=dtype)
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), {spec.name: spec}, seed=1,
                 function_data={spec.name: data}, copy_results=False)
sim.prepare()
for _ in range(3):
    sim.submit_many([spec.name] * 64)
    sim.drain()
t0 = time.perf_counter()
for _ in range(5):
    t = time.perf_counter()
    sim.submit_many([spec.name] * 64)
    ts = time.perf_counter() - t
    sim.drain()
dt = time.perf_counter() - t0
print(f"{dtype}: {dt / 320 * 1e6:.0f} us wall per invocation over 5 bursts of 64 (last submit {ts / 64 * 1e6:.0f} us/inv)")
pr = cProfile.Profile()
pr.enable()
sim.submit_many([spec.name] * 64)
sim.drain()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
sim.close()
