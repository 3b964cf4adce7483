"""One cfg-2 Poisson probe (or several rates) on a warm plane: backlog and
p99 per rate -- the stability inputs of `experiments peak`.
python tools/probe_peak.py chunk_mb rate [rate ...]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.replay import run_probe  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402
from paper_2404_14691_b200.workload import PoissonOpenSpec, generate_arrivals  # noqa: E402

chunk = float(sys.argv[1])
table, data = cfg2_functions()
sim = Simulation(ClusterSpec(gpus=1, chunk_mb=chunk, staging_mb=8 * chunk), policy_preset("SAGE"), table, seed=1,
                 function_data=data, copy_results=False)
try:
    sim.prepare()
    for rate in map(float, sys.argv[2:]):
        arr = generate_arrivals(PoissonOpenSpec(rate, 2.0, {n: 1.0 for n in table}), 1)
        t0 = time.perf_counter()
        n0 = len(sim.invocations)
        loads0 = dict(sim.sharing.ro_loads_performed)
        st = run_probe(sim, arr, 2_000_000)
        invs = sim.invocations[n0:]
        warmth = {}
        for i in invs:
            warmth[i.warmth.name] = warmth.get(i.warmth.name, 0) + 1
        loads = {f"{k[0]}": v - loads0.get(k, 0) for k, v in sim.sharing.ro_loads_performed.items()}
        print(json.dumps({"chunk_mb": chunk, "rate": rate, "queue_early": st.queue_early, "queue_end": st.queue_end,
                          "p99_first_ms": st.p99_first_quartile_ms, "p99_last_ms": st.p99_last_quartile_ms,
                          "wall_s": round(time.perf_counter() - t0, 2), "warmth": warmth, "ro_loads": loads,
                          "residents": {f"{k[0]}": r.state.label for k, r in sim.sharing.residents.items()}}),
              flush=True)
finally:
    sim.close()
