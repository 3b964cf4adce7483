"""Where does the wall-clock loop stall?  Runs cfg-2 Poisson probes (the
`experiments peak` sequence) with a sampling thread that snapshots the main
thread's Python stack every 2 ms; a stretch of >= 30 ms with the same
innermost frames is reported with its stack.  Diagnostic only.
python tools/stall_probe.py rate [rate ...]"""
import collections
import json
import sys
import threading
import time
import traceback
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_14691_b200.parboil import cfg2_functions  # noqa: E402
from paper_2404_14691_b200.policies import policy_preset  # noqa: E402
from paper_2404_14691_b200.replay import run_probe  # noqa: E402
from paper_2404_14691_b200.runtime import ClusterSpec, Simulation  # noqa: E402
from paper_2404_14691_b200.workload import PoissonOpenSpec, generate_arrivals  # noqa: E402

main_id = threading.get_ident()
stalls = collections.Counter()
stop = False


def sampler():
    last_key, since = None, time.perf_counter()
    while not stop:
        f = sys._current_frames().get(main_id)
        if f is not None:
            st = traceback.extract_stack(f)[-6:]
            key = tuple(f"{Path(x.filename).name}:{x.lineno}:{x.name}" for x in st)
            now = time.perf_counter()
            if key != last_key:
                if last_key is not None and now - since >= 0.03:
                    stalls[(round((now - since) * 1e3), last_key)] += 1
                last_key, since = key, now
        time.sleep(0.002)


table, data = cfg2_functions()
sim = Simulation(ClusterSpec(gpus=1), policy_preset("SAGE"), table, seed=1, function_data=data, copy_results=False)
th = threading.Thread(target=sampler, daemon=True)
try:
    sim.prepare()
    sim.prewarm(256)
    th.start()
    for rate in map(float, sys.argv[1:]):
        arr = generate_arrivals(PoissonOpenSpec(rate, 2.0, {n: 1.0 for n in table}), 1)
        st = run_probe(sim, arr, 2_000_000)
        print(json.dumps({"rate": rate, "queue_early": st.queue_early, "queue_end": st.queue_end,
                          "p99_first_ms": st.p99_first_quartile_ms, "p99_last_ms": st.p99_last_quartile_ms}),
              flush=True)
finally:
    stop = True
    sim.close()
for (ms, key), n in sorted(stalls.items(), key=lambda kv: -kv[0][0])[:12]:
    if any("sleep" in k or "poll" in k for k in key[-1:]):
        continue
    print(f"{ms:5d} ms x{n}: " + " <- ".join(reversed(key)))
