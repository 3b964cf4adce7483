"""Reference decisions for tests/test_pressure_gpu.py: four 300 MB functions
(context 64 MB) cycled through a two-resident budget (800 MB), arrivals 1 s
apart so each finishes before the next, as on the real plane.  Imports
gslsim from /root/reference/pkg/src (build container only).

    python tests/golden/make_pressure_golden.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

from gslsim.config import parse_config  # noqa: E402
from gslsim.experiments import run_experiment  # noqa: E402

FUNCS = {f"f{k}": {"ro_mem_mb": 300, "writable_mem_mb": 16, "compute_ms": 1, "context_mem_mb": 64,
                   "input_bytes_host_mb": 2, "input_bytes_pcie_mb": 2} for k in range(4)}
SEQ = [f"f{k % 4}" for k in range(10)] + ["f3", "f3", "f1"]


def main():
    c = parse_config({"cluster": {"gpus": 1, "gpu_mem_mb": 800}, "functions": FUNCS, "policy": "SAGE", "seed": 1,
                      "duration_s": len(SEQ) + 5,
                      "workload": {"kind": "sequence", "arrivals": [[1000 * k, n] for k, n in enumerate(SEQ)]}})
    res = run_experiment(c)
    invs = sorted(res.sim.invocations, key=lambda i: i.id)
    out = {"functions": FUNCS, "sequence": SEQ, "gpu_mem_mb": 800,
           "warmth": [i.warmth.label() for i in invs], "outcome": [i.outcome for i in invs],
           "ro_loads": {k[0]: v for k, v in res.sim.sharing.ro_loads_performed.items()}}
    path = Path(__file__).with_name("pressure_golden.json")
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(out["warmth"])


if __name__ == "__main__":
    main()
