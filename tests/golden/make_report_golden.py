"""Generate tests/golden/report_schema.json from the reference itself: the
artifact schema (invocations.csv / memory_timeline.csv columns, summary.json
keys) and the reference's invocations.csv rows (non-time columns) for the
16-way SAGE burst of BASELINE cfg 1.  Imports gslsim from
/root/reference/pkg/src (build container only; the JSON travels).

    python tests/golden/make_report_golden.py
"""
import csv
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

from gslsim import metrics as M  # noqa: E402
from gslsim.config import parse_config  # noqa: E402
from gslsim.experiments import run_experiment  # noqa: E402


def main():
    table = {"fn100": {"ro_mem_mb": 100, "writable_mem_mb": 10, "compute_ms": 1,
                       "input_bytes_host_mb": 1, "input_bytes_pcie_mb": 1}}
    c = parse_config({"cluster": {"gpus": 1}, "functions": table, "policy": "SAGE", "seed": 1, "duration_s": 30,
                      "workload": {"kind": "sequence", "arrivals": [[0, "fn100"]] * 16}})
    res = run_experiment(c)
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "invocations.csv"
        M.write_invocations_csv(p, res.sim.invocations)
        rows = list(csv.reader(p.open()))
    header = rows[0]
    keep = ["id", "function", "gpu", "warmth", "outcome", "host_bytes_mb", "pcie_bytes_mb"]
    idx = [header.index(k) for k in keep]
    summary = res.summary.to_dict()
    out = {"invocation_columns": list(M.INVOCATION_COLUMNS), "timeline_columns": list(M.TIMELINE_COLUMNS),
           "summary_keys": sorted(summary), "per_function_keys": sorted(next(iter(summary["per_function"].values()))),
           "burst16_SAGE": {"columns": keep, "rows": [[r[i] for i in idx] for r in rows[1:]]}}
    path = Path(__file__).with_name("report_schema.json")
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
