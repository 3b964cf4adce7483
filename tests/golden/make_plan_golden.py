"""Every plan DAG the reference builds for its builtin function table
(functions.py:217-278): all specs x 5 warmth classes x {Serial, Parallel} x
pre_warmed x ctx_external x (wait_ro, wait_ctx) -- node stages, predecessor
sets, durations, byte counts and channels.  Imports gslsim from
/root/reference/pkg/src (build container only).

    python tests/golden/make_plan_golden.py
"""
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

from gslsim.functions import PlanMode, WarmthClass, builtin_spec_table, plan_invocation  # noqa: E402


def main():
    out = {}
    for name, spec in sorted(builtin_spec_table().items()):
        for w, mode, pre, ext, wr, wc in itertools.product(list(WarmthClass), list(PlanMode), (True, False),
                                                           (False, True), (False, True), (False, True)):
            plan = plan_invocation(spec, w, mode, pre_warmed=pre, ctx_external=ext, wait_ro=wr, wait_ctx=wc)
            key = f"{name}|{w.name}|{mode.name}|{int(pre)}{int(ext)}{int(wr)}{int(wc)}"
            out[key] = [[n.stage.value, sorted(n.preds), n.duration_us, n.bytes_umb, n.channel] for n in plan.nodes]
    path = Path(__file__).with_name("plan_golden.json")
    path.write_text(json.dumps(out, separators=(",", ":")) + "\n")
    print(f"wrote {path} ({len(out)} plans)")


if __name__ == "__main__":
    main()
