"""Compare two per-launch ncu lists of one native ResNet-50 forward (same op order).
python tools/layer_cmp.py before.csv after.csv"""
import csv
import io
import sys


def load(path):
    t = open(path).read()
    rows = list(csv.DictReader(io.StringIO(t[t.index('"ID"'):])))
    L = {}
    for r in rows:
        d = L.setdefault(r["ID"], {"k": r["Kernel Name"].split("(")[0].replace("void ", "")})
        d[r["Metric Name"]] = r["Metric Value"]
    out = [(v["k"], v.get("launch__grid_size"), float(v["gpu__time_duration.sum"].replace(",", "")) / 1e3)
           for v in L.values()]
    # the last full forward: from the last pad_c4_kernel through fc_kernel
    starts = [i for i, o in enumerate(out) if o[0].startswith(("pad_c4", "s2d_kernel"))]
    fw = out[starts[-2]:] if len(starts) > 1 else out
    ends = [i for i, o in enumerate(fw) if o[0].startswith("fc_kernel")]
    return fw[:ends[0] + 1] if ends else fw


a, b = load(sys.argv[1]), load(sys.argv[2])
print(f"{'#':>3} {'kernel':28s} {'grid':>5} {'before_us':>10} {'after_us':>10}")
for i, (x, y) in enumerate(zip(a, b)):
    print(f"{i:3d} {x[0][:28]:28s} {x[1]:>5} {x[2]:10.1f} {y[2]:10.1f}")
print(f"total {sum(x[2] for x in a):.1f} -> {sum(y[2] for y in b):.1f} us")
