"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`):
per kernel launches, summed / mean / max duration and share of kernel time."""
import csv
import io
import sys
from collections import defaultdict


def summarise(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(list)
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r["Metric Unit"], 1e-3)
            agg[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values()) or 1.0
    lines = [f"{'kernel':28s} {'launches':>8s} {'total_us':>12s} {'mean_us':>9s} {'max_us':>9s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:28s} {len(v):8d} {sum(v):12.1f} {sum(v) / len(v):9.2f} {max(v):9.2f} {sum(v) / tot:6.3f}")
    lines.append(f"{'(all)':28s} {sum(len(v) for v in agg.values()):8d} {tot:12.1f}")
    # with launch__grid_size in the list: land launches by grid (staged chunk lands vs segment-sized ones)
    grid, dur = {}, {}
    for r in rows:
        if not r["Kernel Name"].startswith("land_kernel"):
            continue
        if r["Metric Name"] == "launch__grid_size":
            grid[r["ID"]] = int(float(r["Metric Value"].replace(",", "")))
        elif r["Metric Name"] == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r["Metric Unit"], 1e-3)
            dur[r["ID"]] = float(r["Metric Value"].replace(",", "")) * scale
    if grid:
        by = defaultdict(list)
        for i, g in grid.items():
            if i in dur:
                by[g].append(dur[i])
        lines.append("land_kernel by grid size (blocks: launches, mean_us)")
        for g in sorted(by):
            lines.append(f"  grid {g:6d}: {len(by[g]):5d} launches, mean {sum(by[g]) / len(by[g]):9.2f} us")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
