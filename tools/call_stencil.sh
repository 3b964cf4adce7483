#!/bin/bash
# stencil4_kernel under ncu (cold cache, serialized): device duration per launch (the variants
# swept in profiles/r2_stencil_variants.txt were removed; SAGE_STENCIL is ignored now)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for m in 0 41 46 48 28 86; do
  SAGE_STENCIL=$m timeout 300 ncu --clock-control none -k regex:stencil -c 10 --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
    python tools/stencil_sweep.py > gpurun_out/st_$m.csv 2>&1
  python - $m <<'PY'
import csv, sys, statistics
rows = [r for r in csv.reader(open(f"gpurun_out/st_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; rows = rows[1:]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
by = {}
for r in rows: by.setdefault(r[mi], []).append(float(r[vi].replace(",", "")))
t = statistics.median(by["gpu__time_duration.sum"])
print(sys.argv[1], "ns", t, "GBps", round(50331648 / t, 1), "dram_rd", statistics.median(by["dram__bytes_read.sum"]),
      "dram_wr", statistics.median(by["dram__bytes_write.sum"]), "warps", statistics.median(by["sm__warps_active.avg.pct_of_peak_sustained_active"]))
PY
done | tee gpurun_out/stencil_ncu.txt
