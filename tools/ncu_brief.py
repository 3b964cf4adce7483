"""One-screen summary of an ncu --set full report (raw page): duration, DRAM
bytes / throughput, SM / tensor activity, occupancy, top stall reasons.
python tools/ncu_brief.py report.ncu-rep"""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(h, vals))
u = dict(zip(h, units))
keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
for k in keys:
    m = [kk for kk in d if kk == k or kk.startswith(k)]
    if m:
        print(f"{m[0]:75s} {d[m[0]]} {u.get(m[0], '')}")
st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
      and not k.endswith("not_issued") and v.replace(".", "").isdigit()]
st.sort(key=lambda x: -x[1])
tot = sum(v for _, v in st) or 1
print("top stalls (pc samples): " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} "
                                             f"{v / tot:.0%}" for k, v in st[:6]))
