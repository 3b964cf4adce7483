"""Per-thread CPU use of a command: runs it, samples /proc/<pid>/task/*/stat
every 0.5 s, prints each thread's (name) CPU share over the run.
python tools/thread_cpu.py -- <command ...>"""
import os
import subprocess
import sys
import time
from collections import defaultdict

cmd = sys.argv[sys.argv.index("--") + 1:]
p = subprocess.Popen(cmd, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
tick = os.sysconf("SC_CLK_TCK")
first, last, names = {}, {}, {}
t0 = time.time()
window = {}   # per 1 s window: thread name -> cpu
prev_tot, next_mark = {}, t0 + 1.0
while p.poll() is None:
    try:
        for tid in os.listdir(f"/proc/{p.pid}/task"):
            with open(f"/proc/{p.pid}/task/{tid}/stat") as f:
                st = f.read()
            name = st[st.index("(") + 1:st.rindex(")")]
            fields = st[st.rindex(")") + 2:].split()
            cpu = (int(fields[11]) + int(fields[12])) / tick
            first.setdefault(tid, cpu)
            last[tid] = cpu
            names[tid] = name
    except (FileNotFoundError, ProcessLookupError, ValueError):
        pass
    if time.time() >= next_mark:
        cur = defaultdict(float)
        for tid in last:
            cur[names[tid]] += last[tid]
        line = {n: round(cur[n] - prev_tot.get(n, 0.0), 2) for n in cur if cur[n] - prev_tot.get(n, 0.0) > 0.05}
        print(f"t={next_mark - t0:5.1f}s", dict(sorted(line.items())), flush=True)
        prev_tot = dict(cur)
        next_mark += 1.0
    time.sleep(0.25)
wall = time.time() - t0
by = defaultdict(float)
for tid in last:
    by[names[tid]] += last[tid] - first[tid]
for n, c in sorted(by.items(), key=lambda kv: -kv[1])[:12]:
    print(f"{n:20s} {c:7.2f} s cpu  {100 * c / wall:6.1f}% of {wall:.1f} s wall")
