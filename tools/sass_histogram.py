"""Blackwell-native evidence from the built library: per kernel, the count of
tcgen05 / TMA / TMEM / multimem SASS instructions (cuobjdump -sass).
python tools/sass_histogram.py [lib] > profiles/r2_sass_histogram.txt"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

lib = sys.argv[1] if len(sys.argv) > 1 else str(Path(__file__).resolve().parents[1] / "paper_2404_14691_b200" / "libsagedp.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "UTCMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCATOMSWS",
        "LDGSTS", "MULTIMEM", "SYNCS", "HMMA", "FENCE.VIEW.ASYNC"]
cur, hist = None, {}
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        hist[cur] = Counter()
        continue
    if cur is None:
        continue
    for k in KEYS:
        if re.search(r"\b" + re.escape(k), line):
            hist[cur][k] += 1
dem = {}
names = list(hist)
out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
for n, d in zip(names, out):
    dem[n] = d
print(f"# cuobjdump -sass {Path(lib).name}: tcgen05 / TMA / TMEM instruction counts per kernel")
print("# UTC*MMA = tcgen05.mma, UTMALDG = TMA tensor load, LDTM = tcgen05.ld, LDGSTS = cp.async, MULTIMEM = multimem.*")
for n in sorted(hist, key=lambda x: dem[x]):
    c = hist[n]
    if not c:
        continue
    print(f"{dem[n][:110]:110s} " + " ".join(f"{k}={v}" for k, v in sorted(c.items())))
