"""Top SASS instructions by stall samples: python tools/sass_hot.py rep.ncu-rep [n] [kernel-regex]"""
import csv
import subprocess
import sys

cmd = ["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"]
if len(sys.argv) > 3:
    cmd += ["--kernel-name", "regex:" + sys.argv[3], "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
tot = {c: 0 for c in cols}
T = 0
data = []
for r in rows[2:]:
    try:
        v = {c: int(r[h.index(c)]) for c in cols}
        s = int(r[si])
    except (ValueError, IndexError):
        continue
    for c in cols:
        tot[c] += v[c]
    T += s
    data.append((s, r[0][-5:], r[1][:56], int(r[ii] or 0), v))
print("total samples", T)
for c in sorted(cols, key=lambda c: -tot[c])[:8]:
    print(f"  {c:24s} {tot[c]:8d} {100 * tot[c] / max(T, 1):5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for s, a, ins, ie, v in sorted(data, key=lambda x: -x[0])[:n]:
    top = sorted(v.items(), key=lambda kv: -kv[1])[:2]
    print(f"{s:7d} {a} {ins:56s} n={ie:<9d} {top[0][0][6:]}={top[0][1]} {top[1][0][6:]}={top[1][1]}")
