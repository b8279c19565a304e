"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches_c2.csv"
sweeps = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:58]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for k, v in agg.items() if "at::" not in k)
print(f"per-sweep (÷{sweeps}); rtb kernels only total {tot / 1e6 / sweeps:.3f} ms")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    if "at::" in k:
        continue
    print(f"{k:58s} n={v[0] / sweeps:6.1f} ms={v[1] / 1e6 / sweeps:7.3f} avg_us={v[1] / v[0] / 1e3:8.2f} "
          f"{100 * v[1] / tot:5.1f}%")
