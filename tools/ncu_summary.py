"""Per-kernel key metrics from an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Achieved Occupancy",
        "Registers Per Thread", "Grid Size", "Block Size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
iid, ik, im, iv, iu = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"),
                       h.index("Metric Value"), h.index("Metric Unit"))
kern = {}
for r in rows[1:]:
    if len(r) <= iv:
        continue
    k = (int(r[iid]), r[ik].split("(")[0].replace("void ", "")[:34])
    if r[im] in KEYS and r[im] not in kern.setdefault(k, {}):
        kern[k][r[im]] = r[iv] + ("" if r[iu] in ("", "%") else " " + r[iu])
print(f"{'id':>3} {'kernel':34s} " + " ".join(f"{x[:10]:>10s}" for x in KEYS[:8]))
for (i, name), m in sorted(kern.items()):
    print(f"{i:>3} {name:34s} " + " ".join(f"{m.get(x, '-')[:10]:>10s}" for x in KEYS[:8]))
