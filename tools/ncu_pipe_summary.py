"""DMMA-pipe / DRAM / stall summary per kernel of an ncu --set full report:
python tools/ncu_pipe_summary.py rep.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
idx = {n: i for i, n in enumerate(h)}
stall = [c for c in h if c.startswith("smsp__average_warps_issue_stalled")
         and c.endswith("per_issue_active.ratio")]
print(f"{'kernel':34s} {'dur_us':>9s} {'DMMA%act':>8s} {'DRAM_rd_GB':>10s} {'DRAM_wr_GB':>10s} "
      f"{'warps%':>6s}  top stalls (per issue)")
for r in rows[2:]:
    name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")[:34]
    scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}

    def g(k):
        try:
            v = float(r[idx[k]].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")
        return v * scale.get(rows[1][idx[k]], 1.0) if k.startswith("dram__bytes") else v
    st = []
    for c in stall:
        try:
            st.append((float(r[idx[c]]), c.replace("smsp__average_warps_issue_stalled_", "")
                       .replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
    st = sorted(st, reverse=True)[:3]
    dur = g("gpu__time_duration.sum")
    unit = rows[1][idx["gpu__time_duration.sum"]]
    dur_us = dur * (1e3 if unit == "ms" else 1e-3 if unit == "ns" else 1.0)
    print(f"{name:34s} {dur_us:9.1f} "
          f"{g('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active'):8.1f} "
          f"{g('dram__bytes_read.sum'):10.3f} {g('dram__bytes_write.sum'):10.3f} "
          f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f}  "
          + ", ".join(f"{n} {v:.2f}" for v, n in st))
