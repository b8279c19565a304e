"""Probe (not the bench): the C1 C-API job's wall time with and without CUDA-graph sweeps,
and where a job's time goes (device sweep time vs setup)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2107_10654_b200 import rtucker as rt  # noqa: E402

x = bench.c1_input(np)
opts = rt.options(lam=bench.C1_LAM, sketched_core=1, tolerance=0.0,
                  sample_count_override=bench.C1_S, max_iterations=bench.C1_SWEEPS, seed=0)
for i in range(3):
    bench.capi_als_job(rt.lib, opts, x, bench.C1_RANKS)
ts = []
for i in range(20):
    t, loss = bench.capi_als_job(rt.lib, opts, x, bench.C1_RANKS)
    ts.append(t)
print(os.environ.get("RTB_NO_GRAPH", "graph"), "median job ms %.3f" % (1e3 * sorted(ts)[10]),
      "min %.3f" % (1e3 * min(ts)), "loss", loss)
xt = rt.Tensor.from_numpy(x)
for i in range(3):
    t0 = time.perf_counter()
    r = rt.als_run(xt, bench.C1_RANKS, opts)
    t1 = time.perf_counter()
    print("als_run only ms %.3f  device sweep_seconds %.4f" % (1e3 * (t1 - t0), r.sweep_seconds))

# host-side phases of a 10-sweep job through the session API
for i in range(3):
    t0 = time.perf_counter()
    s = rt.Session(xt, bench.C1_RANKS, opts)
    t1 = time.perf_counter()
    s.sweeps(1)
    t2 = time.perf_counter()
    s.sweeps(1)
    t3 = time.perf_counter()
    s.sweeps(8)
    t4 = time.perf_counter()
    r = s.result()
    t5 = time.perf_counter()
    s.free()
    t6 = time.perf_counter()
    print("session ms: create %.3f sweep1 %.3f sweep2(capture) %.3f sweeps3-10 %.3f result %.3f "
          "free %.3f" % tuple(1e3 * v for v in (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5)))
