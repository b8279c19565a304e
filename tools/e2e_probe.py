"""Times the phases of one C2 e2e job (RTB_TRACE=1 prints the library's own phase split)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RTB_TRACE", "1")
import torch
import bench
from paper_2107_10654_b200 import rtucker as rt

x = bench.make_input(torch, torch.device("cuda"))
xh = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
xh.copy_(x)
del x
xnp = xh.numpy()
for graph in (True, False, True):
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = rt.Tensor.from_numpy(xnp)
        t1 = time.perf_counter()
        r = rt.als_run(th, bench.RANKS, rt.options(lam=bench.LAM, sketched_core=1,
                                                   sample_count_override=bench.S_CORE,
                                                   tolerance=0.0, max_iterations=10, seed=0),
                       graph=graph)
        t2 = time.perf_counter()
        m = r.model()
        t3 = time.perf_counter()
        print(f"graph={graph} create {1e3*(t1-t0):.1f} ms, als_run {1e3*(t2-t1):.1f} ms, "
              f"model {1e3*(t3-t2):.1f} ms, graph sweeps {r.graph_sweeps}", flush=True)
        r.free()
        th.free()
