"""Where the end-to-end job time goes (tensor_create / als_run / result_model)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2107_10654_b200 import rtucker as rt  # noqa: E402

shape, R = (512, 512, 512), 16
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(shape, dtype=torch.float64, device="cuda", generator=g)
xh = torch.empty(shape, dtype=torch.float64, pin_memory=True)
xh.copy_(x)
xnp = xh.numpy()
xpage = np.array(xnp)  # pageable copy
for label, arr in [("pinned", xnp), ("pageable", xpage)]:
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = rt.Tensor.from_numpy(arr)
        t1 = time.perf_counter()
        r = rt.als_run(th, (R,) * 3, rt.options(lam=1e-2, sketched_core=1, sample_count_override=200000,
                                               tolerance=0.0, max_iterations=10, seed=0))
        t2 = time.perf_counter()
        m = r.model()
        t3 = time.perf_counter()
        r.free()
        th.free()
        t4 = time.perf_counter()
        print(f"{label} it{it}: create {1e3*(t1-t0):.1f} ms, als {1e3*(t2-t1):.1f} ms, model {1e3*(t3-t2):.1f} ms, "
              f"free {1e3*(t4-t3):.1f} ms, sweeps(dev) {r.sweep_seconds*1e3 if False else 0:.1f}")
