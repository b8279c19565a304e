"""Quick perf probe: one config, per-kernel-family device times (not the bench)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2107_10654_b200 import rtucker as rt  # noqa: E402

shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "512,512,512").split(","))
R = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s = int(sys.argv[3]) if len(sys.argv) > 3 else 200000
sweeps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
solver = int(sys.argv[5]) if len(sys.argv) > 5 else 0
fsamples = int(sys.argv[6]) if len(sys.argv) > 6 else 0
ranks = (R,) * len(shape)
g = torch.Generator(device="cuda").manual_seed(0)
core = torch.randn(ranks, dtype=torch.float64, device="cuda", generator=g)
x = core
for n, I in enumerate(shape):
    f = torch.randn(I, R, dtype=torch.float64, device="cuda", generator=g)
    x = torch.movedim(torch.tensordot(f, x, dims=([1], [n])), 0, n)
x = x + 0.01 * x.norm() / x.numel() ** 0.5 * torch.randn(x.shape, dtype=torch.float64,
                                                           device="cuda", generator=g)
x = x.contiguous()
torch.cuda.synchronize()
t = rt.Tensor.from_device(x.data_ptr(), shape)
opts = rt.options(lam=1e-2, sketched_core=1, sample_count_override=s, tolerance=0.0,
                  max_iterations=sweeps + 1)
t0 = time.time()
sess = rt.Session(t, ranks, opts, profile=True, core_solver=solver, factor_samples=fsamples)
sess.sweeps(1)
torch.cuda.synchronize()
t1 = time.time()
sess.sweeps(sweeps)
torch.cuda.synchronize()
t2 = time.time()
r = sess.result()
print(f"shape {shape} R {R} s {s}: warm {t1 - t0:.3f}s, {sweeps} sweeps wall {t2 - t1:.4f}s "
      f"-> {sweeps / (t2 - t1):.2f} sweeps/s; device sweep_seconds {r.sweep_seconds:.4f}")
print("solver", solver, "final loss %.17g" % r.final_loss)
print("sketch:", r.sketch_info())
tot = sum(k[1] for k in r.kernels())
for name, secs, n in sorted(r.kernels(), key=lambda k: -k[1]):
    print(f"  {name:16s} {secs * 1e3:9.3f} ms  {n:6d} launches  {100 * secs / tot:5.1f}%")
