"""BASELINE config 3 probe: 160^4 FP64, planted rank (10,10,10,10), factor rows scaled by
i.i.d. Pareto(1.5) weights, 5% noise, lambda = 0.1, s_core = 500,000, optional sketched
factor updates (argv[1] = factor samples, 0 = exact). Prints sweeps/s, sketch info and the
per-kernel-family device times."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2107_10654_b200 import rtucker as rt  # noqa: E402

fs = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
I, R, lam, s = 160, 10, 0.1, 500000
shape, ranks = (I,) * 4, (R,) * 4
g = torch.Generator(device="cuda").manual_seed(0)
core = torch.randn(ranks, dtype=torch.float64, device="cuda", generator=g)
x = core
for n in range(4):
    f = torch.randn(I, R, dtype=torch.float64, device="cuda", generator=g)
    u = torch.rand(I, 1, dtype=torch.float64, device="cuda", generator=g)
    f = f * (1.0 - u) ** (-1.0 / 1.5)  # Pareto(alpha = 1.5, x_m = 1) row weights
    x = torch.movedim(torch.tensordot(f, x, dims=([1], [n])), 0, n)
x = x + 0.05 * x.norm() / x.numel() ** 0.5 * torch.randn(x.shape, dtype=torch.float64,
                                                           device="cuda", generator=g)
x = x.contiguous()
torch.cuda.synchronize()
t = rt.Tensor.from_device(x.data_ptr(), shape)
opts = rt.options(lam=lam, sketched_core=1, sample_count_override=s, tolerance=0.0,
                  max_iterations=sweeps + 1)
sess = rt.Session(t, ranks, opts, profile=True, factor_samples=fs)
t0 = time.time()
sess.sweeps(1)
torch.cuda.synchronize()
t1 = time.time()
sess.sweeps(sweeps)
torch.cuda.synchronize()
t2 = time.time()
r = sess.result()
print(f"C3 factor_samples={fs}: warm {t1 - t0:.3f}s, {sweeps} sweeps {t2 - t1:.4f}s -> "
      f"{sweeps / (t2 - t1):.2f} sweeps/s; device sweep_seconds {r.sweep_seconds:.4f}")
print("final loss %.17g" % r.final_loss)
print("sketch:", r.sketch_info())
tot = sum(k[1] for k in r.kernels())
for name, secs, n in sorted(r.kernels(), key=lambda k: -k[1]):
    print(f"  {name:16s} {secs * 1e3:9.3f} ms  {n:6d} launches  {100 * secs / tot:5.1f}%")
