"""Probe (not the bench): the expanded-form loss (||X||^2 - 2<X,Xhat> + ||Xhat||^2 from T, P and
the core) against the direct residual pass at C2, and the X-pass kernel times of each."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_10654_b200 import rtucker as rt  # noqa: E402

shape, R, s = (512, 512, 512), 16, 200000
ranks = (R,) * 3
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
rt.set_stream(torch.cuda.current_stream().cuda_stream)
t = rt.Tensor.from_device(x.data_ptr(), shape)
res = {}
for fast in (False, True):
    r = rt.als_run(t, ranks, rt.options(lam=1e-2, sketched_core=1, sample_count_override=s,
                                        tolerance=0.0, max_iterations=8, record_history=1),
                   profile=True, fast_loss=fast)
    res[fast] = r.history()
    fam = {}
    for name, secs, n in r.kernels():
        fam[name] = (fam.get(name, (0, 0))[0] + secs, fam.get(name, (0, 0))[1] + n)
    print("fast" if fast else "direct", {k: (round(v[0] * 1e3 / 8, 3), v[1]) for k, v in fam.items()
                                          if k.startswith("ttm") or k.startswith("loss")})
for a, b in zip(res[False], res[True]):
    print(a[0], a[1], "%.17g %.17g rel %.3e" % (a[2], b[2], abs(a[2] - b[2]) / abs(a[2])))
