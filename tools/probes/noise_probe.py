"""Pure-noise X at C2 shape: which path dominates?"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2107_10654_b200 import rtucker as rt  # noqa: E402
shape, R = (512, 512, 512), 16
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(shape, dtype=torch.float64, device="cuda", generator=g)
t = rt.Tensor.from_device(x.data_ptr(), shape)
opts = rt.options(lam=1e-2, sketched_core=1, sample_count_override=200000, tolerance=0.0,
                  max_iterations=4, seed=0, record_history=1)
r = rt.als_run(t, (R,) * 3, opts, profile=True)
print("sketch", r.sketch_info())
print("hist", [(h[0], h[1], round(h[2], 3)) for h in r.history()])
tot = sum(k[1] for k in r.kernels())
for name, secs, n in sorted(r.kernels(), key=lambda k: -k[1])[:10]:
    print(f"  {name:16s} {secs * 1e3:9.3f} ms  {n:6d}  {100 * secs / tot:5.1f}%")
