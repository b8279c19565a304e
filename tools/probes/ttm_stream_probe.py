"""One F_3 projection (X x_1 A_1^T, the ttm_mid2 pass) through the single-op
update_factor entry; with RTB_TTM_STREAM_ONLY=1 the pass only streams X (result is
garbage) so ncu shows the achievable load bandwidth of the same pipeline."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2107_10654_b200 import rtucker as rt  # noqa: E402
shape, R = (512, 512, 512), 16
x = torch.randn(shape, dtype=torch.float64, device="cuda")
t = rt.Tensor.from_device(x.data_ptr(), shape)
rng = np.random.default_rng(0)
core = rng.standard_normal((R, R, R))
fs = [rng.standard_normal((i, R)) for i in shape]
m = rt.Model(core, fs, 0.01)
for _ in range(3):
    rt.update_factor(t, m, 3)
torch.cuda.synchronize()
print("ok")
