#!/bin/bash
# One-off box probe: FP64 peaks (DMMA, DFMA, cuBLAS DGEMM), host cores, toolchain.
set -x
nvidia-smi; nproc; lscpu | head -20; free -g
./tools/probes/fp64_peak
python - <<'PY'
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device='cuda'); b = torch.randn_like(a)
for _ in range(3): c = a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): c = a @ b
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("cuBLAS DGEMM 8192^3: %.2f TFLOP/s" % (2 * 8192**3 / ms / 1e9))
x = torch.empty(2**28, dtype=torch.float64, device='cuda'); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); e0.record()
for _ in range(10): y.copy_(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("copy GB/s: %.1f" % (2 * x.numel() * 8 / ms / 1e6))
PY
