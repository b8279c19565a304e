"""C5 per-rank probe (not the bench): rank r of the BASELINE config-5 run on one GPU.

BASELINE configs[4]: 4096 x 4096 x 2048 FP64 (275 GB), planted rank (32,32,32), 1% noise,
lambda = 1e-2, s_core = 1e6, s_factor = 1e5, sharded across 8 GPUs. One B200 holds one
rank's 512 x 4096 x 2048 slab (34.4 GB). This script generates that slab on the device
(the same bytes rank r generates in the 8-GPU run) and runs the ALS sweep of rank r with
an identity all-reduce: every kernel rank r launches at P = 8, without the exchanges.

usage: python tools/c5_probe.py [P=8] [sweeps=3] [factor_samples=0] [I1_total=4096]
"""
import os
import sys
import time

import torch

# an identity all-reduce cannot feed the distributed core solve (each shard multiplies only its
# own mode-1 slices and the shares meet in the all-reduce): the probe keeps the replicated solve
os.environ.setdefault("RTB_NO_PCG_DIST", "1")

sys.path.insert(0, ".")
from paper_2107_10654_b200 import rtucker as rt  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
fs = int(sys.argv[3]) if len(sys.argv) > 3 else 0
I1 = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
shape, ranks = (I1, 4096, 2048), (32, 32, 32)
torch.cuda.set_device(0)
rt.set_stream(torch.cuda.current_stream().cuda_stream)
t0 = time.time()
x = rt.Tensor.generate_device(shape, ranks, 0.01, 0, shard=(0, P))
torch.cuda.synchronize()
print(f"generated rank-0 slab of {shape} over {P}: {x.shape} in {time.time() - t0:.2f}s",
      flush=True)


def ident(ptr, count, stream):
    pass


shard = rt.Shard(0, P, I1, ident) if P > 1 else None
opts = rt.options(lam=1e-2, sketched_core=1, sample_count_override=1000000, tolerance=0.0,
                  max_iterations=sweeps + 2)
t0 = time.time()
sess = rt.Session(x, ranks, opts, profile=True, factor_samples=fs, shard=shard)
sess.sweeps(1)
torch.cuda.synchronize()
t1 = time.time()
sess.sweeps(sweeps)
torch.cuda.synchronize()
t2 = time.time()
r = sess.result()
print(f"C5 rank-0 slab {x.shape} (P={P}) R=32 fs={fs}: first sweep {t1 - t0:.3f}s, "
      f"{sweeps} sweeps wall {t2 - t1:.4f}s -> {(t2 - t1) / sweeps * 1e3:.2f} ms/sweep")
print("losses", [h[2] for h in r.history()][-3:])
print("sketch:", r.sketch_info())
tot = sum(k[1] for k in r.kernels())
for name, secs, n in sorted(r.kernels(), key=lambda k: -k[1]):
    print(f"  {name:16s} {secs * 1e3:9.3f} ms  {n:6d} launches  {100 * secs / tot:5.1f}%")
