import sys, os, numpy as np
sys.path.insert(0, '.')
from paper_2107_10654_b200 import rtucker as rt
from oracle.oracle import Oracle
o = Oracle()
shape, ranks = tuple(int(v) for v in sys.argv[1].split(',')), tuple(int(v) for v in sys.argv[2].split(','))
s = int(sys.argv[3])
rng = np.random.default_rng(0)
x = rng.standard_normal(shape)
fs = [rng.standard_normal((i, r)) for i, r in zip(shape, ranks)]
scs, cdfs, sums = [], [], []
for f in fs:
    sc, cdf, tot, _ = o.factor_scores(f); scs.append(sc); cdfs.append(cdf); sums.append(tot)
idx, w, _ = o.kron_draw(shape, int(np.prod(ranks)), scs, cdfs, sums, 5, s)
g, r = rt.kron_normal_eq(shape, ranks, fs, x, 1e-2, idx, w)
np.savez(sys.argv[4], g=g, r=r)
print(rt.variant_count("k_vech_bucket5"))
