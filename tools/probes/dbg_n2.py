"""Debug probe: N=2 sketched ALS sweep vs the oracle, step by step."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle.oracle import Oracle  # noqa: E402
from paper_2107_10654_b200 import rtucker as rt  # noqa: E402
from test_gpu_parity import planted  # noqa: E402

shape, ranks, lam, s = (64, 60), (9, 7), 1e-2, 3000
if len(sys.argv) > 1:
    shape = tuple(int(v) for v in sys.argv[1].split(","))
    ranks = tuple(int(v) for v in sys.argv[2].split(","))
o_ = Oracle()
x = planted(shape, ranks, seed=31)
kw = dict(lam=lam, sketched_core=1, max_iterations=1, tolerance=0.0, sample_count_override=s,
          record_history=1, seed=9)
o = o_.als(x, ranks, **kw)
cs = int(o["core_seeds"][0])
core0, f0 = o_.random_model(shape, ranks, 9)
fs = [f.copy() for f in f0]
for m in range(len(shape)):
    fs[m] = o_.update_factor(shape, ranks, core0, fs, lam, x, m + 1)
oc, oidx, ow, _ = o_.update_core_fast(shape, ranks, core0, fs, lam, x, s, cs)
print("oracle replay core == als core:", np.array_equal(oc.ravel(), o["core"].ravel()))
gc, gidx, gw = rt.update_core_sketched(rt.Tensor.from_numpy(x), rt.Model(core0, fs, lam), s, cs)
print("gpu single-op: idx equal", np.array_equal(gidx, oidx),
      "core rel", np.linalg.norm(gc.ravel() - oc.ravel()) / np.linalg.norm(oc))
r = rt.als_run(rt.Tensor.from_numpy(x), ranks, rt.options(**kw))
m = r.model()
for k in range(len(shape)):
    print("factor", k, "rel", np.linalg.norm(m.factors[k] - o["factors"][k]) / np.linalg.norm(o["factors"][k]))
print("gpu als core rel", np.linalg.norm(m.core.ravel() - o["core"].ravel()) / np.linalg.norm(o["core"]))
print("sketch_info", r.sketch_info())
print("gpu hist", r.history())
print("orc hist", o["history"])
for k, f in enumerate(fs):
    osc, ocdf, otot, orank = o_.factor_scores(f)
    g = rt.factor_scores(f)
    print("mode", k, "oracle rank", orank, "tot", otot, "gpu", [type(v) for v in g] if isinstance(g, tuple) else g)
    gsc = g[0]
    print("   scores rel", np.max(np.abs(gsc - osc)) / np.max(np.abs(osc)), "cdf eq", np.array_equal(g[1], ocdf) if len(g) > 1 else None)
    print("   eig AtA", np.linalg.eigvalsh(f.T @ f))
