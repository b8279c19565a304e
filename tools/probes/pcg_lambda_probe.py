import sys, numpy as np
sys.path.insert(0,'.')
from paper_2107_10654_b200 import rtucker as rt
shape, ranks = (40, 36, 32), (6, 5, 4)
x = np.random.default_rng(12).standard_normal(shape)
kw = dict(lam=0.5, sketched_core=1, max_iterations=3, tolerance=0.0, sample_count_override=6000, record_history=1, seed=4)
r = rt.als_run(rt.Tensor.from_numpy(x), ranks, rt.options(**kw))
print(r.sketch_info())
