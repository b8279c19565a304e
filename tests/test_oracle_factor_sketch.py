"""CPU checks of the oracle's sketched factor update (perf mode; parity unpinned by the
reference, which has no such mode -- SURVEY 8(c)). Pins the restatement's own
properties: its draws are the reference sampler's (orc_kron_draw over the other modes
with d = R_n), it reduces to the exact update as the sketch grows, and ALS with it is
deterministic in the seed."""
import numpy as np


def planted(shape, ranks, seed):
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    fs = [rng.standard_normal((i, r)) for i, r in zip(shape, ranks)]
    x = core
    for n, f in enumerate(fs):
        x = np.moveaxis(np.tensordot(f, x, axes=(1, n)), 0, n)
    return x + 0.01 * rng.standard_normal(x.shape), core, fs


def test_draws_are_the_product_sampler(oracle):
    shape, ranks = (9, 8, 7), (2, 3, 2)
    x, core, fs = planted(shape, ranks, 1)
    _, idx, w = oracle.update_factor_sketched(shape, ranks, core, fs, 0.01, x, 2, 500, 99)
    # same stream through the generic product sampler over modes 1 and 3, d = R_2
    others = [0, 2]
    sc, cdf, sums = [], [], []
    for m in others:
        s_, c_, t_, _ = oracle.factor_scores(fs[m])
        sc.append(s_)
        cdf.append(c_)
        sums.append(t_)
    i2, w2, _ = oracle.kron_draw([shape[m] for m in others], ranks[1], sc, cdf, sums, 99, 500)
    assert np.array_equal(idx, i2) and np.array_equal(w, w2)


def test_sketched_update_approaches_exact(oracle):
    shape, ranks = (12, 10, 9), (3, 2, 3)
    x, core, fs = planted(shape, ranks, 2)
    exact = oracle.update_factor(shape, ranks, core, fs, 0.01, x, 1)
    errs = []
    for s in (500, 50000):
        a, _, _ = oracle.update_factor_sketched(shape, ranks, core, fs, 0.01, x, 1, s, 7)
        errs.append(np.linalg.norm(a - exact) / np.linalg.norm(exact))
    assert errs[1] < errs[0] and errs[1] < 1e-3


def test_als_factor_sketch_deterministic(oracle):
    x, _, _ = planted((10, 9, 8), (2, 2, 2), 3)
    kw = dict(lam=0.01, sketched_core=1, sample_count_override=2000, max_iterations=2,
              tolerance=0.0, record_history=1, seed=4, factor_samples=800)
    a = oracle.als(x, (2, 2, 2), **kw)
    b = oracle.als(x, (2, 2, 2), **kw)
    assert a["history"] == b["history"]
    c = oracle.als(x, (2, 2, 2), **dict(kw, factor_samples=0))
    assert a["history"] != c["history"]
