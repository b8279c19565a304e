"""Sketched factor updates (perf mode, ext.factor_samples > 0) against the oracle
restatement orc_update_factor_sketched / orc_als_fs.

Not in the reference: parity is pinned to the restatement only.
Both sides draw the same sketch (same seed stream, same sampler) from leverage scores
that agree to ~1e-14 (GPU Cholesky route vs the oracle's Jacobi SVD), so the normal
equations match up to summation order and the losses up to the usual noise floor.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def planted(shape, ranks, noise=0.01, seed=0):
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    factors = [rng.standard_normal((i, r)) for i, r in zip(shape, ranks)]
    x = core
    for n, f in enumerate(factors):
        x = np.moveaxis(np.tensordot(f, x, axes=(1, n)), 0, n)
    sigma = noise * np.linalg.norm(x) / np.sqrt(x.size)
    return x + sigma * rng.standard_normal(x.shape)


def noise_floor(oracle, x, ranks, base, **kw):
    """The restatement's own sensitivity: max relative loss change per history row (running
    max over earlier rows) when x moves by one ulp (two sign patterns)."""
    fl = np.zeros(len(base["history"]))
    for k in range(2):
        sgn = np.random.default_rng(50 + k).choice([-1.0, 1.0], size=x.shape)
        p = oracle.als(x * (1 + 2.0 ** -52 * sgn), ranks, **kw)
        for i, (a, b) in enumerate(zip(p["history"], base["history"])):
            fl[i] = max(fl[i], abs(a[2] - b[2]) / abs(b[2]))
    return np.maximum.accumulate(fl)


@pytest.mark.parametrize("shape,ranks,lam,sc,sf,sweeps", [
    ((30, 28, 26), (4, 4, 4), 1e-2, 8000, 3000, 4),
    ((20, 18, 16), (3, 5, 2), 1e-2, 5000, 2000, 3),
    ((10, 9, 8, 7), (2, 3, 2, 2), 0.05, 3000, 1500, 3),
    ((40, 300), (5, 5), 1e-2, 4000, 2000, 3),
])
def test_als_factor_sketch_matches_oracle(oracle, rt, shape, ranks, lam, sc, sf, sweeps):
    x = planted(shape, ranks, seed=3)
    o = oracle.als(x, ranks, lam=lam, sketched_core=1, max_iterations=sweeps, tolerance=0.0,
                   sample_count_override=sc, record_history=1, seed=5, factor_samples=sf)
    resid = rt.variant_count("k_ttm_last5_resid")
    r = rt.als_run(rt.Tensor.from_numpy(x), ranks,
                   rt.options(lam=lam, sketched_core=1, max_iterations=sweeps, tolerance=0.0,
                              sample_count_override=sc, record_history=1, seed=5),
                   factor_samples=sf)
    if shape[-1] % 2 == 0:  # sketched factor updates never read T: residual-only loss passes
        assert rt.variant_count("k_ttm_last5_resid") > resid
    gh = r.history()
    assert [(h[0], h[1]) for h in gh] == [(h[0], h[1]) for h in o["history"]]
    floor = noise_floor(oracle, x, ranks, o, lam=lam, sketched_core=1, max_iterations=sweeps,
                        tolerance=0.0, sample_count_override=sc, record_history=1, seed=5,
                        factor_samples=sf)
    for k, ((gi, gs, gl, _), (_, _, ol, _)) in enumerate(zip(gh, o["history"])):
        assert abs(gl - ol) / ol <= 30 * floor[k] + 1e-12, (gi, gs, gl, ol, floor[k])


def test_factor_sketch_exact_core(oracle, rt):
    # sketched factors with the exact core update
    shape, ranks = (24, 22, 20), (3, 3, 3)
    x = planted(shape, ranks, seed=8)
    o = oracle.als(x, ranks, lam=1e-2, sketched_core=0, max_iterations=3, tolerance=0.0,
                   record_history=1, seed=2, factor_samples=2500)
    r = rt.als_run(rt.Tensor.from_numpy(x), ranks,
                   rt.options(lam=1e-2, sketched_core=0, max_iterations=3, tolerance=0.0,
                              record_history=1, seed=2), factor_samples=2500)
    floor = noise_floor(oracle, x, ranks, o, lam=1e-2, sketched_core=0, max_iterations=3,
                        tolerance=0.0, record_history=1, seed=2, factor_samples=2500)
    for k, ((gi, gs, gl, _), (_, _, ol, _)) in enumerate(zip(r.history(), o["history"])):
        assert abs(gl - ol) / ol <= 30 * floor[k] + 1e-12, (gi, gs)


def test_factor_sketch_keeps_a_converged_model(rt):
    # subspace-embedding property: from a converged model (exact updates), sweeps with
    # sketched factor updates stay within a few percent of the same objective
    shape, ranks = (40, 40, 40), (4, 4, 4)
    x = planted(shape, ranks, seed=4)
    xt = rt.Tensor.from_numpy(x)
    opts = dict(lam=1e-3, sketched_core=0, tolerance=0.0, seed=1)
    ex = rt.als_run(xt, ranks, rt.options(max_iterations=40, **opts))
    m = ex.model()
    base = rt.als_run(xt, ranks, rt.options(max_iterations=2, **opts), init_model=m)
    sk = rt.als_run(xt, ranks, rt.options(max_iterations=2, **opts), init_model=m,
                    factor_samples=20000)
    assert sk.final_loss <= 1.05 * base.final_loss
