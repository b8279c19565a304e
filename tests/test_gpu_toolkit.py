"""The dense ridge toolkit on the GPU (ref capi.cpp:299-362) against the oracle, which is
bit-pinned to the reference (tests/test_oracle_pin.py; the AugmentedSampler draws also to the
reference's own RowSketch, tests/test_oracle_golden.py):
  rtucker_ridge_scores   one-sided Jacobi SVD of A, any shape and lambda  (leverage.cpp:39-52)
  rtucker_solve_ridge    pinv(A^T A + lambda I) A^T b                      (linalg.cpp:28-41)
  rtucker_sketched_ridge AugmentedSampler draws bit-exact, DMMA sketched Gram, solve
                                                  (sampler.cpp:9-57, sketch_ridge.cpp:52-164)
  the factor-score route of the ALS core step for ill-conditioned factors (kronecker.cpp:18-23)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


def mat(n, d, seed, kind="normal"):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, d))
    if kind == "graded":  # columns scaled over 9 orders of magnitude: kappa ~ 1e9
        a *= np.logspace(0, -9, d)
    elif kind == "deficient":  # rank d - 2: two duplicated columns
        a[:, -1] = a[:, 0]
        a[:, -2] = 2.0 * a[:, 1]
    elif kind == "rows":  # heavy-tailed row norms
        a *= (rng.pareto(1.5, n) + 1.0)[:, None]
    return a


@pytest.mark.parametrize("n,d,kind,lam", [(200, 3, "normal", 0.0), (500, 40, "normal", 0.1),
                                          (300, 100, "rows", 1e-3), (1000, 130, "normal", 10.0),
                                          (400, 24, "graded", 0.0), (400, 24, "deficient", 0.0),
                                          (30, 80, "normal", 0.5), (60, 60, "deficient", 1e-2)])
def test_ridge_scores_vs_oracle(oracle, rt, n, d, kind, lam):
    a = mat(n, d, n + d, kind)
    g = rt.ridge_scores(a, lam)
    o = oracle.ridge_scores(a, lam)
    err = float(np.max(np.abs(g - o)) / np.max(np.abs(o)))
    print(f"ridge_scores {n}x{d} {kind} lambda={lam}: err {err:.2e}")
    assert err < 1e-9


def test_ridge_scores_zero_matrix(rt):
    assert not rt.ridge_scores(np.zeros((7, 3)), 0.1).any()


@pytest.mark.parametrize("rows,cols,scale", [(512, 16, 9), (300, 10, 11), (160, 10, 7)])
def test_factor_scores_ill_conditioned_keep_reference_rank(oracle, rt, rows, cols, scale):
    """kappa(A) = 1e7..1e11: the Gram's Cholesky fails, and the rank cut must be the
    reference's, on singular values of A (max(I, R) eps sigma_max), not on Gram eigenvalues
    (which would drop the directions below ~sqrt(eps))."""
    f = mat(rows, cols, rows * 3 + cols) * np.logspace(0, -scale, cols)
    sc, cdf, tot, rank = rt.factor_scores(f)
    osc, ocdf, otot, orank = oracle.factor_scores(f)
    assert rank == orank == cols
    assert np.max(np.abs(sc - osc)) / np.max(osc) < 1e-9
    assert abs(tot - otot) / otot < 1e-9


def test_factor_scores_rank_deficient(oracle, rt):
    f = mat(200, 8, 5, "deficient")
    sc, cdf, tot, rank = rt.factor_scores(f)
    osc, ocdf, otot, orank = oracle.factor_scores(f)
    assert rank == orank == 6
    assert np.max(np.abs(sc - osc)) / np.max(osc) < 1e-9


@pytest.mark.parametrize("n,d,del_,s,seed", [(50, 4, 0.0, 3000, 99), (1000, 30, 29.5, 20000, 3),
                                             (200, 12, 12.0, 5000, 7), (5000, 64, 10.0, 200000, 1)])
def test_aug_draw_bit_exact(oracle, rt, n, d, del_, s, seed):
    cand = np.random.default_rng(n).random(n) ** 3
    cand[::7] = 0.0  # zero-mass rows (the walk-back rule)
    gi, gw = rt.aug_draw(cand, d, del_, seed, s)
    oi, ow = oracle.aug_draw(cand, d, del_, seed, s)
    assert np.array_equal(gi, oi)
    assert np.array_equal(gw, ow)


def test_aug_draw_rejects_bad_scores(rt):
    with pytest.raises(rt.RtuckerError) as e:
        rt.aug_draw(np.array([1.0, -1.0]), 2, 0.0, 1, 10)
    assert e.value.code == rt.ERR_INVALID_ARGUMENT
    with pytest.raises(rt.RtuckerError):
        rt.aug_draw(np.zeros(5), 2, 0.0, 1, 10)


@pytest.mark.parametrize("n,d,lam,s", [(300, 5, 0.1, 4000), (2000, 64, 1e-2, 30000),
                                       (500, 200, 1.0, 20000)])
def test_dense_normal_eq_vs_oracle(oracle, rt, n, d, lam, s):
    a = mat(n, d, 2 * n + d, "rows")
    b = np.random.default_rng(n).standard_normal(n)
    cand = oracle.ridge_scores(a, 0.0)
    idx, w = oracle.aug_draw(cand, d, 0.0, 17, s)
    gg, gr = rt.dense_normal_eq(a, b, lam, idx, w)
    og, orr = oracle.dense_normal_eq(a, b, lam, idx, w)
    dg = np.sqrt(np.outer(np.diag(og), np.diag(og)))
    assert np.max(np.abs(gg - og) / dg) < 1e-12
    assert np.linalg.norm(gr - orr) / np.linalg.norm(orr) < 1e-12


@pytest.mark.parametrize("n,d,lam", [(400, 6, 0.0), (1000, 50, 1e-3), (300, 120, 0.5),
                                     (50, 90, 1e-2)])
def test_solve_ridge_vs_oracle(oracle, rt, n, d, lam):
    a = mat(n, d, n * 5 + d, "rows")
    b = np.random.default_rng(d).standard_normal(n)
    g = rt.solve_ridge(a, b, lam)
    o = oracle.solve_ridge(a, b, lam)
    kappa = np.linalg.cond(a.T @ a + lam * np.eye(d))
    err = np.linalg.norm(g - o) / np.linalg.norm(o)
    print(f"solve_ridge {n}x{d} lambda={lam}: kappa {kappa:.2e} err {err:.2e}")
    assert err < 64 * (kappa + np.sqrt(n)) * EPS


@pytest.mark.parametrize("beta,d,eps_,delta,want", [(0.5, 4, 0.1, 0.1, 68211),
                                                    (1.0, 2, 0.9, 0.001, 30197),
                                                    (1.0, 2, 0.001, 0.5, 16000)])
def test_sample_count_known_answers(rt, beta, d, eps_, delta, want):
    """ref tests/test_sketch_ridge.cpp:17-21, through the library's own formula and through
    rtucker_sketched_ridge with no override (beta' = 1 / (1 + min(1, d - d_eff_lower)))."""
    assert rt.sample_count(beta, d, eps_, delta) == want
    a = mat(40, d, 1)
    b = np.ones(40)
    d_eff = d - 1.0 if beta == 0.5 else float(d)
    _, s, bp = rt.sketched_ridge(a, b, None, 0.1, d_eff, eps_, delta, 0, 5)
    assert s == want and bp == beta


def test_sample_count_rejects_bad_range(rt):
    with pytest.raises(rt.RtuckerError):
        rt.sample_count(0.0, 4, 0.1, 0.1)
    with pytest.raises(rt.RtuckerError):
        rt.sample_count(0.5, 4, 1.5, 0.1)


@pytest.mark.parametrize("n,d,lam,del_,s", [(500, 5, 0.1, 0.0, 5000), (2000, 40, 1e-2, 20.0, 40000),
                                            (800, 100, 1.0, 0.0, 60000)])
def test_sketched_ridge_vs_oracle(oracle, rt, n, d, lam, del_, s):
    a = mat(n, d, 3 * n + d, "rows")
    b = np.random.default_rng(n + 1).standard_normal(n)
    gx, gs, gbp = rt.sketched_ridge(a, b, None, lam, del_, 0.1, 0.1, s, 11)
    ox, os_, obp = oracle.sketched_ridge(a, b, None, lam, del_, 0.1, 0.1, s, 11)
    assert gs == os_ and gbp == obp
    cand = oracle.ridge_scores(a, 0.0)
    idx, w = oracle.aug_draw(cand, d, del_, 11, s)
    og, _ = oracle.dense_normal_eq(a, b, lam, idx, w)
    kappa = np.linalg.cond(og)
    err = np.linalg.norm(gx - ox) / np.linalg.norm(ox)
    print(f"sketched_ridge {n}x{d}: kappa {kappa:.2e} err {err:.2e}")
    assert err < 64 * kappa * EPS
