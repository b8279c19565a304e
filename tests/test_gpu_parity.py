"""GPU parity tests: the CUDA path (through the C ABI) against the oracle.

Parity ladder of SURVEY.md 8(c):
  rung 1  sampled indices bit-exact given the same CDFs and seed
  rung 2  per-mode leverage scores within 1e-9 (relative to max score)
  rung 3  Gram/RHS from the same RowSketch within 1e-9 (normalised entries)
  rung 4  solve of the same Gram within c * kappa * eps
  rung 5  end to end (factors, core, loss) within a small multiple of the
          reference's own noise floor (reordered sums move it by ~kappa*eps)
The oracle (oracle/rtucker_oracle.c) is bit-identical to the compiled
reference (tests/test_oracle_pin.py).
"""
import numpy as np
import pytest

from tests.bars import core_exact_kappa, factor_bar, frel, kkt_kappa

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


def planted(shape, ranks, noise=0.01, seed=0):
    """BASELINE-style input: N(0,1) core/factors, dense noise at noise*||X||/sqrt(N)."""
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    factors = [rng.standard_normal((i, r)) for i, r in zip(shape, ranks)]
    x = core
    for n, f in enumerate(factors):
        x = np.moveaxis(np.tensordot(f, x, axes=(1, n)), 0, n)
    sigma = noise * np.linalg.norm(x) / np.sqrt(x.size)
    return x + sigma * rng.standard_normal(x.shape)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def random_model(oracle, shape, ranks, seed):
    core, factors = oracle.random_model(shape, ranks, seed)
    return core.reshape(ranks), factors


# ---------------------------------------------------------------- rung 2
@pytest.mark.parametrize("rows,cols,kind", [(100, 5, "uniform"), (512, 16, "normal"),
                                            (160, 10, "pareto"), (7, 7, "normal"),
                                            (33, 1, "uniform")])
def test_factor_scores(oracle, rt, rows, cols, kind):
    rng = np.random.default_rng(rows * 31 + cols)
    if kind == "uniform":
        f = rng.random((rows, cols))
    elif kind == "normal":
        f = rng.standard_normal((rows, cols))
    else:
        f = rng.standard_normal((rows, cols)) * (rng.pareto(1.5, rows) + 1.0)[:, None]
    sc, cdf, tot, rank = rt.factor_scores(f)
    osc, ocdf, otot, orank = oracle.factor_scores(f)
    assert rank == orank
    assert rel(sc, osc) < 1e-9
    assert rel(cdf, ocdf) < 1e-9
    assert abs(tot - otot) / otot < 1e-9


def test_factor_scores_zero_factor(rt):
    sc, cdf, tot, rank = rt.factor_scores(np.zeros((9, 3)))
    assert rank == 0 and tot == 0.0 and not sc.any()


# ---------------------------------------------------------------- rung 1
@pytest.mark.parametrize("shape,ranks,s,seed", [((100, 100, 100), (5, 5, 5), 20000, 7),
                                                 ((30, 20, 10, 8), (3, 2, 4, 2), 5000, 11),
                                                 ((64,), (5,), 3000, 3),
                                                 ((40, 50), (4, 6), 7777, 99),
                                                 # > 8192 sub-chunks: two-level map composition
                                                 ((100, 100, 100), (5, 5, 5), 1000000, 5),
                                                 ((2048, 2048), (32, 32), 2000000, 1)])
def test_draws_bit_exact_given_reference_cdfs(oracle, rt, shape, ranks, s, seed):
    rng = np.random.default_rng(seed)
    fs = [rng.random((i, r)) for i, r in zip(shape, ranks)]
    scs, cdfs, sums = [], [], []
    for f in fs:
        sc, cdf, tot, _ = oracle.factor_scores(f)
        scs.append(sc)
        cdfs.append(cdf)
        sums.append(tot)
    d = int(np.prod(ranks))
    oidx, ow, _ = oracle.kron_draw(shape, d, scs, cdfs, sums, seed, s)
    gidx, gw = rt.kron_draw(shape, d, scs, cdfs, sums, seed, s)
    assert np.array_equal(oidx, gidx)
    assert np.array_equal(ow, gw)  # same IEEE ops -> bitwise weights


_SERIAL_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from oracle.oracle import Oracle
from paper_2107_10654_b200 import rtucker as rt
o = Oracle()
shape, ranks, s, seed = (60, 50, 40), (4, 3, 5), 30000, 13
rng = np.random.default_rng(seed)
fs = [rng.random((i, r)) for i, r in zip(shape, ranks)]
scs, cdfs, sums = [], [], []
for f in fs:
    sc, cdf, tot, _ = o.factor_scores(f)
    scs.append(sc); cdfs.append(cdf); sums.append(tot)
d = int(np.prod(ranks))
oidx, ow, _ = o.kron_draw(shape, d, scs, cdfs, sums, seed, s)
gidx, gw = rt.kron_draw(shape, d, scs, cdfs, sums, seed, s)
assert np.array_equal(oidx, gidx) and np.array_equal(ow, gw)
print("serial walk bit-exact", len(gidx))
"""


def test_draws_serial_walk_bit_exact():
    """The draw decoder's exact serial fallback (k_draw_scan with the overflow flag: the path a
    next_below rejection takes) forced by RTB_DRAW_FORCE_SERIAL, in a child process (the
    library reads the switch once): bit-exact vs the oracle like the parallel decode."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RTB_DRAW_FORCE_SERIAL="1")
    r = subprocess.run([sys.executable, "-c", _SERIAL_SCRIPT.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bit-exact" in r.stdout


# ---------------------------------------------------------------- rung 3
@pytest.mark.parametrize("shape,ranks,lam,s", [((30, 25, 20), (4, 3, 5), 1e-3, 4000),
                                                ((20, 18, 16, 12), (3, 2, 2, 3), 0.1, 3000),
                                                # order 4 with draws >> (i1, i2) pairs: the
                                                # (i1, i2)-bucketed path of k_gram.cu
                                                ((16, 14, 12, 10), (4, 3, 5, 2), 0.05, 20000),
                                                ((12, 10, 9, 8), (3, 3, 3, 3), 0.1, 600),
                                                ((50, 40), (6, 5), 1e-2, 2000),
                                                ((70,), (9,), 1e-2, 500)])
def test_normal_equations_from_reference_sketch(oracle, rt, shape, ranks, lam, s):
    x = planted(shape, ranks, seed=3)
    core, factors = random_model(oracle, shape, ranks, 5)
    _, idx, w, _ = oracle.update_core_fast(shape, ranks, core, factors, lam, x, s, 1234)
    og, orhs = oracle.kron_normal_eq(shape, ranks, factors, x, lam, idx, w)
    c2 = rt.variant_count("k_vech_contract2")
    gg, grhs = rt.kron_normal_eq(shape, ranks, factors, x, lam, idx, w)
    if shape == (30, 25, 20):  # small vech blocks: the cp.async contraction k_vech_contract2
        assert rt.variant_count("k_vech_contract2") == c2 + 1
    dg = np.sqrt(np.outer(np.diag(og), np.diag(og)))
    assert np.max(np.abs(gg - og) / dg) < 1e-9
    assert np.linalg.norm(grhs - orhs) / np.linalg.norm(orhs) < 1e-9


# ---------------------------------------------------------------- rung 4
@pytest.mark.parametrize("d", [8, 64, 125, 200])
def test_spd_solve_on_reference_gram(oracle, rt, d):
    rng = np.random.default_rng(d)
    a = rng.standard_normal((3 * d, d))
    g = a.T @ a + 1e-3 * np.eye(d)
    b = rng.standard_normal(d)
    ox, orank = oracle.pinv_solve(g, b)
    gx, grank, path = rt.spd_solve(g, b)
    kappa = np.linalg.cond(g)
    assert grank == orank == d
    assert np.linalg.norm(gx - ox) / np.linalg.norm(ox) < 100 * kappa * EPS


@pytest.mark.parametrize("d,kappa_target", [(1000, 1e6), (4096, 1e8), (4100, 1e4)])
def test_spd_solve_large(rt, d, kappa_target):
    """Large SPD systems (the C2 core solve is d = 4096): checked against LAPACK
    (numpy) since the oracle's Jacobi SVD takes hours at this size."""
    rng = np.random.default_rng(d)
    q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    ev = np.logspace(0, -np.log10(kappa_target), d)
    g = (q * ev) @ q.T
    g = 0.5 * (g + g.T)
    b = rng.standard_normal(d)
    xr = np.linalg.solve(g, b)
    gx, grank, path = rt.spd_solve(g, b)
    assert path == 0 and grank == d
    assert np.linalg.norm(gx - xr) / np.linalg.norm(xr) < 100 * kappa_target * EPS * np.sqrt(d)


def test_spd_solve_rank_deficient_small(oracle, rt):
    rng = np.random.default_rng(1)
    a = rng.standard_normal((20, 3))
    g = np.zeros((6, 6))
    g[:3, :3] = a.T @ a  # rank 3 PSD
    b = rng.standard_normal(6)
    ox, orank = oracle.pinv_solve(g, b)
    gx, grank, path = rt.spd_solve(g, b)
    assert path == 1 and grank == orank == 3
    assert np.linalg.norm(gx - ox) / np.linalg.norm(ox) < 1e-9


@pytest.mark.parametrize("d,r", [(100, 60), (150, 150)])
def test_spd_solve_rank_deficient_large(oracle, rt, d, r):
    """d > 64 pinv fallback (k_pinv.cu): rank-deficient PSD Gram, checked against the
    oracle's Jacobi-SVD pinv with the reference cutoff (ref linalg.cpp:8-26, svd.cpp:92-97);
    (150, 150): a full-rank indefinite symmetric matrix (Cholesky fails; the SVD pinv keeps
    the negative eigenvalues as singular values |mu|)."""
    rng = np.random.default_rng(d + r)
    q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    ev = np.zeros(d)
    ev[:r] = np.logspace(2, -2, r)
    if r == d:
        ev[-5:] = -np.logspace(-1, -3, 5)
    g = (q * ev) @ q.T
    g = 0.5 * (g + g.T)
    b = rng.standard_normal(d)
    ox, orank = oracle.pinv_solve(g, b)
    gx, grank, path = rt.spd_solve(g, b)
    assert path == 1
    assert grank == orank
    assert np.linalg.norm(gx - ox) / np.linalg.norm(ox) < 1e-9


# ---------------------------------------------------------------- model steps
CASES = [((12, 10, 8), (3, 2, 4), 0.01), ((30, 30, 30), (4, 4, 4), 1e-3),
         ((9, 8, 7, 6), (2, 3, 2, 2), 0.05), ((40, 35), (5, 4), 1e-2), ((50,), (4,), 1e-2)]


@pytest.mark.parametrize("shape,ranks,lam", CASES)
def test_update_factor(oracle, rt, shape, ranks, lam):
    x = planted(shape, ranks, seed=1)
    core, factors = random_model(oracle, shape, ranks, 2)
    xt = rt.Tensor.from_numpy(x)
    m = rt.Model(core, factors, lam)
    for mode in range(1, len(shape) + 1):
        g = rt.update_factor(xt, m, mode)
        o = oracle.update_factor(shape, ranks, core, factors, lam, x, mode)
        kappa = kkt_kappa(core, factors, mode - 1, lam)
        err, bar = frel(g, o), factor_bar(kappa, shape, mode - 1)
        print(f"update_factor {shape} F{mode}: kappa {kappa:.3e} err {err:.3e} bar {bar:.3e}")
        assert err < bar, (mode, kappa, err)


@pytest.mark.parametrize("shape,ranks,lam", CASES)
def test_update_core_exact(oracle, rt, shape, ranks, lam):
    x = planted(shape, ranks, seed=4)
    core, factors = random_model(oracle, shape, ranks, 6)
    g = rt.update_core_exact(rt.Tensor.from_numpy(x), rt.Model(core, factors, lam))
    o = oracle.update_core_exact(shape, ranks, core, factors, lam, x)
    kappa = core_exact_kappa(factors)
    err, bar = frel(g, o), 64 * (kappa + np.sqrt(x.size)) * EPS
    print(f"core_exact {shape}: kappa {kappa:.3e} err {err:.3e} bar {bar:.3e}")
    assert err < bar, (kappa, err)


@pytest.mark.parametrize("shape,ranks,lam", CASES)
def test_loss(oracle, rt, shape, ranks, lam):
    x = planted(shape, ranks, seed=8)
    core, factors = random_model(oracle, shape, ranks, 9)
    gl, gr = rt.loss(rt.Tensor.from_numpy(x), rt.Model(core, factors, lam))
    ol, orr = oracle.tucker_loss(shape, ranks, core, factors, lam, x)
    assert abs(gl - ol) / ol < 1e-12
    assert abs(gr - orr) / orr < 1e-12


@pytest.mark.parametrize("shape,ranks,lam,s", [((30, 30, 30), (4, 4, 4), 1e-3, 6000),
                                                ((12, 10, 8), (3, 2, 4), 0.01, 3000),
                                                ((9, 8, 7, 6), (2, 3, 2, 2), 0.05, 2000),
                                                ((64, 60), (9, 7), 1e-2, 3000),
                                                ((50, 40), (6, 5), 1e-2, 2000)])
def test_update_core_sketched(oracle, rt, shape, ranks, lam, s):
    x = planted(shape, ranks, seed=10)
    core, factors = random_model(oracle, shape, ranks, 12)
    gcore, gidx, gw = rt.update_core_sketched(rt.Tensor.from_numpy(x),
                                              rt.Model(core, factors, lam), s, 777)
    ocore, oidx, ow, _ = oracle.update_core_fast(shape, ranks, core, factors, lam, x, s, 777)
    assert np.array_equal(gidx, oidx)      # no index flips from the score route
    assert rel(gw, ow) < 1e-12
    og, _ = oracle.kron_normal_eq(shape, ranks, factors, x, lam, oidx, ow)
    kappa = np.linalg.cond(og)
    assert rel(gcore, ocore) < max(1e-9, 1e3 * kappa * EPS)


def test_zero_factor_gives_zero_core(oracle, rt):
    shape, ranks = (4, 3, 2), (2, 2, 2)
    x = planted(shape, ranks, seed=2)
    core, factors = random_model(oracle, shape, ranks, 3)
    factors[1] = np.zeros_like(factors[1])
    g, _, _ = rt.update_core_sketched(rt.Tensor.from_numpy(x), rt.Model(core, factors, 0.3), 50, 1)
    assert not g.any()
    g = rt.update_core_exact(rt.Tensor.from_numpy(x), rt.Model(core, factors, 0.3))
    assert not g.any()


# ---------------------------------------------------------------- end to end
@pytest.mark.parametrize("shape,ranks,lam,s,sweeps,tol", [
    ((40, 40, 40), (5, 5, 5), 1e-3, 20000, 5, 1e-5),
    ((20, 18, 16), (3, 3, 3), 1e-2, 5000, 4, 1e-6),
    ((10, 9, 8, 7), (2, 2, 2, 2), 0.05, 3000, 3, 1e-6),
])
def test_als_sketched_end_to_end(oracle, rt, shape, ranks, lam, s, sweeps, tol):
    x = planted(shape, ranks, seed=21)
    o = oracle.als(x, ranks, lam=lam, sketched_core=1, max_iterations=sweeps, tolerance=0.0,
                   sample_count_override=s, record_history=1, seed=3)
    r = rt.als_run(rt.Tensor.from_numpy(x), ranks,
                   rt.options(lam=lam, sketched_core=1, max_iterations=sweeps, tolerance=0.0,
                              sample_count_override=s, record_history=1, seed=3))
    gh = r.history()
    assert [(h[0], h[1]) for h in gh] == [(h[0], h[1]) for h in o["history"]]
    for (gi, gs, gl, grm), (oi, os_, ol, orm) in zip(gh, o["history"]):
        assert abs(gl - ol) / ol < tol, (gi, gs)
    m = r.model()
    xg = oracle.reconstruct(shape, ranks, m.core, m.factors)
    xo = oracle.reconstruct(shape, ranks, o["core"], o["factors"])
    assert np.linalg.norm(xg - xo) / np.linalg.norm(xo) < tol * 10


def test_als_exact_end_to_end(oracle, rt):
    shape, ranks = (15, 14, 13), (3, 3, 3)
    x = planted(shape, ranks, seed=5)
    o = oracle.als(x, ranks, lam=0.01, max_iterations=6, tolerance=0.0, seed=4)
    r = rt.als_run(rt.Tensor.from_numpy(x), ranks,
                   rt.options(lam=0.01, max_iterations=6, tolerance=0.0, seed=4))
    assert r.iterations == 6
    assert abs(r.final_loss - o["final_loss"]) / o["final_loss"] < 1e-9


def test_als_tolerance_stops_like_reference(oracle, rt):
    shape, ranks = (12, 11, 10), (2, 2, 2)
    x = planted(shape, ranks, seed=6)
    o = oracle.als(x, ranks, lam=0.02, max_iterations=50, tolerance=1e-4, seed=1)
    r = rt.als_run(rt.Tensor.from_numpy(x), ranks,
                   rt.options(lam=0.02, max_iterations=50, tolerance=1e-4, seed=1))
    assert r.iterations == o["iterations"]


def test_history_and_timings_shape(rt):
    x = planted((6, 5, 4), (2, 2, 2), seed=1)
    r = rt.als_run(rt.Tensor.from_numpy(x), (2, 2, 2),
                   rt.options(max_iterations=3, record_history=1, tolerance=0.0))
    assert r.iterations == 3
    h = r.history()
    assert len(h) == 12 and h[0][:2] == (1, "F1") and h[3][1] == "Core"
    t = r.timings()
    assert [row[0] for row in t] == ["F1", "F2", "F3", "Core"]
    assert all(row[2] == 3 for row in t)


def test_rejects_bad_ranks(rt):
    x = rt.Tensor.from_numpy(np.ones((4, 4)))
    with pytest.raises(rt.RtuckerError) as e:
        rt.als_run(x, (5, 2))
    assert e.value.code == rt.ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("shape,ranks,lam,s", [((40, 36, 32), (6, 5, 4), 1e-2, 8000),
                                               ((30, 28, 26), (6, 6, 6), 1e-2, 30000),
                                               ((20, 18, 16, 14), (4, 3, 3, 2), 1e-3, 6000),
                                               ((64, 60), (7, 7), 1e-2, 3000)])
def test_pcg_core_solve_matches_cholesky_and_oracle(oracle, rt, shape, ranks, lam, s):
    """Sketched core by Kronecker-preconditioned CG (solver_path 2) vs the Cholesky
    path (core_solver=1) and the reference restatement, sweep by sweep."""
    x = planted(shape, ranks, seed=31)
    kw = dict(lam=lam, sketched_core=1, max_iterations=3, tolerance=0.0,
              sample_count_override=s, record_history=1, seed=9)
    xt = rt.Tensor.from_numpy(x)
    rp = rt.als_run(xt, ranks, rt.options(**kw))
    rc = rt.als_run(xt, ranks, rt.options(**kw), core_solver=1)
    assert rp.sketch_info()["solver_path"] == 2
    assert rp.sketch_info()["pcg_iterations"] > 0
    assert rc.sketch_info()["solver_path"] == 0
    o = oracle.als(x, ranks, **kw)
    for hp, hc, ho in zip(rp.history(), rc.history(), o["history"]):
        assert abs(hp[2] - hc[2]) / hc[2] < 1e-7, hp[:2]
        assert abs(hp[2] - ho[2]) / ho[2] < 1e-6, hp[:2]
    mp, mc = rp.model(), rc.model()
    assert np.linalg.norm(mp.core - mc.core) / np.linalg.norm(mc.core) < 1e-5


@pytest.mark.parametrize("shape,ranks,s", [((64, 64, 64), (16, 16, 16), 200000),
                                          ((80, 70, 60), (12, 10, 14), 100000),
                                          # d beyond shared memory: vectors in global slices
                                          ((40, 36, 32, 30), (10, 10, 10, 8), 400000),
                                          ((48, 44, 40), (24, 20, 18), 400000)])
def test_pcg_matches_cholesky_large_d(rt, shape, ranks, s):
    """d = 4096 / 1680 / 8000 / 8640: CG and Cholesky solve the same sketched system (no
    oracle: the reference's Jacobi SVD at this d takes hours). s is large enough that every
    augmented column is drawn (else G may be singular and CG does not apply)."""
    x = planted(shape, ranks, seed=33)
    kw = dict(lam=1e-2, sketched_core=1, max_iterations=4, tolerance=0.0,
              sample_count_override=s, record_history=1, seed=2)
    xt = rt.Tensor.from_numpy(x)
    rp = rt.als_run(xt, ranks, rt.options(**kw))
    rc = rt.als_run(xt, ranks, rt.options(**kw), core_solver=1)
    assert rp.sketch_info()["solver_path"] == 2
    for hp, hc in zip(rp.history(), rc.history()):
        assert abs(hp[2] - hc[2]) / hc[2] < 1e-7, hp[:2]
    mp, mc = rp.model(), rc.model()
    assert np.linalg.norm(mp.core - mc.core) / np.linalg.norm(mc.core) < 1e-5


def test_loss_near_exact_fit_takes_direct_residual(oracle, rt):
    """Noise-free low-rank data: the residual is ~1e-13 of ||X||^2, where the fast loss
    formula would cancel; the guarded direct pass must give the direct residual of the
    returned model (checked against the single-op direct loss and the reference)."""
    shape, ranks = (14, 12, 10), (3, 3, 3)
    x = planted(shape, ranks, noise=0.0, seed=8)
    kw = dict(lam=1e-9, max_iterations=8, tolerance=0.0, record_history=1, seed=2)
    r = rt.als_run(rt.Tensor.from_numpy(x), ranks, rt.options(**kw))
    m = r.model()
    gl, grm = rt.loss(rt.Tensor.from_numpy(x), m)
    ol, orm = oracle.tucker_loss(shape, ranks, m.core, m.factors, 1e-9, x)
    assert abs(r.final_rmse - grm) <= 1e-9 * grm, (r.final_rmse, grm)
    assert abs(r.final_rmse - orm) <= 1e-6 * orm, (r.final_rmse, orm)
    assert abs(r.final_loss - ol) <= 1e-9 * ol


@pytest.mark.parametrize("shape,ranks,noise", [((40, 36, 32), (5, 4, 6), 0.01),
                                               ((64, 64, 64), (16, 16, 16), 0.01),
                                               ((30, 28, 26, 24), (3, 3, 3, 3), 0.05)])
def test_fast_loss_matches_direct_residual(rt, shape, ranks, noise):
    """Same ALS trajectory, loss by the opt-in fast formula vs the default direct residual
    pass: agreement to ~1e-12 ||X||^2 absolute (bounded here by 1e-7 relative)."""
    x = planted(shape, ranks, noise=noise, seed=9)
    kw = dict(lam=1e-3, sketched_core=1, sample_count_override=20 * int(np.prod(ranks)),
              max_iterations=3, tolerance=0.0, record_history=1, seed=5)
    xt = rt.Tensor.from_numpy(x)
    rf = rt.als_run(xt, ranks, rt.options(**kw), fast_loss=True)
    rd = rt.als_run(xt, ranks, rt.options(**kw))
    for (fi, fs, fl, frm), (di, ds, dl, drm) in zip(rf.history(), rd.history()):
        assert (fi, fs) == (di, ds)
        assert abs(fl - dl) / dl < 1e-7, (fi, fs, fl, dl)
        assert abs(frm - drm) / drm < 1e-7, (fi, fs, frm, drm)


def test_pcg_lambda_dominated_system(rt):
    """lambda far above the smallest eigenvalue of K^T K (here: data scaled down): the
    eigen-form preconditioner (x) A_n^T A_n + lambda I keeps CG fast; the result
    matches the Cholesky path."""
    shape, ranks = (40, 36, 32), (6, 5, 4)
    x = np.random.default_rng(12).standard_normal(shape)  # no structure: a noise fit
    kw = dict(lam=0.5, sketched_core=1, max_iterations=3, tolerance=0.0,
              sample_count_override=6000, record_history=1, seed=4)
    xt = rt.Tensor.from_numpy(x)
    ra = rt.als_run(xt, ranks, rt.options(**kw))
    rc = rt.als_run(xt, ranks, rt.options(**kw), core_solver=1)
    assert ra.sketch_info()["solver_path"] == 2
    assert ra.sketch_info()["pcg_iterations"] < 60
    for ha, hc in zip(ra.history(), rc.history()):
        assert abs(ha[2] - hc[2]) / hc[2] < 1e-9, (ha[:2], ha[2], hc[2])


def test_pcg_split_eigen_form_rank16(rt):
    """The same lambda-dominated regime at ranks (16, 16, 16): the split-role solve
    (k_pcg_split) with the eigen-form preconditioner of its 16 x 16 x 16 path (two
    swizzled fragment passes around the diagonal scaling) matches the Cholesky path."""
    shape, ranks = (64, 64, 64), (16, 16, 16)
    x = np.random.default_rng(13).standard_normal(shape)  # a noise fit: lambda dominates
    # (s = 200,000 puts augmented draws on every diagonal entry, which the split solve
    # needs; this regime was checked to take the eigen form with RTB_PCG_PROF)
    kw = dict(lam=0.5, sketched_core=1, max_iterations=3, tolerance=0.0,
              sample_count_override=200000, record_history=1, seed=5)
    xt = rt.Tensor.from_numpy(x)
    before = rt.variant_count("k_pcg_split")
    ra = rt.als_run(xt, ranks, rt.options(**kw))
    assert rt.variant_count("k_pcg_split") > before
    rc = rt.als_run(xt, ranks, rt.options(**kw), core_solver=1)
    assert ra.sketch_info()["solver_path"] == 2
    for ha, hc in zip(ra.history(), rc.history()):
        assert abs(ha[2] - hc[2]) / hc[2] < 1e-9, (ha[:2], ha[2], hc[2])


# ---------------------------------------------------------------- sweep execution
@pytest.mark.parametrize("shape,ranks,lam,s,fs", [((40, 36, 32), (6, 5, 4), 1e-2, 8000, 0),
                                                 ((64, 64, 64), (16, 16, 16), 1e-2, 200000, 0),
                                                 ((20, 18, 16, 14), (4, 3, 3, 2), 1e-3, 6000, 0),
                                                 ((40, 36, 32), (6, 5, 4), 1e-2, 8000, 3000)])
def test_graph_sweeps_match_eager(rt, shape, ranks, lam, s, fs):
    """From the second sweep on a sweep runs as one CUDA graph launch (device seeds from
    device counters, the core verdict read behind the loss pass); the histories and the
    model must be bitwise those of the kernel-by-kernel path."""
    x = planted(shape, ranks, seed=51)
    # (runs shorter than 16 sweeps stay eager: capturing costs about one sweep)
    kw = dict(lam=lam, sketched_core=1, max_iterations=16, tolerance=0.0,
              sample_count_override=s, record_history=1, seed=8)
    xt = rt.Tensor.from_numpy(x)
    rg = rt.als_run(xt, ranks, rt.options(**kw), factor_samples=fs)
    re = rt.als_run(xt, ranks, rt.options(**kw), factor_samples=fs, graph=False)
    assert rg.graph_sweeps == 15 and re.graph_sweeps == 0
    assert rg.history() == re.history()
    mg, me = rg.model(), re.model()
    assert np.array_equal(mg.core, me.core)
    assert all(np.array_equal(a, b) for a, b in zip(mg.factors, me.factors))
    assert rg.sketch_info() == re.sketch_info()
    tg, te = rg.timings(), re.timings()
    assert [t[0] for t in tg] == [t[0] for t in te] and all(t[2] == 16 for t in tg)


def test_session_sweeps_beyond_max_iterations(rt):
    """History storage grows past max_iterations (sessions run sweeps on demand)."""
    x = planted((12, 10, 8), (2, 2, 2), seed=3)
    opts = rt.options(lam=1e-2, sketched_core=1, max_iterations=2, tolerance=0.0,
                      sample_count_override=2000, record_history=1, seed=1)
    xt = rt.Tensor.from_numpy(x)
    ses = rt.Session(xt, (2, 2, 2), opts)
    for _ in range(7):
        ses.sweeps(3)
    r = ses.result()
    h = r.history()
    assert len(h) == 21 * 4 and h[-1][:2] == (21, "Core")
    ref = rt.als_run(xt, (2, 2, 2), rt.options(lam=1e-2, sketched_core=1, max_iterations=21,
                                              tolerance=0.0, sample_count_override=2000,
                                              record_history=1, seed=1))
    assert h == ref.history()
