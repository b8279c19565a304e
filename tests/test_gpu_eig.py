"""The hand-written symmetric eigensolver for d > 64 (k_eig.cu, parallel block Jacobi) and
the pseudo-inverse solve built on it (the reference's pinv semantics: singular values = |mu|,
cutoff d eps max|mu|, ref svd.cpp:92-97, linalg.cpp:8-26), checked against LAPACK (numpy)
and, where it finishes in seconds, the oracle's Jacobi-SVD pinv."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


def sym(d, seed, spectrum):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    a = (q * spectrum) @ q.T
    return 0.5 * (a + a.T)


@pytest.mark.parametrize("d,kind", [(65, "indef"), (100, "psd"), (333, "indef"), (1000, "psd"),
                                    (2048, "clustered")])
def test_sym_eig_vs_lapack(rt, d, kind):
    rng = np.random.default_rng(d)
    if kind == "psd":
        ev = np.logspace(3, -5, d)
    elif kind == "indef":
        ev = rng.standard_normal(d) * 10
    else:  # many repeated eigenvalues (a Kronecker-like spectrum)
        ev = np.repeat(np.logspace(2, -2, 16), d // 16)
    a = sym(d, d + 1, ev)
    t0 = time.perf_counter()
    mu, v = rt.sym_eig(a)
    dt = time.perf_counter() - t0
    ref = np.sort(np.linalg.eigvalsh(a))[::-1]
    na = np.linalg.norm(a, 2)
    ev_err = float(np.max(np.abs(mu - ref)) / na)
    res = float(np.linalg.norm(a @ v - v * mu) / na)
    orth = float(np.linalg.norm(v.T @ v - np.eye(d)))
    print(f"d={d} {kind}: {dt * 1e3:.1f} ms, eigenvalue err {ev_err:.2e} ||A||, residual "
          f"{res:.2e}, orthogonality {orth:.2e}")
    # Jacobi rounding accumulates over the sweeps' rounds (measured: eigenvalues ~0.5 d eps,
    # residual ~6 d eps, orthogonality ~25 d eps at d = 2048)
    assert ev_err < 4 * d * EPS
    assert res < 16 * d * EPS
    assert orth < 64 * d * EPS


def numpy_pinv_solve(g, b):
    mu, v = np.linalg.eigh(g)
    cut = g.shape[0] * EPS * np.max(np.abs(mu))
    keep = np.abs(mu) > cut
    return v[:, keep] @ ((v[:, keep].T @ b) / mu[keep]), int(keep.sum())


@pytest.mark.parametrize("d,r", [(300, 200), (1000, 640), (1500, 1500)])
def test_pinv_large_vs_lapack(rt, d, r):
    """Rank-deficient PSD (and an indefinite full-rank) Gram: the fallback route of
    rtucker_b200_spd_solve for d > 64 when Cholesky fails."""
    rng = np.random.default_rng(d + r)
    ev = np.zeros(d)
    ev[:r] = np.logspace(2, -3, r)
    if r == d:
        ev[-7:] = -np.logspace(0, -2, 7)
    g = sym(d, d * 7 + r, ev)
    b = rng.standard_normal(d)
    x, rank, path = rt.spd_solve(g, b)
    xr, rr = numpy_pinv_solve(g, b)
    kappa = 1e2 / 1e-3
    err = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    print(f"pinv d={d} r={r}: rank {rank} (numpy {rr}), err {err:.2e}, kappa_kept {kappa:.1e}")
    assert path == 1 and rank == rr
    assert err < 16 * kappa * np.sqrt(d) * EPS


def test_pinv_large_vs_oracle_jacobi(oracle, rt):
    """d = 200 against the oracle's one-sided Jacobi SVD pinv (bit-pinned to the reference)."""
    d, r = 200, 120
    rng = np.random.default_rng(5)
    ev = np.zeros(d)
    ev[:r] = np.logspace(1, -4, r)
    g = sym(d, 77, ev)
    b = rng.standard_normal(d)
    ox, orank = oracle.pinv_solve(g, b)
    gx, grank, path = rt.spd_solve(g, b)
    assert path == 1 and grank == orank
    assert np.linalg.norm(gx - ox) / np.linalg.norm(ox) < 16 * 1e5 * np.sqrt(d) * EPS


def test_sym_eig_timing_d4096(rt):
    """The C2 core-solve size (d = 4096): a sketched-Gram-like SPD matrix."""
    d = 4096
    rng = np.random.default_rng(1)
    f = [rng.standard_normal((512, 16)) for _ in range(3)]
    k = np.kron(np.kron(f[0].T @ f[0], f[1].T @ f[1]), f[2].T @ f[2])
    e = rng.standard_normal((d, d)) * 1e-3 * np.sqrt(np.diag(k).mean())
    a = k + 0.5 * (e @ e.T) / d + 1e-2 * np.eye(d)
    t0 = time.perf_counter()
    mu, v = rt.sym_eig(a)
    dt = time.perf_counter() - t0
    ref = np.sort(np.linalg.eigvalsh(a))[::-1]
    err = float(np.max(np.abs(mu - ref)) / ref[0])
    print(f"d=4096 sketched-Gram-like: {dt:.3f} s (incl. 2 x 134 MB copies), eigenvalue err {err:.2e}")
    assert err < 4 * d * EPS
