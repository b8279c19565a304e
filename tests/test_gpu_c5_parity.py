"""Parity of the rank-32 kernels the C5 line runs (BASELINE configs[4]: R = (32,32,32), d = 32768).

  * rung 3: the sketched Gram/RHS of k_vech_bucket6 (144 x 144 tiles of the 528-pair vech
    tables) + the contraction, from the oracle's own draws, vs orc_kron_sketch_normal_eq at
    ranks (4, 32, 32) (d = 4096, where the oracle's row-by-row stream finishes in seconds)
                                                                  (ref sketch_ridge.cpp:105-128)
  * the large-d core solve (PCG on the blocked Gram) at R_2 = R_3 = 32 vs a cuSOLVER solve of
    an independently built FP64 Gram of the same draws (the reference's Jacobi SVD at
    d = 8192 .. 32768 takes days)                                 (ref sketch_ridge.cpp:130-139)

Bars are c * kappa * eps with kappa printed, as in test_gpu_c2_parity.py.
"""
import numpy as np
import pytest

from tests.bars import frel
from tests.test_gpu_c2_parity import _oracle_draws, _torch_normal_eq, model, planted

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


@pytest.mark.parametrize("shape,ranks", [((16, 64, 48), (4, 32, 32)),
                                         ((12, 40, 64), (3, 20, 32))])
def test_normal_equations_r32_from_oracle_sketch(oracle, rt, shape, ranks):
    x = planted(shape, ranks, seed=51)
    lam, s = 1e-2, 4000
    core, factors = model(oracle, shape, ranks, "uniform", 13)
    idx, w = _oracle_draws(oracle, shape, ranks, factors, 77, s)
    b6 = rt.variant_count("k_vech_bucket6")
    gg, grhs = rt.kron_normal_eq(shape, ranks, factors, x, lam, idx, w)
    assert rt.variant_count("k_vech_bucket6") == b6 + 1, "large-rank Gram did not take bucket6"
    og, orhs = oracle.kron_normal_eq(shape, ranks, factors, x, lam, idx, w)
    dg = np.sqrt(np.outer(np.diag(og), np.diag(og)))
    eg = float(np.max(np.abs(gg - og) / dg))
    er = float(np.linalg.norm(grhs - orhs) / np.linalg.norm(orhs))
    print(f"{ranks} rung 3: Gram {eg:.3e} (normalised), rhs {er:.3e}")
    assert eg < 1e-12 and er < 1e-12


def _kappa_spd(torch, G, L, iters=60):
    """kappa_2 of an SPD matrix by power iteration on G (largest eigenvalue) and on G^-1
    through its Cholesky factor (smallest): a d^2 per step instead of an O(d^3) eigensolve
    (d = 32768); accurate to a few percent, which is all a c * kappa * eps bar needs."""
    g = torch.Generator(device=G.device).manual_seed(0)
    v = torch.randn(G.shape[0], 1, dtype=G.dtype, device=G.device, generator=g)
    u = v.clone()
    hi = lo = 1.0
    for _ in range(iters):
        v = G @ v
        hi = float(v.norm())
        v /= hi
        u = torch.cholesky_solve(u, L)
        lo = float(u.norm())
        u /= lo
    return hi * lo


@pytest.mark.parametrize("shape,ranks,s", [((40, 64, 48), (8, 32, 32), 60000),
                                           ((64, 64, 48), (32, 32, 32), 120000)])
def test_pcg_r32_core_solve_vs_cusolver(oracle, rt, shape, ranks, s):
    torch = pytest.importorskip("torch")
    x = planted(shape, ranks, seed=52)
    lam = 1e-2
    core, factors = model(oracle, shape, ranks, "normal", 17)
    xt = rt.Tensor.from_numpy(x)
    gcore, gidx, gw = rt.update_core_sketched(xt, rt.Model(core, factors, lam), s, 5)
    oidx, ow = _oracle_draws(oracle, shape, ranks, factors, 5, s)
    assert np.array_equal(gidx, oidx)
    G, b = _torch_normal_eq(shape, ranks, factors, x, lam, gidx, gw)
    L = torch.linalg.cholesky(G)
    xs = torch.cholesky_solve(b[:, None], L)[:, 0].cpu().numpy()
    kappa = _kappa_spd(torch, G, L)
    del G, L
    torch.cuda.empty_cache()
    err = frel(gcore, xs)
    print(f"{ranks} d={int(np.prod(ranks))} core: kappa {kappa:.3e} err {err:.3e} "
          f"err/(kappa eps) {err / (kappa * EPS):.3g}")
    assert err < 64 * kappa * EPS, (kappa, err)


def _torch_update_factor(torch, x, core, factors, lam, mode):
    """Independent FP64 update_factor on the GPU (ref tucker.cpp:70-89): A_n = X_(n) K^T
    (K K^T + lam I)^-1 with K = G_(n) (kron_{m != n} A_m)^T, formed by mode products."""
    dev = "cuda"
    y = torch.from_numpy(x).to(dev)
    A = [torch.from_numpy(np.ascontiguousarray(f)).to(dev) for f in factors]
    G = torch.from_numpy(np.ascontiguousarray(core)).to(dev)
    q = G
    for m in range(len(factors)):
        if m == mode:
            continue
        y = torch.movedim(torch.tensordot(A[m].T, y, dims=([1], [m])), 0, m)
        q = torch.movedim(torch.tensordot(A[m].T @ A[m], q, dims=([1], [m])), 0, m)
    yn = torch.movedim(y, mode, 0).reshape(x.shape[mode], -1)
    gn = torch.movedim(G, mode, 0).reshape(core.shape[mode], -1)
    qn = torch.movedim(q, mode, 0).reshape(core.shape[mode], -1)
    M = yn @ gn.T
    kk = gn @ qn.T + lam * torch.eye(core.shape[mode], dtype=torch.float64, device=dev)
    return torch.linalg.solve(kk, M.T).T.cpu().numpy()


def test_update_factor_f3_r32_mid5(oracle, rt):
    """Rank 32 with I_1 = 384 (beyond k_ttm_mid2's shared memory, as C5's I_1 = 512): the F_3
    projection X x_1 A_1^T takes k_ttm_mid5<32> (16-row TMA boxes, five stages); all three
    modes vs an independent FP64 update_factor."""
    from tests.bars import factor_bar, kkt_kappa
    torch = pytest.importorskip("torch")
    shape, ranks, lam = (384, 40, 2048), (32, 32, 32), 1e-2
    x = planted(shape, ranks, seed=53)
    core, factors = model(oracle, shape, ranks, "normal", 19)
    xt = rt.Tensor.from_numpy(x)
    m = rt.Model(core, factors, lam)
    for mode in (1, 2, 3):
        m5 = rt.variant_count("k_ttm_mid5<32>")
        g = rt.update_factor(xt, m, mode)
        if mode == 3:
            assert rt.variant_count("k_ttm_mid5<32>") == m5 + 1, "F3 did not take k_ttm_mid5<32>"
        o = _torch_update_factor(torch, x, core, factors, lam, mode - 1)
        kappa = kkt_kappa(core, factors, mode - 1, lam)
        err = frel(g, o)
        bar = factor_bar(kappa, shape, mode - 1)
        print(f"R=32 F{mode}: kappa {kappa:.3e} err {err:.3e} bar {bar:.3e}")
        assert err < bar, (mode, kappa, err)


def _torch_normal_eq_nway(shape, ranks, factors, x, lam, idx, w):
    """N-way version of test_gpu_c2_parity._torch_normal_eq (independent FP64 Gram/RHS)."""
    import torch
    dev = "cuda"
    d = int(np.prod(ranks))
    total = int(np.prod(shape))
    A = [torch.from_numpy(np.ascontiguousarray(f)).to(dev) for f in factors]
    xi = torch.from_numpy(x.ravel()).to(dev)
    ti = torch.from_numpy(idx.astype(np.int64)).to(dev)
    tw = torch.from_numpy(w).to(dev)
    data = ti < total
    i, wd = ti[data], tw[data]
    G = torch.zeros((d, d), dtype=torch.float64, device=dev)
    rhs = torch.zeros(d, dtype=torch.float64, device=dev)
    for c in range(0, i.numel(), 4096):
        ic, wc = i[c:c + 4096], wd[c:c + 4096]
        rem, js = ic.clone(), []
        for I in reversed(shape):
            js.append(rem % I)
            rem = rem // I
        js = js[::-1]
        r = A[0][js[0]]
        for n in range(1, len(shape)):
            r = (r[:, :, None] * A[n][js[n]][:, None, :]).reshape(r.shape[0], -1)
        r = r * wc[:, None]
        G += r.T @ r
        rhs += r.T @ (wc * xi[ic])
    j = ti[~data] - total
    G.view(-1).index_put_((j * d + j,), lam * tw[~data] ** 2, accumulate=True)
    return G, rhs


def test_pcg_order4_large_d_vs_cusolver(oracle, rt):
    """The order-4 large-d core solve (C3's: k_pcg_dv with the tiled order-4 matvec,
    d = 10^4) vs a cuSOLVER Cholesky solve of an independently built Gram of the same draws."""
    torch = pytest.importorskip("torch")
    shape, ranks, s, lam = (24, 22, 20, 18), (10, 10, 10, 10), 200000, 0.1
    x = planted(shape, ranks, seed=54)
    core, factors = model(oracle, shape, ranks, "normal", 23)
    dv, t4 = rt.variant_count("k_pcg_dv"), rt.variant_count("k_pcg_t4")
    gcore, gidx, gw = rt.update_core_sketched(rt.Tensor.from_numpy(x),
                                              rt.Model(core, factors, lam), s, 8)
    assert rt.variant_count("k_pcg_dv") == dv + 1 and rt.variant_count("k_pcg_t4") == t4 + 1
    G, b = _torch_normal_eq_nway(shape, ranks, factors, x, lam, gidx, gw)
    L = torch.linalg.cholesky(G)
    xs = torch.cholesky_solve(b[:, None], L)[:, 0].cpu().numpy()
    kappa = _kappa_spd(torch, G, L)
    del G, L
    torch.cuda.empty_cache()
    err = frel(gcore, xs)
    print(f"order 4 d=10^4 core: kappa {kappa:.3e} err {err:.3e} err/(kappa eps) "
          f"{err / (kappa * EPS):.3g}")
    assert err < 64 * kappa * EPS, (kappa, err)


@pytest.mark.parametrize("shape,ranks", [((40, 24, 24), (20, 12, 12)), ((36, 40, 36), (24, 20, 16))])
def test_normal_equations_large_r1_contraction(oracle, rt, shape, ranks):
    """Rung 3 with m_1 above one CTA's 136 rows (k_vech_contract3 in row blocks, as C5's
    m_1 = 528 runs it) vs the oracle's row-by-row stream."""
    x = planted(shape, ranks, seed=55)
    lam, s = 1e-2, 3000
    core, factors = model(oracle, shape, ranks, "uniform", 29)
    idx, w = _oracle_draws(oracle, shape, ranks, factors, 91, s)
    before = rt.variant_count("k_vech_contract3_rows")
    gg, grhs = rt.kron_normal_eq(shape, ranks, factors, x, lam, idx, w)
    assert rt.variant_count("k_vech_contract3_rows") == before + 1
    og, orhs = oracle.kron_normal_eq(shape, ranks, factors, x, lam, idx, w)
    dg = np.sqrt(np.outer(np.diag(og), np.diag(og)))
    eg = float(np.max(np.abs(gg - og) / dg))
    er = float(np.linalg.norm(grhs - orhs) / np.linalg.norm(orhs))
    print(f"{ranks} rung 3 (row-blocked contraction): Gram {eg:.3e}, rhs {er:.3e}")
    assert eg < 1e-12 and er < 1e-12
