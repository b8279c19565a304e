"""Parity at the headline configuration (BASELINE configs[1], "C2": 512^3, R = 16, d = 4096).

The kernels the C2 bench line runs are checked here at that configuration, against the
oracle (oracle/rtucker_oracle.c, bit-identical to the compiled reference) where the
oracle finishes in seconds, and against an independent FP64 computation (numpy/LAPACK,
torch cuBLAS) where it does not (the reference's Jacobi SVD at d = 4096 takes hours):

  * exact factor updates at R = 16 through k_ttm_mid3 (the F_3 projection) and
    k_ttm_last3 (T = X x_3 A_3^T), all modes, vs orc_update_factor   (ref tucker.cpp:70-89)
  * the fused loss pass (k_ttm_last3<FUSED>) vs orc_tucker_loss       (ref tucker.cpp:216-229)
  * rung 3 at d = 4096: the sketched Gram/RHS built by k_vech_bucket5 +
    k_vech_contract3 from the oracle's own draws vs orc_kron_sketch_normal_eq
                                                                      (ref sketch_ridge.cpp:105-128)
  * the PCG fast path k_pcg_split (the C2 core solve) vs a LAPACK solve of the same
    sketched system                                                   (ref sketch_ridge.cpp:130-139)

Every floating-point bar is c * kappa * eps with kappa the condition number of the system
the step solves (printed with the measured error), as SURVEY.md 8(c) prescribes. The
variant counters (rtucker_b200_variant_count) prove each test ran the C2 kernel.
"""
import numpy as np
import pytest

from tests.bars import factor_bar, frel, kkt_kappa

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


def planted(shape, ranks, noise=0.01, seed=0, kind="normal"):
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    factors = [rng.standard_normal((i, r)) for i, r in zip(shape, ranks)]
    x = core
    for n, f in enumerate(factors):
        x = np.moveaxis(np.tensordot(f, x, axes=(1, n)), 0, n)
    sigma = noise * np.linalg.norm(x) / np.sqrt(x.size)
    x += sigma * rng.standard_normal(x.shape)
    return np.ascontiguousarray(x)


def model(oracle, shape, ranks, kind, seed):
    if kind == "uniform":  # the reference's own init (tucker.cpp:168-190)
        core, factors = oracle.random_model(shape, ranks, seed)
        return core.reshape(ranks), factors
    rng = np.random.default_rng(seed)  # BASELINE's random-normal init
    return rng.standard_normal(ranks), [rng.standard_normal((i, r)) for i, r in zip(shape, ranks)]


@pytest.fixture(scope="module")
def x_mid():
    """64 x 512 x 512: the F_3 projection X x_1 A_1^T has J = 262144 columns, so it takes
    k_ttm_mid3 exactly as C2 does (gate J % 128 == 0 and O J / 128 >= 4 * 148)."""
    return planted((64, 512, 512), (16, 16, 16), seed=41)


@pytest.fixture(scope="module")
def x_c2():
    return planted((512, 512, 512), (16, 16, 16), seed=42)


@pytest.mark.parametrize("kind", ["uniform", "normal"])
def test_update_factor_r16_all_modes_mid3(oracle, rt, x_mid, kind):
    shape, ranks, lam = x_mid.shape, (16, 16, 16), 1e-2
    core, factors = model(oracle, shape, ranks, kind, 3)
    xt = rt.Tensor.from_numpy(x_mid)
    m = rt.Model(core, factors, lam)
    for mode in (1, 2, 3):
        mid3 = rt.variant_count("k_ttm_mid3")
        g = rt.update_factor(xt, m, mode)
        if mode == 3:
            assert rt.variant_count("k_ttm_mid3") == mid3 + 1, "F3 did not take k_ttm_mid3"
        o = oracle.update_factor(shape, ranks, core, factors, lam, x_mid, mode)
        kappa = kkt_kappa(core, factors, mode - 1, lam)
        err = frel(g, o)
        bar = factor_bar(kappa, shape, mode - 1)
        print(f"[{kind}] F{mode}: kappa {kappa:.3e} err {err:.3e} bar {bar:.3e}")
        assert err < bar, (mode, kappa, err)


def test_update_factor_f3_c2_shape(oracle, rt, x_c2):
    """The literal C2 F_3 (I_1 = 512 rows of A_1 resident in k_ttm_mid3)."""
    shape, ranks, lam = x_c2.shape, (16, 16, 16), 1e-2
    core, factors = model(oracle, shape, ranks, "uniform", 5)
    xt = rt.Tensor.from_numpy(x_c2)
    mid3 = rt.variant_count("k_ttm_mid3")
    g = rt.update_factor(xt, rt.Model(core, factors, lam), 3)
    assert rt.variant_count("k_ttm_mid3") == mid3 + 1
    o = oracle.update_factor(shape, ranks, core, factors, lam, x_c2, 3)
    kappa = kkt_kappa(core, factors, 2, lam)
    err = frel(g, o)
    bar = factor_bar(kappa, shape, 2)
    print(f"C2 F3: kappa {kappa:.3e} err {err:.3e} bar {bar:.3e}")
    assert err < bar


@pytest.mark.parametrize("kind", ["uniform", "normal"])
def test_loss_c2_shape_fused_pass(oracle, rt, x_c2, kind):
    shape, ranks, lam = x_c2.shape, (16, 16, 16), 1e-2
    core, factors = model(oracle, shape, ranks, kind, 7)
    before = rt.variant_count("k_ttm_last3_fused")
    gl, gr = rt.loss(rt.Tensor.from_numpy(x_c2), rt.Model(core, factors, lam))
    assert rt.variant_count("k_ttm_last3_fused") == before + 1
    ol, orr = oracle.tucker_loss(shape, ranks, core, factors, lam, x_c2)
    print(f"[{kind}] loss {gl!r} oracle {ol!r} rel {abs(gl - ol) / ol:.3e}")
    # a sum of 1.3e8 squared residuals in a different order: ~sqrt(n) eps relative
    assert abs(gl - ol) / ol < 1e-11
    assert abs(gr - orr) / orr < 1e-11


def _oracle_draws(oracle, shape, ranks, factors, seed, s):
    scs, cdfs, sums = [], [], []
    for f in factors:
        sc, cdf, tot, _ = oracle.factor_scores(f)
        scs.append(sc)
        cdfs.append(cdf)
        sums.append(tot)
    idx, w, _ = oracle.kron_draw(shape, int(np.prod(ranks)), scs, cdfs, sums, seed, s)
    return idx, w


@pytest.mark.parametrize("i1,kernel", [(32, "k_vech_bucket5"), (512, "k_vech_bucket2<17>")])
def test_normal_equations_d4096_from_oracle_sketch(oracle, rt, x_c2, i1, kernel):
    """Rung 3 at d = 4096, R = 16 (the C2 Gram kernels: k_vech_bucket5 for C2's ~390 draws per
    i_1 bucket, here 32 buckets of ~60 data draws; k_vech_bucket2<17> for short buckets;
    k_vech_table1 + k_vech_contract3, k_vech_blocks), the draws made by the oracle's sampler, the Gram/RHS by
    the oracle's restatement of the reference's row-by-row stream."""
    x = np.ascontiguousarray(x_c2[:i1])
    shape, ranks, lam, s = x.shape, (16, 16, 16), 1e-2, 4000
    core, factors = model(oracle, shape, ranks, "uniform", 9)
    idx, w = _oracle_draws(oracle, shape, ranks, factors, 2024, s)
    b17 = rt.variant_count(kernel)
    c3 = rt.variant_count("k_vech_contract3")
    gg, grhs = rt.kron_normal_eq(shape, ranks, factors, x, lam, idx, w)
    assert rt.variant_count(kernel) == b17 + 1
    assert rt.variant_count("k_vech_contract3") == c3 + 1
    og, orhs = oracle.kron_normal_eq(shape, ranks, factors, x, lam, idx, w)
    dg = np.sqrt(np.outer(np.diag(og), np.diag(og)))
    eg = float(np.max(np.abs(gg - og) / dg))
    er = float(np.linalg.norm(grhs - orhs) / np.linalg.norm(orhs))
    print(f"d=4096 rung 3: Gram {eg:.3e} (normalised), rhs {er:.3e}")
    assert eg < 1e-12 and er < 1e-12


def _torch_normal_eq(shape, ranks, factors, x, lam, idx, w):
    """Independent FP64 Gram/RHS of the augmented Kronecker sketch (cuBLAS DGEMM on dense
    Kronecker rows, chunked): G = sum w^2 r r^T, rhs = sum w^2 x r (ref
    sketch_ridge.cpp:105-128)."""
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
    I2, I3 = shape[1], shape[2]
    for c in range(0, i.numel(), 8192):
        ic, wc = i[c:c + 8192], wd[c:c + 8192]
        i1, i2, i3 = ic // (I2 * I3), (ic // I3) % I2, ic % I3
        r = (A[0][i1][:, :, None, None] * A[1][i2][:, None, :, None] *
             A[2][i3][:, None, None, :]).reshape(-1, d) * wc[:, None]
        G += r.T @ r
        rhs += r.T @ (wc * xi[ic])
    j = ti[~data] - total
    G.view(-1).index_put_((j * d + j,), lam * tw[~data] ** 2, accumulate=True)
    return G, rhs


@pytest.mark.parametrize("kind", ["normal", "uniform"])
def test_pcg_c2_core_solve_vs_lapack(oracle, rt, x_c2, kind):
    """The C2 core update (s = 200,000, d = 4096) through k_pcg_split: the GPU core vs
    x = G^-1 b by LAPACK on an independently built FP64 Gram of the same draws; the Gram
    itself vs the library's normal equations at C2's draw density (~195 data draws per
    i_1 bucket)."""
    torch = pytest.importorskip("torch")
    shape, ranks, lam, s = x_c2.shape, (16, 16, 16), 1e-2, 200000
    core, factors = model(oracle, shape, ranks, kind, 11)
    xt = rt.Tensor.from_numpy(x_c2)
    pcg = rt.variant_count("k_pcg_split")
    gcore, gidx, gw = rt.update_core_sketched(xt, rt.Model(core, factors, lam), s, 99)
    assert rt.variant_count("k_pcg_split") == pcg + 1, "C2 core solve did not take k_pcg_split"
    # the draws are the oracle's: indices bitwise; weights to the scores' agreement (the
    # scores come from the Cholesky route here, the oracle's from the Jacobi SVD: rung 2)
    oidx, ow = _oracle_draws(oracle, shape, ranks, factors, 99, s)
    assert np.array_equal(gidx, oidx)
    assert np.max(np.abs(gw - ow) / ow) < 1e-12
    G, b = _torch_normal_eq(shape, ranks, factors, x_c2, lam, gidx, gw)
    b5 = rt.variant_count("k_vech_bucket5")
    gg, grhs = rt.kron_normal_eq(shape, ranks, factors, x_c2, lam, gidx, gw)
    assert rt.variant_count("k_vech_bucket5") == b5 + 1  # the C2 bucket kernel at C2's density
    Gh, bh = G.cpu().numpy(), b.cpu().numpy()
    dg = np.sqrt(np.outer(np.diag(Gh), np.diag(Gh)))
    eg = float(np.max(np.abs(gg - Gh) / dg))
    er = float(np.linalg.norm(grhs - bh) / np.linalg.norm(bh))
    assert eg < 1e-12 and er < 1e-12, (eg, er)
    ev = torch.linalg.eigvalsh(G).cpu().numpy()
    kappa = float(ev[-1] / ev[0])
    xs = np.linalg.solve(Gh, bh)  # LAPACK dgesv
    err = frel(gcore, xs)
    print(f"[{kind}] C2 core: kappa {kappa:.3e} err {err:.3e} err/(kappa eps) "
          f"{err / (kappa * EPS):.3g}; Gram {eg:.2e} rhs {er:.2e}")
    assert err < 64 * kappa * EPS, (kappa, err)
