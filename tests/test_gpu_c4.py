"""BASELINE config 4 microbench kernels (rtucker_b200_kron_fiber_sketch): Kronecker-product
sampling of [A2 (x) A3; sqrt(lambda) I], the W x W sketched Gram (order-2 vech machinery) and
the fused fiber-gather RHS (W x I1, FP32 tensor upcast in-kernel), against a direct numpy
evaluation from the same draws and against the oracle's draw stream."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fm", [False, True])
@pytest.mark.parametrize("I1,I2,I3,R2,R3,s", [(48, 40, 36, 4, 4, 3000),
                                               (32, 64, 50, 8, 5, 20000),
                                               (40, 20, 24, 3, 7, 500),
                                               (37, 9, 11, 3, 2, 5000),
                                               (70, 33, 35, 32, 32, 40000),
                                               # sparse canonical: strided gathers, not windows
                                               (16, 64, 64, 3, 4, 200)])
def test_c4_gram_rhs_match_definition(rt, oracle, fm, I1, I2, I3, R2, R3, s):
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(I1, I2, I3, dtype=torch.float32, device="cuda", generator=g)
    xk = x
    if fm:  # fiber-major copy: mode 1 fastest
        xk = torch.empty_like(x)
        rt.tensor_fiber_major(x.data_ptr(), (I1, I2, I3), xk.data_ptr())
        assert torch.equal(xk.view(I2, I3, I1), x.permute(1, 2, 0))
    a2 = torch.randn(I2, R2, dtype=torch.float64, device="cuda", generator=g)
    a3 = torch.randn(I3, R3, dtype=torch.float64, device="cuda", generator=g)
    W = R2 * R3
    gram = torch.zeros(W, W, dtype=torch.float64, device="cuda")
    rhs = torch.zeros(W, I1, dtype=torch.float64, device="cuda")
    lam = 1e-2
    out = rt.kron_fiber_sketch(xk.data_ptr(), (I1, I2, I3), a2.data_ptr(), a3.data_ptr(), R2, R3,
                               lam, s, 11, gram.data_ptr(), rhs.data_ptr(), want_draws=True,
                               fiber_major=fm)
    torch.cuda.synchronize()
    idx, w = out["indices"], out["weights"]
    A2, A3, X = a2.cpu().numpy(), a3.cpu().numpy(), x.cpu().numpy().astype(np.float64)
    # the draw stream is the reference sampler's (scores from the oracle's Jacobi SVD)
    sc, cdf, sums = [], [], []
    for f in (A2, A3):
        a, b, c, _ = oracle.factor_scores(f)
        sc.append(a)
        cdf.append(b)
        sums.append(c)
    oi, ow, _ = oracle.kron_draw([I2, I3], W, sc, cdf, sums, 11, s)
    assert np.mean(oi == idx) > 0.999
    total = I2 * I3
    data = idx < total
    assert out["data_draws"] == int(data.sum())
    # distinct sampled rows (equal draws are merged into one record, weights summed)
    assert out["unique_rows"] == len(np.unique(idx[data]))
    j2, j3 = idx[data] // I3, idx[data] % I3
    Z = np.einsum("tp,tq->tpq", A2[j2], A3[j3]).reshape(-1, W)
    wd = w[data]
    G = (Z * (wd ** 2)[:, None]).T @ Z
    aug = idx[~data] - total
    for j, wt in zip(aug, w[~data]):
        G[j, j] += wt * wt * lam
    Gg = gram.cpu().numpy()
    nrm = np.sqrt(np.outer(np.diag(G), np.diag(G)))
    assert np.max(np.abs(Gg - G) / nrm) < 1e-12
    F = X[:, j2, j3].T  # data draws x I1
    Rr = (Z * (wd ** 2)[:, None]).T @ F
    Rg = rhs.cpu().numpy()
    assert np.linalg.norm(Rg - Rr) / np.linalg.norm(Rr) < 1e-12


def test_c4_gram_only_and_validation(rt):
    import torch
    I2, I3, R = 30, 30, 4
    a2 = torch.randn(I2, R, dtype=torch.float64, device="cuda")
    a3 = torch.randn(I3, R, dtype=torch.float64, device="cuda")
    gram = torch.zeros(R * R, R * R, dtype=torch.float64, device="cuda")
    out = rt.kron_fiber_sketch(None, (8, I2, I3), a2.data_ptr(), a3.data_ptr(), R, R, 1e-2, 2000,
                               1, gram.data_ptr(), None)
    assert out["data_draws"] > 0 and torch.isfinite(gram).all()
    with pytest.raises(rt.RtuckerError):
        rt.kron_fiber_sketch(None, (8, I2, I3), a2.data_ptr(), a3.data_ptr(), 40, R, 1e-2, 10, 1)


def test_c4_rhs_only_and_layouts_agree(rt):
    """RHS without the Gram; canonical X (k_c4_dslab: row windows) and fiber-major X
    (k_c4_dfib: fiber gathers) give the same RHS to rounding (the DMMA k-steps group the
    records differently), each run is deterministic, and the draws are deterministic per seed."""
    import torch
    I1, I2, I3, R = 64, 48, 40, 8
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(I1, I2, I3, dtype=torch.float32, device="cuda", generator=g)
    xf = torch.empty_like(x)
    rt.tensor_fiber_major(x.data_ptr(), (I1, I2, I3), xf.data_ptr())
    a2 = torch.randn(I2, R, dtype=torch.float64, device="cuda", generator=g)
    a3 = torch.randn(I3, R, dtype=torch.float64, device="cuda", generator=g)
    r0 = torch.zeros(R * R, I1, dtype=torch.float64, device="cuda")
    r1 = torch.zeros_like(r0)
    o0 = rt.kron_fiber_sketch(x.data_ptr(), (I1, I2, I3), a2.data_ptr(), a3.data_ptr(), R, R,
                              1e-2, 30000, 9, None, r0.data_ptr())
    o1 = rt.kron_fiber_sketch(xf.data_ptr(), (I1, I2, I3), a2.data_ptr(), a3.data_ptr(), R, R,
                              1e-2, 30000, 9, None, r1.data_ptr(), fiber_major=True)
    torch.cuda.synchronize()
    assert o0["data_draws"] == o1["data_draws"] > 0
    assert o0["unique_rows"] == o1["unique_rows"] > 0
    assert float(torch.linalg.norm(r0 - r1) / torch.linalg.norm(r1)) < 1e-13
    assert torch.count_nonzero(r0) > 0
    r2 = torch.zeros_like(r0)
    rt.kron_fiber_sketch(x.data_ptr(), (I1, I2, I3), a2.data_ptr(), a3.data_ptr(), R, R, 1e-2,
                         30000, 9, None, r2.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(r0, r2)  # run-to-run deterministic


@pytest.mark.parametrize("P", [2, 3])
def test_c4_shards_sum_to_full(rt, P):
    """rtucker_b200_kron_fiber_sketch_shard: the P shards' partial Gram / RHS (run one after
    another on this GPU, summed on the host) equal the unsharded result."""
    import torch
    I1, I2, I3, R2, R3, s = 40, 37, 29, 5, 6, 30000
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randn(I1, I2, I3, dtype=torch.float32, device="cuda", generator=g)
    xf = torch.empty_like(x)
    rt.tensor_fiber_major(x.data_ptr(), (I1, I2, I3), xf.data_ptr())
    a2 = torch.randn(I2, R2, dtype=torch.float64, device="cuda", generator=g)
    a3 = torch.randn(I3, R3, dtype=torch.float64, device="cuda", generator=g)
    W = R2 * R3
    G = torch.zeros(W, W, dtype=torch.float64, device="cuda")
    R = torch.zeros(W, I1, dtype=torch.float64, device="cuda")
    full = rt.kron_fiber_sketch(xf.data_ptr(), (I1, I2, I3), a2.data_ptr(), a3.data_ptr(), R2, R3,
                                1e-2, s, 5, G.data_ptr(), R.data_ptr(), fiber_major=True)
    Gs, Rs = torch.zeros_like(G), torch.zeros_like(R)
    for r in range(P):
        gp, rp = torch.zeros_like(G), torch.zeros_like(R)
        out = rt.kron_fiber_sketch(xf.data_ptr(), (I1, I2, I3), a2.data_ptr(), a3.data_ptr(), R2,
                                   R3, 1e-2, s, 5, gp.data_ptr(), rp.data_ptr(), fiber_major=True,
                                   shard=(r, P))
        assert out["data_draws"] == full["data_draws"]
        Gs += gp
        Rs += rp
    torch.cuda.synchronize()
    dg = torch.sqrt(torch.outer(torch.diag(G), torch.diag(G)))
    assert float(torch.max(torch.abs(Gs - G) / dg)) < 1e-12
    assert float(torch.linalg.norm(Rs - R) / torch.linalg.norm(R)) < 1e-12
    with pytest.raises(rt.RtuckerError):
        rt.kron_fiber_sketch(xf.data_ptr(), (I1, I2, I3), a2.data_ptr(), a3.data_ptr(), R2, R3,
                             1e-2, 100, 5, G.data_ptr(), R.data_ptr(), shard=(3, 3))


@pytest.mark.parametrize("s,seed", [(1, 1), (1, 2), (2, 3), (7, 4), (7, 5)])
def test_c4_tiny_sketches(rt, s, seed):
    """Edge cases of the sort/merge pipeline: a handful of draws, possibly all augmented (no
    distinct data rows: every bucket empty, D = 0) -- Gram and RHS still match the
    definition."""
    import torch
    I1, I2, I3, R2, R3 = 20, 9, 7, 3, 2
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(I1, I2, I3, dtype=torch.float32, device="cuda", generator=g)
    xf = torch.empty_like(x)
    rt.tensor_fiber_major(x.data_ptr(), (I1, I2, I3), xf.data_ptr())
    a2 = torch.randn(I2, R2, dtype=torch.float64, device="cuda", generator=g)
    a3 = torch.randn(I3, R3, dtype=torch.float64, device="cuda", generator=g)
    W = R2 * R3
    G = torch.full((W, W), 7.0, dtype=torch.float64, device="cuda")
    R = torch.full((W, I1), 7.0, dtype=torch.float64, device="cuda")
    out = rt.kron_fiber_sketch(xf.data_ptr(), (I1, I2, I3), a2.data_ptr(), a3.data_ptr(), R2, R3,
                               0.5, s, seed, G.data_ptr(), R.data_ptr(), want_draws=True,
                               fiber_major=True)
    torch.cuda.synchronize()
    idx, w = out["indices"], out["weights"]
    A2, A3, X = a2.cpu().numpy(), a3.cpu().numpy(), x.cpu().numpy().astype(np.float64)
    total = I2 * I3
    data = idx < total
    assert out["data_draws"] == int(data.sum())
    assert out["unique_rows"] == len(np.unique(idx[data]))
    j2, j3 = idx[data] // I3, idx[data] % I3
    Z = np.einsum("tp,tq->tpq", A2[j2], A3[j3]).reshape(-1, W)
    Gr = (Z * (w[data] ** 2)[:, None]).T @ Z
    for j, wt in zip(idx[~data] - total, w[~data]):
        Gr[j, j] += wt * wt * 0.5
    Rr = (Z * (w[data] ** 2)[:, None]).T @ X[:, j2, j3].T
    assert np.allclose(G.cpu().numpy(), Gr, rtol=1e-12, atol=1e-12)
    assert np.allclose(R.cpu().numpy(), Rr, rtol=1e-12, atol=1e-12)
