"""BASELINE config 4 microbench kernels (rtucker_b200_kron_fiber_sketch): Kronecker-product
sampling of [A2 (x) A3; sqrt(lambda) I], the W x W sketched Gram (order-2 vech machinery) and
the fused fiber-gather RHS (W x I1, FP32 tensor upcast in-kernel), against a direct numpy
evaluation from the same draws and against the oracle's draw stream."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("I1,I2,I3,R2,R3,s", [(48, 40, 36, 4, 4, 3000),
                                               (32, 64, 50, 8, 5, 20000),
                                               (40, 20, 24, 3, 7, 500)])
def test_c4_gram_rhs_match_definition(rt, oracle, I1, I2, I3, R2, R3, s):
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(I1, I2, I3, dtype=torch.float32, device="cuda", generator=g)
    a2 = torch.randn(I2, R2, dtype=torch.float64, device="cuda", generator=g)
    a3 = torch.randn(I3, R3, dtype=torch.float64, device="cuda", generator=g)
    W = R2 * R3
    gram = torch.zeros(W, W, dtype=torch.float64, device="cuda")
    rhs = torch.zeros(W, I1, dtype=torch.float64, device="cuda")
    lam = 1e-2
    out = rt.kron_fiber_sketch(x.data_ptr(), (I1, I2, I3), a2.data_ptr(), a3.data_ptr(), R2, R3,
                               lam, s, 11, gram.data_ptr(), rhs.data_ptr(), want_draws=True)
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
