"""Condition-number-scaled error bars for the parity tests (an FP64 result
that solves a linear system can only be claimed to c * kappa * eps of another correct
implementation that sums in a different order)."""
import numpy as np

EPS = np.finfo(np.float64).eps


def kkt_kappa(core, factors, mode, lam):
    """kappa(K K^T + lam I), K = G_(n) (kron_{m != n} A_m)^T: the system update_factor
    solves (ref tucker.cpp:70-89)."""
    q = core
    for m, a in enumerate(factors):
        if m != mode:
            q = np.moveaxis(np.tensordot(a.T @ a, q, axes=(1, m)), 0, m)
    gn = np.moveaxis(core, mode, 0).reshape(core.shape[mode], -1)
    qn = np.moveaxis(q, mode, 0).reshape(core.shape[mode], -1)
    kk = gn @ qn.T + lam * np.eye(core.shape[mode])
    return float(np.linalg.cond(kk))


def factor_bar(kappa, shape, mode, c=64):
    """c (kappa + sqrt(J)) eps: the solve amplifies by kappa(K K^T + lam I); M = X_(n) K^T
    sums J = prod_{m != n} I_m products in a different order (~sqrt(J) eps)."""
    j = int(np.prod(shape)) // shape[mode]
    return c * (kappa + np.sqrt(j)) * EPS


def core_exact_kappa(factors):
    """prod_n kappa(A_n): the exact core is X projected on the factors' SVD bases and scaled
    by sigma / (sigma^2 + lambda) (ref tucker.cpp:91-129); ours come from eigenpairs of
    A_n^T A_n, the oracle's from the one-sided Jacobi SVD of A_n."""
    k = 1.0
    for a in factors:
        k *= float(np.linalg.cond(a))
    return k


def frel(a, b):
    a, b = np.asarray(a, float).ravel(), np.asarray(b, float).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
