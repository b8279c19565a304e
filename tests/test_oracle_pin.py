"""CPU: pins the C restatement (oracle/) to the reference compiled from its own
sources (oracle/_ref) on randomized inputs -- bitwise equality of every
hot-path routine. Skipped when oracle/_ref was not built (no /root/reference)."""
import os

import numpy as np
import pytest

from oracle.oracle import REF_SO, OracleError

pytestmark = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Reference
    return Reference()


CASES = [((10, 9, 8), (3, 2, 4)), ((6, 5, 4), (2, 2, 2)), ((12, 7, 5, 6), (2, 3, 2, 2)),
         ((15, 11), (4, 3)), ((30,), (5,)), ((5, 4, 3), (5, 4, 3))]


@pytest.mark.parametrize("m,n,kind", [(9, 4, "normal"), (4, 9, "normal"), (30, 30, "spd"),
                                      (12, 5, "rankdef"), (6, 6, "zero"), (50, 8, "pareto")])
def test_compact_svd(oracle, ref, m, n, kind):
    rng = np.random.default_rng(m * 100 + n)
    if kind == "normal":
        a = rng.standard_normal((m, n))
    elif kind == "spd":
        q = rng.standard_normal((m, n))
        a = q.T @ q + 1e-3 * np.eye(n)
    elif kind == "rankdef":
        a = rng.standard_normal((m, 2)) @ rng.standard_normal((2, n))
    elif kind == "pareto":
        a = rng.standard_normal((m, n)) * (rng.pareto(1.5, m) + 1)[:, None]
    else:
        a = np.zeros((m, n))
    ou, os_, ovt = oracle.compact_svd(a)
    ru, rs, rvt = ref.compact_svd(a)
    assert np.array_equal(os_, rs) and np.array_equal(ou, ru) and np.array_equal(ovt, rvt)


@pytest.mark.parametrize("shape,ranks", CASES)
def test_model_steps_bitwise(oracle, ref, shape, ranks):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    core, factors = ref.random_model(shape, ranks, 11)
    oc, of = oracle.random_model(shape, ranks, 11)
    assert np.array_equal(core, oc) and all(np.array_equal(a, b) for a, b in zip(factors, of))
    for mode in range(1, len(shape) + 1):
        assert np.array_equal(oracle.update_factor(shape, ranks, core, factors, 0.02, x, mode),
                              ref.update_factor(shape, ranks, core, factors, 0.02, x, mode))
    assert np.array_equal(oracle.update_core_exact(shape, ranks, core, factors, 0.02, x),
                          ref.update_core_exact(shape, ranks, core, factors, 0.02, x))
    assert oracle.tucker_loss(shape, ranks, core, factors, 0.02, x)[0] == \
        ref.tucker_loss(shape, ranks, core, factors, 0.02, x)
    for n, f in enumerate(factors):
        sc, _, tot, rank = oracle.factor_scores(f)
        rsc, rtot, rrank = ref.factor_scores(f)
        assert np.array_equal(sc, rsc) and tot == rtot and rank == rrank


@pytest.mark.parametrize("shape,ranks", CASES)
@pytest.mark.parametrize("lam,s,seed", [(0.01, 700, 5), (0.5, 300, 123456789), (0.0, 900, 2)])
def test_sketched_core_bitwise(oracle, ref, shape, ranks, lam, s, seed):
    rng = np.random.default_rng(7)
    x = rng.standard_normal(shape)
    core, factors = ref.random_model(shape, ranks, 3)
    oc, oidx, ow, ord_ = oracle.update_core_fast(shape, ranks, core, factors, lam, x, s, seed)
    rc, ridx, rw, rrd, _ = ref.core_sketch(shape, ranks, core, factors, lam, x, s, seed)
    assert np.array_equal(oidx, ridx) and np.array_equal(ow, rw)
    assert np.array_equal(oc, rc) and ord_ == rrd


def test_sketched_core_zero_factor(oracle, ref):
    shape, ranks = (4, 3, 2), (2, 2, 2)
    x = np.random.default_rng(1).standard_normal(shape)
    core, factors = ref.random_model(shape, ranks, 3)
    factors[1] = np.zeros_like(factors[1])
    oc, _, _, _ = oracle.update_core_fast(shape, ranks, core, factors, 0.3, x, 50, 1)
    rc = ref.update_core_fast(shape, ranks, core, factors, 0.3, x, 50, 1)
    assert not oc.any() and not rc.any()


@pytest.mark.parametrize("shape,ranks,sk", [((10, 9, 8), (3, 2, 4), 1), ((8, 8, 8), (2, 2, 2), 0),
                                            ((7, 6, 5, 4), (2, 2, 2, 2), 1), ((25, 20), (3, 4), 1)])
def test_als_bitwise(oracle, ref, shape, ranks, sk):
    x = np.random.default_rng(3).standard_normal(shape)
    kw = dict(lam=0.01, sketched_core=sk, max_iterations=3, tolerance=0.0,
              sample_count_override=1500, record_history=1, seed=9)
    o = oracle.als(x, ranks, **kw)
    r = ref.als(x, ranks, **kw)
    assert o["history"] == r["history"]
    assert np.array_equal(oracle.reconstruct(shape, ranks, o["core"], o["factors"]),
                          r["reconstruction"])


def test_als_tolerance_stop(oracle, ref):
    x = np.random.default_rng(4).standard_normal((9, 8, 7))
    kw = dict(lam=0.02, max_iterations=40, tolerance=1e-3, seed=2)
    assert oracle.als(x, (2, 2, 2), **kw)["iterations"] == ref.als(x, (2, 2, 2), **kw)["iterations"]


def test_error_paths_match(oracle, ref):
    x = np.ones((4, 4))
    for kw in [dict(max_iterations=0), dict(max_iterations=1)]:
        ranks = (5, 2) if kw["max_iterations"] else (2, 2)
        with pytest.raises(OracleError) as eo:
            oracle.als(x, ranks, **kw)
        with pytest.raises(OracleError) as er:
            ref.als(x, ranks, **kw)
        assert eo.value.code == er.value.code == 1


@pytest.mark.parametrize("n,d,del_,s,seed", [(50, 4, 0.0, 3000, 99), (300, 12, 11.5, 5000, 3),
                                             (120, 6, 6.0, 2000, 8)])
def test_aug_draw_matches_reference_sketch(oracle, ref, n, d, del_, s, seed):
    """The oracle's AugmentedSampler draws (the GPU test's checker) are the RowSketch of the
    reference's own approximate_ridge_regression, bit for bit (sampler.cpp:9-57)."""
    rng = np.random.default_rng(n + d)
    a = rng.standard_normal((n, d))
    b = rng.standard_normal(n)
    cand = rng.random(n) ** 2
    cand[::5] = 0.0
    oi, ow = oracle.aug_draw(cand, d, del_, seed, s)
    ri, rw = ref.aug_sketch(a, b, cand, 0.1, del_, s, seed)
    assert np.array_equal(oi, ri)
    assert np.array_equal(ow, rw)
