"""Full-size C1 run pinned to the REFERENCE's own output (tests/golden/golden_c1.json,
made by tests/golden/make_golden_c1.py through oracle/_ref).

C1 = BASELINE config 0: 100^3, Tucker rank (5,5,5), lambda 1e-3, 20,000 sampled core rows,
10 sweeps. The input comes from rtucker_tensor_generate (ref synthetic.cpp), which our C ABI
re-implements on the GPU (reconstruction on device, same SplitMix64 streams), so the planted
checksum must match exactly and the tensor to a reordered-sum tolerance; the whole ALS history
(40 rows: F1,F2,F3,Core per sweep) must match the reference within its noise floor.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_c1.json")))


def _h(s):
    return float.fromhex(s)


@pytest.fixture(scope="module")
def c1(rt):
    g = G["generate"]
    x, ck = rt.Tensor.generate(g["shape"], g["planted"], g["noise_fraction"], g["noise_sigma"],
                               g["seed"])
    return x, ck


def test_c1_generator_matches_reference(c1):
    x, ck = c1
    assert ck == G["planted_checksum"]
    a = x.numpy()
    assert abs(a.sum() - _h(G["tensor_sum"])) <= 1e-11 * np.abs(a).sum()
    assert abs((a * a).sum() - _h(G["tensor_sumsq"])) <= 1e-12 * _h(G["tensor_sumsq"])


def test_c1_als_history_matches_reference(rt, oracle, c1):
    x, _ = c1
    a = G["als"]
    r = rt.als_run(x, a["ranks"], rt.options(lam=a["lam"], sketched_core=a["sketched_core"],
                                             sample_count_override=a["sample_count_override"],
                                             max_iterations=a["max_iterations"],
                                             tolerance=a["tolerance"],
                                             record_history=a["record_history"], seed=a["seed"]))
    gh = r.history()
    ref = G["history"]
    assert [(h[0], h[1]) for h in gh] == [(h[0], h[1]) for h in ref]
    # the same sampled rows and the same normal equations; only summation order differs.
    # The bar per row is 10x the reference's own noise floor there (its change under a
    # one-ulp input perturbation, golden_c1.json "noise_floor"): uniform planted factors
    # are ill-conditioned, so the floor grows from 1e-15 (first factor updates) to 1e-5.
    floor = G["noise_floor"]
    for k, ((gi, gs, gl, grm), (ri, rs, rl, rrm)) in enumerate(zip(gh, ref)):
        e = abs(gl - _h(rl)) / _h(rl)
        assert e <= 10 * floor[k] + 1e-13, (gi, gs, gl, _h(rl), e, floor[k])
    m = r.model()
    xh = oracle.reconstruct(tuple(x.shape), tuple(a["ranks"]), m.core, m.factors)
    ss = float((xh * xh).sum())
    assert abs(ss - _h(G["reconstruction_sumsq"])) <= 10 * max(floor) * _h(G["reconstruction_sumsq"])
