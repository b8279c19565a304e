"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

The reference ships no stored golden vectors; every fixture
here is produced by oracle/_ref/librtucker_ref.so -- the reference compiled
from /root/reference/proj sources by oracle/Makefile -- through its own C API
(rtucker_*) and its own C++ routines (oracle/ref_harness.cpp). Floats are
stored as hex strings so the fixtures are exact.

    python tests/golden/make_golden.py        (needs oracle/_ref; run here)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402


def hx(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def splitmix_tensor(shape, seed):
    """Deterministic input without numpy RNG dependence: SplitMix64 uniforms in
    [-1, 1) (the reference's test oracles use the same construction,
    ref tests/oracles.hpp:19-40)."""
    from oracle.oracle import Oracle
    n = int(np.prod(shape))
    u = Oracle().splitmix_stream(seed, n)
    vals = (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return (2.0 * vals - 1.0).reshape(shape)


def main():
    ref = Reference()
    out = {"generator": "tests/golden/make_golden.py via oracle/_ref (reference built from "
                        "/root/reference/proj sources)"}

    # sample_count known answers (ref tests/test_sketch_ridge.cpp:17-21)
    out["sample_count"] = [
        {"args": [0.5, 4, 0.1, 0.1], "s": ref.sample_count(0.5, 4, 0.1, 0.1)},
        {"args": [1.0, 2, 0.9, 0.001], "s": ref.sample_count(1.0, 2, 0.9, 0.001)},
        {"args": [1.0, 2, 0.001, 0.5], "s": ref.sample_count(1.0, 2, 0.001, 0.5)},
        {"args": [0.5, 125, 0.1, 0.1], "s": ref.sample_count(0.5, 125, 0.1, 0.1)},
        {"args": [0.5, 4096, 0.1, 0.1], "s": ref.sample_count(0.5, 4096, 0.1, 0.1)},
    ]

    # uniform init (ref tucker.cpp:168-190)
    core, factors = ref.random_model((7, 6, 5), (3, 2, 2), 42)
    out["random_model"] = {"shape": [7, 6, 5], "ranks": [3, 2, 2], "seed": 42,
                           "core": hx(core), "factors": [hx(f) for f in factors]}

    # factor scores (ref kronecker.cpp:9-35)
    f = splitmix_tensor((40, 5), 9)
    sc, tot, rank = ref.factor_scores(f)
    out["factor_scores"] = {"factor_seed": 9, "shape": [40, 5], "scores": hx(sc),
                            "sum": float(tot).hex(), "rank": rank}

    # a sketched core update: indices, weights, core (ref tucker.cpp:141-166)
    shape, ranks = (12, 10, 8), (3, 2, 2)
    x = splitmix_tensor(shape, 5)
    core, factors = ref.random_model(shape, ranks, 3)
    c, idx, w, rd, obj = ref.core_sketch(shape, ranks, core, factors, 0.01, x, 600, 77)
    out["core_sketch"] = {"shape": list(shape), "ranks": list(ranks), "x_seed": 5,
                          "model_seed": 3, "lambda": 0.01, "s": 600, "seed": 77,
                          "indices": [int(v) for v in idx], "weights": hx(w), "core": hx(c),
                          "rank_deficient": rd, "sketched_objective": float(obj).hex()}

    # full ALS through the reference C API (ref capi.cpp:176-201)
    runs = []
    for shape, ranks, lam, sk, s, iters, seed in [((10, 9, 8), (3, 2, 2), 0.01, 1, 800, 3, 1),
                                                  ((10, 9, 8), (3, 2, 2), 0.01, 0, 0, 3, 1),
                                                  ((8, 7, 6, 5), (2, 2, 2, 2), 0.05, 1, 500, 2, 4),
                                                  ((20, 20, 20), (4, 4, 4), 1e-3, 1, 3000, 4, 0)]:
        x = splitmix_tensor(shape, 100 + len(runs))
        r = ref.als(x, ranks, lam=lam, sketched_core=sk, max_iterations=iters, tolerance=0.0,
                    sample_count_override=s, record_history=1, seed=seed)
        runs.append({"shape": list(shape), "ranks": list(ranks), "lambda": lam,
                     "sketched_core": sk, "s": s, "iterations": iters, "seed": seed,
                     "x_seed": 100 + len(runs),
                     "history": [[h[0], h[1], float(h[2]).hex(), float(h[3]).hex()]
                                 for h in r["history"]],
                     "reconstruction": hx(r["reconstruction"])})
    out["als"] = runs

    # ridge toolkit on the C-API test system (ref tests/test_capi.cpp:176-213)
    import ctypes as C
    a = np.array([1.0, 0.0, 0.0, 1.0, 1.0, 1.0, -1.0, 1.0])
    b = np.array([1.0, 2.0, 3.0, 0.0])
    L = ref.lib
    xo = np.zeros(2)
    p = lambda v: v.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    assert L.rtucker_solve_ridge(p(a), C.c_uint64(4), C.c_uint64(2), p(b), C.c_double(0.1),
                                 p(xo)) == 0
    sc = np.zeros(4)
    assert L.rtucker_ridge_scores(p(a), C.c_uint64(4), C.c_uint64(2), C.c_double(0.5),
                                  p(sc)) == 0
    xs = np.zeros(2)
    s_out = C.c_uint64()
    bp = C.c_double()
    assert L.rtucker_sketched_ridge(p(a), C.c_uint64(4), C.c_uint64(2), p(b), None,
                                    C.c_double(0.1), C.c_double(0.0), C.c_double(0.25),
                                    C.c_double(0.2), C.c_uint64(4000), C.c_uint64(17), p(xs),
                                    C.byref(s_out), C.byref(bp)) == 0
    out["toolkit"] = {"a": hx(a), "b": hx(b), "solve_ridge_lambda_0.1": hx(xo),
                      "ridge_scores_lambda_0.5": hx(sc), "sketched_ridge": hx(xs),
                      "sketched_s": s_out.value, "beta_prime": float(bp.value).hex()}

    path = os.path.join(HERE, "golden_ref.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
