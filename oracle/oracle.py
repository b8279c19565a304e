"""ctypes bindings to the parity checkers -- TEST INFRASTRUCTURE ONLY.

* ``Oracle``    -> oracle/build/liboracle.so, our C restatement of the reference
                   path (oracle/rtucker_oracle.c).
* ``Reference`` -> oracle/_ref/librtucker_ref.so, the reference itself compiled
                   from /root/reference/proj sources (its C API ``rtucker_*``
                   plus the ``ref_*`` shim in oracle/ref_harness.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module. The product package
(paper_2107_10654_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librtucker_ref.so")

_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)


def build(ref: bool = True) -> None:
    """Compile the oracle (and, when /root/reference is present, the reference)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj"):
        targets.append("ref")
        lib = os.path.join(HERE, "..", "paper_2107_10654_b200", "lib", "librtucker_b200.so")
        if os.path.exists(lib):
            targets.append("capi_test")  # the reference's test_capi.cpp against our library
    subprocess.check_call(["make", "-s", "-C", HERE] + targets)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _p(a: np.ndarray):
    if a is None:
        return None
    if a.dtype == np.float64:
        return a.ctypes.data_as(_f64p)
    if a.dtype == np.uint64:
        return a.ctypes.data_as(_u64p)
    if a.dtype == np.int32:
        return a.ctypes.data_as(C.POINTER(C.c_int))
    if a.dtype == np.uint32:
        return a.ctypes.data_as(C.POINTER(C.c_uint32))
    raise TypeError(a.dtype)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"status {code}: {msg}")
        self.code = code
        self.msg = msg


class AlsOptions(C.Structure):
    """Mirror of rtucker_als_options (rtucker.h:58-68)."""

    _fields_ = [
        ("lambda_", C.c_double),
        ("sketched_core", C.c_int),
        ("epsilon", C.c_double),
        ("delta", C.c_double),
        ("seed", C.c_uint64),
        ("max_iterations", C.c_uint32),
        ("tolerance", C.c_double),
        ("sample_count_override", C.c_uint64),
        ("record_history", C.c_int),
    ]


def model_split(shape, ranks, factors_cat):
    out, off = [], 0
    for i, r in zip(shape, ranks):
        out.append(factors_cat[off:off + i * r].reshape(i, r))
        off += i * r
    return out


class Oracle:
    """Our C restatement (bit-identical to the reference; pinned by tests)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = C.CDLL(path)
        self.lib.oracle_last_error.restype = C.c_char_p
        self.lib.orc_splitmix_at.restype = C.c_uint64
        self.lib.orc_splitmix_at.argtypes = [C.c_uint64, C.c_uint64]

    def _chk(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.oracle_last_error().decode())

    def splitmix_stream(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self.lib.orc_splitmix_stream(C.c_uint64(seed), C.c_uint64(n), _p(out))
        return out

    def compact_svd(self, a):
        a = _f64(a)
        m, n = a.shape
        k = min(m, n)
        u, s, vt = np.zeros((m, k)), np.zeros(k), np.zeros((k, n))
        rank = C.c_size_t()
        self._chk(self.lib.orc_compact_svd(_p(a), C.c_size_t(m), C.c_size_t(n), _p(u), _p(s),
                                           _p(vt), C.byref(rank)))
        r = rank.value
        return u[:, :r], s[:r], vt[:r]

    def ridge_scores(self, a, lam: float) -> np.ndarray:
        a = _f64(a)
        out = np.zeros(a.shape[0])
        self._chk(self.lib.orc_ridge_scores(_p(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
                                            C.c_double(lam), _p(out)))
        return out

    def solve_ridge(self, a, b, lam: float) -> np.ndarray:
        a, b = _f64(a), _f64(b)
        x = np.zeros(a.shape[1])
        self._chk(self.lib.orc_solve_ridge_exact(_p(a), C.c_size_t(a.shape[0]),
                                                 C.c_size_t(a.shape[1]), _p(b), C.c_double(lam),
                                                 _p(x)))
        return x

    def sample_count(self, beta_prime, d, eps, delta) -> int:
        out = C.c_uint64()
        self._chk(self.lib.orc_sample_count(C.c_double(beta_prime), C.c_size_t(d),
                                            C.c_double(eps), C.c_double(delta), C.byref(out)))
        return out.value

    def sketched_ridge(self, a, b, scores, lam, d_eff_lower, eps, delta, s_override, seed):
        a, b = _f64(a), _f64(b)
        n, d = a.shape
        x = np.zeros(d)
        s = C.c_uint64()
        bp = C.c_double()
        sc = None if scores is None else _f64(scores)
        self._chk(self.lib.orc_sketched_ridge(_p(a), C.c_uint64(n), C.c_uint64(d), _p(b),
                                              _p(sc) if sc is not None else None,
                                              C.c_double(lam), C.c_double(d_eff_lower),
                                              C.c_double(eps), C.c_double(delta),
                                              C.c_uint64(s_override), C.c_uint64(seed), _p(x),
                                              C.byref(s), C.byref(bp)))
        return x, s.value, bp.value

    def aug_draw(self, cand, d, d_eff_lower, seed, s):
        """AugmentedSampler draws of the dense toolkit (sampler.cpp:9-57)."""
        cand = _f64(cand)
        idx, w = np.zeros(s, np.uint64), np.zeros(s)
        self._chk(self.lib.orc_aug_draw(_p(cand), C.c_uint64(len(cand)), C.c_uint64(d),
                                        C.c_double(d_eff_lower), C.c_uint64(seed), C.c_uint64(s),
                                        _p(idx), _p(w)))
        return idx, w

    def dense_normal_eq(self, a, b, lam, idx, w):
        a, b = _f64(a), _f64(b)
        n, d = a.shape
        idx, w = _u64(idx), _f64(w)
        g, rhs = np.zeros((d, d)), np.zeros(d)
        self._chk(self.lib.orc_dense_normal_eq(_p(a), C.c_uint64(n), C.c_uint64(d), _p(b),
                                               C.c_double(lam), C.c_uint64(len(idx)), _p(idx),
                                               _p(w), _p(g), _p(rhs)))
        return g, rhs

    def factor_scores(self, f):
        f = _f64(f)
        rows, cols = f.shape
        sc, cdf = np.zeros(rows), np.zeros(rows)
        tot = C.c_double()
        rank = C.c_size_t()
        self._chk(self.lib.orc_factor_scores(_p(f), C.c_size_t(rows), C.c_size_t(cols), _p(sc),
                                             _p(cdf), C.byref(tot), C.byref(rank)))
        return sc, cdf, tot.value, rank.value

    def kron_draw(self, rows, d, scores_list, cdf_list, sums, seed, s):
        rows = _u64(rows)
        sc = _f64(np.concatenate(scores_list))
        cdf = _f64(np.concatenate(cdf_list))
        sums = _f64(sums)
        idx, w = np.zeros(s, np.uint64), np.zeros(s)
        used = C.c_uint64()
        self._chk(self.lib.orc_kron_draw(C.c_uint32(len(rows)), _p(rows), C.c_uint64(d), _p(sc),
                                         _p(cdf), _p(sums), C.c_uint64(seed), C.c_uint64(s),
                                         _p(idx), _p(w), C.byref(used)))
        return idx, w, used.value

    def kron_normal_eq(self, shape, ranks, factors, x, lam, idx, w):
        shape, ranks = _u64(shape), _u64(ranks)
        fc = _f64(np.concatenate([_f64(f).ravel() for f in factors]))
        d = int(np.prod(ranks))
        g, rhs = np.zeros((d, d)), np.zeros(d)
        idx, w = _u64(idx), _f64(w)
        self._chk(self.lib.orc_kron_sketch_normal_eq(C.c_uint32(len(shape)), _p(shape), _p(ranks),
                                                     _p(fc), _p(_f64(x).ravel()), C.c_double(lam),
                                                     C.c_uint64(len(idx)), _p(idx), _p(w), _p(g),
                                                     _p(rhs)))
        return g, rhs

    def pinv_solve(self, g, rhs):
        g, rhs = _f64(g), _f64(rhs)
        x = np.zeros(len(rhs))
        rank = C.c_size_t()
        self._chk(self.lib.orc_pinv_solve(_p(g), _p(rhs), C.c_size_t(len(rhs)), _p(x),
                                          C.byref(rank)))
        return x, rank.value

    def _model_args(self, shape, ranks, core, factors):
        shape, ranks = _u64(shape), _u64(ranks)
        core = _f64(core).ravel()
        fc = _f64(np.concatenate([_f64(f).ravel() for f in factors]))
        return shape, ranks, core, fc

    def reconstruct(self, shape, ranks, core, factors):
        shape, ranks, core, fc = self._model_args(shape, ranks, core, factors)
        out = np.zeros(int(np.prod(shape)))
        self._chk(self.lib.orc_reconstruct(C.c_uint32(len(shape)), _p(shape), _p(ranks),
                                           _p(core), _p(fc), _p(out)))
        return out.reshape(tuple(int(v) for v in shape))

    def tucker_loss(self, shape, ranks, core, factors, lam, x):
        shape, ranks, core, fc = self._model_args(shape, ranks, core, factors)
        loss, rmse = C.c_double(), C.c_double()
        self._chk(self.lib.orc_tucker_loss(C.c_uint32(len(shape)), _p(shape), _p(ranks), _p(core),
                                           _p(fc), C.c_double(lam), _p(_f64(x).ravel()),
                                           C.byref(loss), C.byref(rmse)))
        return loss.value, rmse.value

    def update_factor(self, shape, ranks, core, factors, lam, x, mode):
        shape, ranks, core, fc = self._model_args(shape, ranks, core, factors)
        self._chk(self.lib.orc_update_factor(C.c_uint32(len(shape)), _p(shape), _p(ranks),
                                             _p(core), _p(fc), C.c_double(lam),
                                             _p(_f64(x).ravel()), C.c_uint32(mode)))
        return model_split(shape, ranks, fc)[mode - 1].copy()

    def update_factor_sketched(self, shape, ranks, core, factors, lam, x, mode, s, seed):
        """Perf-mode sketched factor update (not in the reference; parity unpinned).
        Returns (new factor, indices, weights)."""
        shape, ranks, core, fc = self._model_args(shape, ranks, core, factors)
        idx, w = np.zeros(s, np.uint64), np.zeros(s)
        self._chk(self.lib.orc_update_factor_sketched(
            C.c_uint32(len(shape)), _p(shape), _p(ranks), _p(core), _p(fc), C.c_double(lam),
            _p(_f64(x).ravel()), C.c_uint32(mode), C.c_uint64(s), C.c_uint64(seed), _p(idx),
            _p(w)))
        return model_split(shape, ranks, fc)[mode - 1].copy(), idx, w

    def update_core_exact(self, shape, ranks, core, factors, lam, x):
        shape, ranks, core, fc = self._model_args(shape, ranks, core, factors)
        out = np.zeros(int(np.prod(ranks)))
        self._chk(self.lib.orc_update_core_exact(C.c_uint32(len(shape)), _p(shape), _p(ranks),
                                                 _p(core), _p(fc), C.c_double(lam),
                                                 _p(_f64(x).ravel()), _p(out)))
        return out

    def update_core_fast(self, shape, ranks, core, factors, lam, x, s, seed, eps=0.1,
                         delta=0.1):
        shape, ranks, core, fc = self._model_args(shape, ranks, core, factors)
        out = np.zeros(int(np.prod(ranks)))
        idx, w = np.zeros(max(s, 1), np.uint64), np.zeros(max(s, 1))
        rd = C.c_int()
        s_out = C.c_uint64()
        self._chk(self.lib.orc_update_core_fast(C.c_uint32(len(shape)), _p(shape), _p(ranks),
                                                _p(core), _p(fc), C.c_double(lam),
                                                _p(_f64(x).ravel()), C.c_uint64(s),
                                                C.c_double(eps), C.c_double(delta),
                                                C.c_uint64(seed), _p(out),
                                                _p(idx) if s else None, _p(w) if s else None,
                                                C.byref(rd), C.byref(s_out)))
        return out, idx, w, bool(rd.value)

    def random_model(self, shape, ranks, seed):
        shape, ranks = _u64(shape), _u64(ranks)
        core = np.zeros(int(np.prod(ranks)))
        fc = np.zeros(int(np.sum(shape * ranks)))
        self._chk(self.lib.orc_random_model(C.c_uint32(len(shape)), _p(shape), _p(ranks),
                                            C.c_uint64(seed), _p(core), _p(fc)))
        return core, model_split(shape, ranks, fc)

    def als(self, x, ranks, lam=1e-3, sketched_core=0, epsilon=0.1, delta=0.1, seed=0,
            max_iterations=50, tolerance=1e-6, sample_count_override=0, record_history=0,
            factor_samples=0):
        x = _f64(x)
        shape = _u64(x.shape)
        ranks = _u64(ranks)
        o = (C.c_double * 0)()
        opts = AlsOptions(lam, sketched_core, epsilon, delta, seed, max_iterations, tolerance,
                          sample_count_override, record_history)
        order = len(shape)
        core = np.zeros(int(np.prod(ranks)))
        fc = np.zeros(int(np.sum(shape * ranks)))
        hmax = max_iterations * (order + 1)
        hi = np.zeros(hmax, np.uint32)
        hs = np.zeros(hmax, np.int32)
        hl, hr = np.zeros(hmax), np.zeros(hmax)
        hlen = C.c_uint64()
        iters = C.c_uint32()
        fl, fr = C.c_double(), C.c_double()
        seeds = np.zeros(max_iterations, np.uint64)
        del o
        self._chk(self.lib.orc_als_fs(C.c_uint32(order), _p(shape), _p(ranks), _p(x.ravel()),
                                      C.byref(opts), C.c_uint64(factor_samples), _p(core),
                                      _p(fc), _p(hi), _p(hs), _p(hl), _p(hr), C.byref(hlen),
                                      C.byref(iters), C.byref(fl), C.byref(fr), _p(seeds)))
        n = hlen.value
        steps = ["Core" if v == order else f"F{v + 1}" for v in hs[:n]]
        return {
            "core": core.reshape(tuple(int(r) for r in ranks)),
            "factors": model_split(shape, ranks, fc),
            "history": list(zip(hi[:n].tolist(), steps, hl[:n].tolist(), hr[:n].tolist())),
            "iterations": iters.value,
            "final_loss": fl.value,
            "final_rmse": fr.value,
            "core_seeds": seeds[:iters.value],
        }


class Reference:
    """The reference compiled from its own sources (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p
        self.lib.rtucker_last_error.restype = C.c_char_p
        self.lib.rtucker_result_final_loss.restype = C.c_double
        self.lib.rtucker_result_final_rmse.restype = C.c_double
        self.lib.rtucker_result_iterations.restype = C.c_uint32
        self.lib.rtucker_result_history_size.restype = C.c_uint64
        self.lib.rtucker_result_timing_size.restype = C.c_uint64
        self.lib.rtucker_tensor_data.restype = C.POINTER(C.c_double)
        self.lib.rtucker_tensor_size.restype = C.c_uint64
        self.lib.rtucker_model_lambda.restype = C.c_double

    def _chk(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _capi(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.rtucker_last_error().decode())

    def sample_count(self, beta_prime, d, eps, delta) -> int:
        out = C.c_uint64()
        self._chk(self.lib.ref_sample_count(C.c_double(beta_prime), C.c_uint64(d),
                                            C.c_double(eps), C.c_double(delta), C.byref(out)))
        return out.value

    def compact_svd(self, a):
        a = _f64(a)
        m, n = a.shape
        k = min(m, n)
        u, s, vt = np.zeros((m, k)), np.zeros(k), np.zeros((k, n))
        rank = C.c_uint64()
        self._chk(self.lib.ref_compact_svd(_p(a), C.c_uint64(m), C.c_uint64(n), _p(u), _p(s),
                                           _p(vt), C.byref(rank)))
        r = rank.value
        return u[:, :r], s[:r], vt[:r]

    def factor_scores(self, f):
        f = _f64(f)
        sc = np.zeros(f.shape[0])
        tot = C.c_double()
        rank = C.c_uint64()
        self._chk(self.lib.ref_factor_scores(_p(f), C.c_uint64(f.shape[0]), C.c_uint64(f.shape[1]),
                                             _p(sc), C.byref(tot), C.byref(rank)))
        return sc, tot.value, rank.value

    def _margs(self, shape, ranks, core, factors):
        shape, ranks = _u64(shape), _u64(ranks)
        return (C.c_uint32(len(shape)), shape, ranks, _f64(core).ravel(),
                _f64(np.concatenate([_f64(f).ravel() for f in factors])))

    def core_sketch(self, shape, ranks, core, factors, lam, x, s, seed):
        o, shape, ranks, core, fc = self._margs(shape, ranks, core, factors)
        out = np.zeros(int(np.prod(ranks)))
        idx, w = np.zeros(s, np.uint64), np.zeros(s)
        rd = C.c_int()
        obj = C.c_double()
        self._chk(self.lib.ref_core_sketch(o, _p(shape), _p(ranks), _p(core), _p(fc),
                                           C.c_double(lam), _p(_f64(x).ravel()), C.c_uint64(s),
                                           C.c_uint64(seed), _p(out), _p(idx), _p(w),
                                           C.byref(rd), C.byref(obj)))
        return out, idx, w, bool(rd.value), obj.value

    def update_core_fast(self, shape, ranks, core, factors, lam, x, s, seed):
        o, shape, ranks, core, fc = self._margs(shape, ranks, core, factors)
        out = np.zeros(int(np.prod(ranks)))
        self._chk(self.lib.ref_update_core_fast(o, _p(shape), _p(ranks), _p(core), _p(fc),
                                                C.c_double(lam), _p(_f64(x).ravel()),
                                                C.c_uint64(s), C.c_uint64(seed), _p(out)))
        return out

    def update_factor(self, shape, ranks, core, factors, lam, x, mode):
        o, shape, ranks, core, fc = self._margs(shape, ranks, core, factors)
        out = np.zeros(int(shape[mode - 1] * ranks[mode - 1]))
        self._chk(self.lib.ref_update_factor(o, _p(shape), _p(ranks), _p(core), _p(fc),
                                             C.c_double(lam), _p(_f64(x).ravel()),
                                             C.c_uint32(mode), _p(out)))
        return out.reshape(int(shape[mode - 1]), int(ranks[mode - 1]))

    def update_core_exact(self, shape, ranks, core, factors, lam, x):
        o, shape, ranks, core, fc = self._margs(shape, ranks, core, factors)
        out = np.zeros(int(np.prod(ranks)))
        self._chk(self.lib.ref_update_core_exact(o, _p(shape), _p(ranks), _p(core), _p(fc),
                                                 C.c_double(lam), _p(_f64(x).ravel()), _p(out)))
        return out

    def tucker_loss(self, shape, ranks, core, factors, lam, x):
        o, shape, ranks, core, fc = self._margs(shape, ranks, core, factors)
        out = C.c_double()
        self._chk(self.lib.ref_tucker_loss(o, _p(shape), _p(ranks), _p(core), _p(fc),
                                           C.c_double(lam), _p(_f64(x).ravel()), C.byref(out)))
        return out.value

    def random_model(self, shape, ranks, seed):
        shape, ranks = _u64(shape), _u64(ranks)
        core = np.zeros(int(np.prod(ranks)))
        fc = np.zeros(int(np.sum(shape * ranks)))
        self._chk(self.lib.ref_random_model(C.c_uint32(len(shape)), _p(shape), _p(ranks),
                                            C.c_uint64(seed), _p(core), _p(fc)))
        return core, model_split(shape, ranks, fc)

    def time_sweep_phases(self, shape, ranks, core, factors, lam, x, s, seed, mode,
                          gram_samples, svd_dim, do_factor=True, do_loss=True):
        o, shape, ranks, core, fc = self._margs(shape, ranks, core, factors)
        out = np.zeros(6)
        self._chk(self.lib.ref_time_sweep_phases(o, _p(shape), _p(ranks), _p(core), _p(fc),
                                                 C.c_double(lam), _p(_f64(x).ravel()),
                                                 C.c_uint64(s), C.c_uint64(seed),
                                                 C.c_uint32(mode), C.c_uint64(gram_samples),
                                                 C.c_uint64(svd_dim), C.c_int(int(do_factor)),
                                                 C.c_int(int(do_loss)), _p(out)))
        return out

    def aug_sketch(self, a, b, cand, lam, d_eff_lower, s, seed):
        """The RowSketch of the reference's approximate_ridge_regression (ref_aug_sketch)."""
        a, b, cand = _f64(a), _f64(b), _f64(cand)
        n, d = a.shape
        idx, w = np.zeros(s, np.uint64), np.zeros(s)
        self._chk(self.lib.ref_aug_sketch(_p(a), C.c_uint64(n), C.c_uint64(d), _p(b), _p(cand),
                                          C.c_double(lam), C.c_double(d_eff_lower),
                                          C.c_uint64(s), C.c_uint64(seed), _p(idx), _p(w)))
        return idx, w

    def time_core_fast(self, shape, ranks, core, factors, lam, x, s, seed):
        """The reference's own update_core_fast, timed inside the harness (ref_time_core_fast):
        [total, setup, draw, gather, solve, data_rows]."""
        o, shape, ranks, core, fc = self._margs(shape, ranks, core, factors)
        out = np.zeros(6)
        self._chk(self.lib.ref_time_core_fast(o, _p(shape), _p(ranks), _p(core), _p(fc),
                                              C.c_double(lam), _p(_f64(x).ravel()),
                                              C.c_uint64(s), C.c_uint64(seed), _p(out)))
        return out

    def als(self, x, ranks, lam=1e-3, sketched_core=0, epsilon=0.1, delta=0.1, seed=0,
            max_iterations=50, tolerance=1e-6, sample_count_override=0, record_history=0):
        """rtucker_als_run through the reference C API; returns the same dict as Oracle.als."""
        x = _f64(x)
        L = self.lib
        shape = _u64(x.shape)
        ranks = _u64(ranks)
        t = C.c_void_p()
        self._capi(L.rtucker_tensor_create(_p(shape), C.c_uint32(len(shape)), _p(x.ravel()),
                                           C.byref(t)))
        opts = AlsOptions(lam, sketched_core, epsilon, delta, seed, max_iterations, tolerance,
                          sample_count_override, record_history)
        r = C.c_void_p()
        try:
            self._capi(L.rtucker_als_run(t, _p(ranks), C.c_uint32(len(ranks)), C.byref(opts),
                                         C.byref(r)))
        finally:
            L.rtucker_tensor_free(t)
        hist = []
        buf = C.create_string_buffer(32)
        for i in range(L.rtucker_result_history_size(r)):
            it, lo, rm = C.c_uint32(), C.c_double(), C.c_double()
            self._capi(L.rtucker_result_history_row(r, C.c_uint64(i), C.byref(it), buf, 32,
                                                    C.byref(lo), C.byref(rm)))
            hist.append((it.value, buf.value.decode(), lo.value, rm.value))
        m = C.c_void_p()
        self._capi(L.rtucker_result_model(r, C.byref(m)))
        # model internals are not exposed by the C API: reconstruct instead
        xt = C.c_void_p()
        self._capi(L.rtucker_model_reconstruct(m, C.byref(xt)))
        n = L.rtucker_tensor_size(xt)
        xhat = np.ctypeslib.as_array(L.rtucker_tensor_data(xt), shape=(n,)).copy()
        L.rtucker_tensor_free(xt)
        L.rtucker_model_free(m)
        out = {
            "history": hist,
            "iterations": L.rtucker_result_iterations(r),
            "final_loss": L.rtucker_result_final_loss(r),
            "final_rmse": L.rtucker_result_final_rmse(r),
            "reconstruction": xhat.reshape(x.shape),
        }
        L.rtucker_result_free(r)
        return out
