"""Python mirror of the rtucker C API, bound to librtucker_b200.so with ctypes.

This is the binding a Python user of the reference would write against
/root/reference/proj/include/rtucker.h; the same names,
argument meanings and status codes. Everything computes on the GPU; if the
shared library is missing this module raises at import (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RTB_LIB_PATH: developer experiments with variant builds (tools/varlib.sh builds one); never
# set in use
LIB_PATH = os.environ.get("RTB_LIB_PATH") or os.path.join(_HERE, "lib", "librtucker_b200.so")

OK, ERR_INVALID_ARGUMENT, ERR_IO, ERR_NUMERICAL, ERR_UNKNOWN = 0, 1, 2, 3, 4

_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p


class RtuckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"rtucker status {code}: {msg}")
        self.code = code
        self.msg = msg


class AlsOptions(C.Structure):
    """rtucker_als_options (rtucker.h; ref rtucker.h:58-68)."""

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


_ALLREDUCE = C.CFUNCTYPE(None, _f64p, C.c_uint64, C.c_void_p, C.c_void_p)


class AlsExt(C.Structure):
    """rtucker_b200_als_ext (include/rtucker_b200.h)."""

    _fields_ = [
        ("init_core", _f64p),
        ("init_factors", _f64p),
        ("shard_rank", C.c_uint32),
        ("shard_count", C.c_uint32),
        ("allreduce", _ALLREDUCE),
        ("allreduce_user", C.c_void_p),
        ("async_sweeps_when_no_tolerance", C.c_int),
        ("profile_kernels", C.c_int),
        ("core_solver", C.c_int),
        ("fast_loss", C.c_int),
        ("shard_rows_total", C.c_int),
        ("factor_samples", C.c_uint32),
        ("disable_graph", C.c_int),
        ("reserved", C.c_int * 2),
    ]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2107_10654_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    S = C.c_int  # rtucker_status
    sig = {
        "rtucker_version": (C.c_char_p, []),
        "rtucker_last_error": (C.c_char_p, []),
        "rtucker_tensor_create": (S, [_u64p, C.c_uint32, _f64p, C.POINTER(_vp)]),
        "rtucker_tensor_read": (S, [C.c_char_p, C.POINTER(_vp)]),
        "rtucker_tensor_read_csv": (S, [C.c_char_p, C.POINTER(_vp)]),
        "rtucker_tensor_write": (S, [_vp, C.c_char_p]),
        "rtucker_tensor_order": (C.c_uint32, [_vp]),
        "rtucker_tensor_shape": (S, [_vp, _u64p]),
        "rtucker_tensor_size": (C.c_uint64, [_vp]),
        "rtucker_tensor_data": (_f64p, [_vp]),
        "rtucker_tensor_free": (None, [_vp]),
        "rtucker_tensor_generate": (S, [_u64p, _u64p, C.c_uint32, C.c_double, C.c_double,
                                        C.c_uint64, C.POINTER(_vp), _u64p]),
        "rtucker_als_options_init": (None, [C.POINTER(AlsOptions)]),
        "rtucker_als_run": (S, [_vp, _u64p, C.c_uint32, C.POINTER(AlsOptions), C.POINTER(_vp)]),
        "rtucker_result_history_size": (C.c_uint64, [_vp]),
        "rtucker_result_history_row": (S, [_vp, C.c_uint64, C.POINTER(C.c_uint32), C.c_char_p,
                                           C.c_size_t, _f64p, _f64p]),
        "rtucker_result_timing_size": (C.c_uint64, [_vp]),
        "rtucker_result_timing_row": (S, [_vp, C.c_uint64, C.c_char_p, C.c_size_t, _f64p,
                                          _u64p]),
        "rtucker_result_final_loss": (C.c_double, [_vp]),
        "rtucker_result_final_rmse": (C.c_double, [_vp]),
        "rtucker_result_iterations": (C.c_uint32, [_vp]),
        "rtucker_result_model": (S, [_vp, C.POINTER(_vp)]),
        "rtucker_result_free": (None, [_vp]),
        "rtucker_model_write": (S, [_vp, C.c_char_p]),
        "rtucker_model_read": (S, [C.c_char_p, C.POINTER(_vp)]),
        "rtucker_model_reconstruct": (S, [_vp, C.POINTER(_vp)]),
        "rtucker_model_lambda": (C.c_double, [_vp]),
        "rtucker_model_order": (C.c_uint32, [_vp]),
        "rtucker_model_ranks": (S, [_vp, _u64p]),
        "rtucker_model_free": (None, [_vp]),
        "rtucker_solve_ridge": (S, [_f64p, C.c_uint64, C.c_uint64, _f64p, C.c_double, _f64p]),
        "rtucker_ridge_scores": (S, [_f64p, C.c_uint64, C.c_uint64, C.c_double, _f64p]),
        "rtucker_sketched_ridge": (S, [_f64p, C.c_uint64, C.c_uint64, _f64p, _f64p, C.c_double,
                                       C.c_double, C.c_double, C.c_double, C.c_uint64,
                                       C.c_uint64, _f64p, _u64p, _f64p]),
        "rtucker_verify_suite": (S, [C.c_char_p, C.c_uint64, C.POINTER(C.c_int),
                                     C.POINTER(C.c_char_p)]),
        "rtucker_string_free": (None, [C.c_char_p]),
        # extensions
        "rtucker_b200_set_device": (S, [C.c_int]),
        "rtucker_b200_set_stream": (S, [_vp]),
        "rtucker_b200_launch_count": (C.c_ulonglong, []),
        "rtucker_b200_variant_count": (C.c_ulonglong, [C.c_char_p]),
        "rtucker_b200_tensor_create_device": (S, [_u64p, C.c_uint32, _vp, C.POINTER(_vp)]),
        "rtucker_b200_tensor_device_data": (_vp, [_vp]),
        "rtucker_b200_tensor_generate_device": (S, [_u64p, _u64p, C.c_uint32, C.c_double, C.c_double,
                                                    C.c_uint64, C.c_uint32, C.c_uint32,
                                                    C.POINTER(_vp), _f64p, _f64p]),
        "rtucker_b200_als_run_ex": (S, [_vp, _u64p, C.c_uint32, C.POINTER(AlsOptions),
                                        C.POINTER(AlsExt), C.POINTER(_vp)]),
        "rtucker_b200_session_create": (S, [_vp, _u64p, C.c_uint32, C.POINTER(AlsOptions),
                                            C.POINTER(AlsExt), C.POINTER(_vp)]),
        "rtucker_b200_session_sweeps": (S, [_vp, C.c_uint32]),
        "rtucker_b200_session_result": (S, [_vp, C.POINTER(_vp)]),
        "rtucker_b200_session_free": (None, [_vp]),
        "rtucker_b200_result_sweep_seconds": (C.c_double, [_vp]),
        "rtucker_b200_result_graph_sweeps": (C.c_uint64, [_vp]),
        "rtucker_b200_model_data": (S, [_vp, _f64p, _f64p]),
        "rtucker_b200_model_create": (S, [_u64p, _u64p, C.c_uint32, _f64p, _f64p, C.c_double,
                                          C.POINTER(_vp)]),
        "rtucker_b200_result_sketch_info": (S, [_vp, _u64p, _u64p, C.POINTER(C.c_int),
                                                C.POINTER(C.c_int)]),
        "rtucker_b200_result_pcg_iterations": (C.c_int, [_vp]),
        "rtucker_b200_result_kernel_count": (C.c_uint64, [_vp]),
        "rtucker_b200_result_kernel_row": (S, [_vp, C.c_uint64, C.c_char_p, C.c_size_t, _f64p,
                                               _u64p]),
        "rtucker_b200_factor_scores": (S, [_f64p, C.c_uint64, C.c_uint64, _f64p, _f64p, _f64p,
                                           _u64p]),
        "rtucker_b200_kron_draw": (S, [C.c_uint32, _u64p, C.c_uint64, _f64p, _f64p, _f64p,
                                       C.c_uint64, C.c_uint64, _u64p, _f64p]),
        "rtucker_b200_kron_normal_eq": (S, [C.c_uint32, _u64p, _u64p, _f64p, _f64p, C.c_double,
                                            C.c_uint64, _u64p, _f64p, _f64p, _f64p]),
        "rtucker_b200_kron_fiber_sketch": (S, [_vp, _u64p, C.c_uint32, _vp, _vp, C.c_uint32,
                                               C.c_uint32, C.c_double, C.c_uint64, C.c_uint64,
                                               _vp, _vp, _u64p, _f64p, _u64p, _u64p, _f64p]),
        "rtucker_b200_tensor_fiber_major": (S, [_vp, _u64p, _vp]),
        "rtucker_b200_kron_fiber_sketch_shard": (S, [_vp, _u64p, C.c_uint32, _vp, _vp, C.c_uint32,
                                                     C.c_uint32, C.c_double, C.c_uint64,
                                                     C.c_uint64, _vp, _vp, _u64p, _f64p, _u64p,
                                                     _u64p, _f64p, C.c_uint32, C.c_uint32]),
        "rtucker_b200_sym_eig": (S, [_f64p, C.c_uint64, _f64p, _f64p]),
        "rtucker_b200_aug_draw": (S, [_f64p, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                      C.c_uint64, _u64p, _f64p]),
        "rtucker_b200_dense_normal_eq": (S, [_f64p, C.c_uint64, C.c_uint64, _f64p, C.c_double,
                                             C.c_uint64, _u64p, _f64p, _f64p, _f64p]),
        "rtucker_b200_sample_count": (S, [C.c_double, C.c_uint64, C.c_double, C.c_double,
                                          _u64p]),
        "rtucker_b200_spd_solve": (S, [_f64p, _f64p, C.c_uint64, _f64p, _u64p,
                                       C.POINTER(C.c_int)]),
        "rtucker_b200_update_core_sketched": (S, [_vp, _vp, C.c_uint64, C.c_uint64, _f64p, _u64p,
                                                  _f64p]),
        "rtucker_b200_update_factor": (S, [_vp, _vp, C.c_uint32, _f64p]),
        "rtucker_b200_update_core_exact": (S, [_vp, _vp, _f64p]),
        "rtucker_b200_loss": (S, [_vp, _vp, _f64p, _f64p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

# symbols the drop-in must export (include/rtucker.h)
REFERENCE_SYMBOLS = [
    "rtucker_version", "rtucker_last_error", "rtucker_tensor_create", "rtucker_tensor_read",
    "rtucker_tensor_read_csv", "rtucker_tensor_write", "rtucker_tensor_order",
    "rtucker_tensor_shape", "rtucker_tensor_size", "rtucker_tensor_data", "rtucker_tensor_free",
    "rtucker_tensor_generate", "rtucker_als_options_init", "rtucker_als_run",
    "rtucker_result_history_size", "rtucker_result_history_row", "rtucker_result_timing_size",
    "rtucker_result_timing_row", "rtucker_result_final_loss", "rtucker_result_final_rmse",
    "rtucker_result_iterations", "rtucker_result_model", "rtucker_result_free",
    "rtucker_model_write", "rtucker_model_read", "rtucker_model_reconstruct",
    "rtucker_model_lambda", "rtucker_model_order", "rtucker_model_ranks", "rtucker_model_free",
    "rtucker_solve_ridge", "rtucker_ridge_scores", "rtucker_sketched_ridge",
    "rtucker_verify_suite", "rtucker_string_free",
]


def _check(rc: int) -> None:
    if rc != OK:
        raise RtuckerError(rc, lib.rtucker_last_error().decode())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _p(a):
    if a is None:
        return None
    if a.dtype == np.float64:
        return a.ctypes.data_as(_f64p)
    if a.dtype == np.uint64:
        return a.ctypes.data_as(_u64p)
    raise TypeError(a.dtype)


def options(**kw) -> AlsOptions:
    """rtucker_als_options_init defaults (ref capi.cpp:163-174) with overrides."""
    o = AlsOptions()
    lib.rtucker_als_options_init(C.byref(o))
    for k, v in kw.items():
        setattr(o, "lambda_" if k in ("lam", "lambda_") else k, v)
    return o


def _own(handle):
    """Copy a handle value (callers may reuse their c_void_p out-parameter)."""
    return C.c_void_p(handle.value if isinstance(handle, C.c_void_p) else handle)


class Tensor:
    """rtucker_tensor handle (host + resident device copy)."""

    def __init__(self, handle):
        self.h = _own(handle)

    @classmethod
    def from_numpy(cls, x) -> "Tensor":
        x = _f64(x)
        shape = _u64(x.shape)
        h = _vp()
        _check(lib.rtucker_tensor_create(_p(shape), len(x.shape), _p(x.reshape(-1)), C.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, ptr: int, shape) -> "Tensor":
        shape = _u64(shape)
        h = _vp()
        _check(lib.rtucker_b200_tensor_create_device(_p(shape), len(shape), _vp(ptr), C.byref(h)))
        return cls(h)

    @classmethod
    def generate(cls, shape, planted_ranks, noise_fraction, noise_sigma, seed):
        shape, pr = _u64(shape), _u64(planted_ranks)
        h = _vp()
        ck = C.c_uint64()
        _check(lib.rtucker_tensor_generate(_p(shape), _p(pr), len(shape), noise_fraction,
                                           noise_sigma, seed, C.byref(h), C.byref(ck)))
        return cls(h), ck.value

    @classmethod
    def generate_device(cls, shape, planted_ranks, noise_level, seed, pareto_alpha=0.0,
                        shard=(0, 1), want_model=False):
        """Planted tensor generated on the GPU (rtucker_b200_tensor_generate_device); with
        want_model, also (core, factors) of the planted model."""
        shape, pr = _u64(shape), _u64(planted_ranks)
        h = _vp()
        core = np.zeros(int(np.prod(pr))) if want_model else None
        fac = np.zeros(int(np.sum(shape * pr))) if want_model else None
        _check(lib.rtucker_b200_tensor_generate_device(_p(shape), _p(pr), len(shape),
                                                       noise_level, pareto_alpha, seed, shard[0],
                                                       shard[1], C.byref(h), _p(core), _p(fac)))
        t = cls(h)
        if not want_model:
            return t
        fs, off = [], 0
        for i, r in zip(shape, pr):
            fs.append(fac[off:off + int(i * r)].reshape(int(i), int(r)))
            off += int(i * r)
        return t, core.reshape(tuple(int(r) for r in pr)), fs

    @property
    def shape(self):
        n = lib.rtucker_tensor_order(self.h)
        out = np.zeros(n, np.uint64)
        _check(lib.rtucker_tensor_shape(self.h, _p(out)))
        return tuple(int(v) for v in out)

    @property
    def size(self) -> int:
        return int(lib.rtucker_tensor_size(self.h))

    def numpy(self) -> np.ndarray:
        p = lib.rtucker_tensor_data(self.h)
        if not p:
            raise RtuckerError(ERR_INVALID_ARGUMENT, lib.rtucker_last_error().decode())
        return np.ctypeslib.as_array(p, shape=(self.size,)).reshape(self.shape).copy()

    def free(self):
        if self.h:
            lib.rtucker_tensor_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


@dataclass
class Model:
    core: np.ndarray
    factors: list
    lam: float

    def handle(self):
        shape = _u64([f.shape[0] for f in self.factors])
        ranks = _u64([f.shape[1] for f in self.factors])
        fc = _f64(np.concatenate([_f64(f).ravel() for f in self.factors]))
        h = _vp()
        _check(lib.rtucker_b200_model_create(_p(shape), _p(ranks), len(shape),
                                             _p(_f64(self.core).ravel()), _p(fc),
                                             C.c_double(self.lam), C.byref(h)))
        return h


def _model_from_handle(h) -> Model:
    n = lib.rtucker_model_order(h)
    ranks = np.zeros(n, np.uint64)
    _check(lib.rtucker_model_ranks(h, _p(ranks)))
    return ranks, lib.rtucker_model_lambda(h)


class Result:
    """rtucker_als_result handle."""

    def __init__(self, h, shape):
        self.h = _own(h)
        self.shape = tuple(shape)

    def history(self):
        rows = []
        buf = C.create_string_buffer(32)
        for i in range(lib.rtucker_result_history_size(self.h)):
            it, lo, rm = C.c_uint32(), C.c_double(), C.c_double()
            _check(lib.rtucker_result_history_row(self.h, i, C.byref(it), buf, 32, C.byref(lo),
                                                  C.byref(rm)))
            rows.append((it.value, buf.value.decode(), lo.value, rm.value))
        return rows

    def timings(self):
        rows = []
        buf = C.create_string_buffer(32)
        for i in range(lib.rtucker_result_timing_size(self.h)):
            m, c = C.c_double(), C.c_uint64()
            _check(lib.rtucker_result_timing_row(self.h, i, buf, 32, C.byref(m), C.byref(c)))
            rows.append((buf.value.decode(), m.value, c.value))
        return rows

    def kernels(self):
        rows = []
        buf = C.create_string_buffer(64)
        for i in range(lib.rtucker_b200_result_kernel_count(self.h)):
            t, c = C.c_double(), C.c_uint64()
            _check(lib.rtucker_b200_result_kernel_row(self.h, i, buf, 64, C.byref(t), C.byref(c)))
            rows.append((buf.value.decode(), t.value, c.value))
        return rows

    def sketch_info(self):
        s, dd = C.c_uint64(), C.c_uint64()
        rd, sp = C.c_int(), C.c_int()
        _check(lib.rtucker_b200_result_sketch_info(self.h, C.byref(s), C.byref(dd), C.byref(rd),
                                                   C.byref(sp)))
        return {"sample_count": s.value, "data_draws": dd.value, "rank_deficient": rd.value,
                "solver_path": sp.value,
                "pcg_iterations": lib.rtucker_b200_result_pcg_iterations(self.h)}

    @property
    def final_loss(self) -> float:
        return lib.rtucker_result_final_loss(self.h)

    @property
    def final_rmse(self) -> float:
        return lib.rtucker_result_final_rmse(self.h)

    @property
    def iterations(self) -> int:
        return lib.rtucker_result_iterations(self.h)

    @property
    def graph_sweeps(self) -> int:
        return int(lib.rtucker_b200_result_graph_sweeps(self.h))

    @property
    def sweep_seconds(self) -> float:
        return lib.rtucker_b200_result_sweep_seconds(self.h)

    def model(self) -> Model:
        m = _vp()
        _check(lib.rtucker_result_model(self.h, C.byref(m)))
        try:
            ranks, lam = _model_from_handle(m)
            core = np.zeros(int(np.prod(ranks)))
            fsz = int(sum(int(i) * int(r) for i, r in zip(self.shape, ranks)))
            fc = np.zeros(fsz)
            _check(lib.rtucker_b200_model_data(m, _p(core), _p(fc)))
        finally:
            lib.rtucker_model_free(m)
        factors, off = [], 0
        for i, r in zip(self.shape, ranks):
            factors.append(fc[off:off + int(i) * int(r)].reshape(int(i), int(r)))
            off += int(i) * int(r)
        return Model(core.reshape(tuple(int(r) for r in ranks)), factors, lam)

    def free(self):
        if self.h:
            lib.rtucker_result_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def shard_rows(rank: int, count: int, rows_total: int):
    """Rows [lo, hi) of mode 1 held by shard `rank` of `count` (the library's even split)."""
    return rank * rows_total // count, (rank + 1) * rows_total // count


@dataclass
class Shard:
    """Multi-GPU run: X split along mode 1. `allreduce(ptr, count, stream)` must sum
    `count` doubles at device address `ptr` across all shards, in place, ordered after
    the work already enqueued on `stream` (e.g. an NCCL all-reduce)."""
    rank: int
    count: int
    rows_total: int
    allreduce: object


def _ext(init_model: Model | None = None, profile: bool = False, core_solver: int = 0,
         fast_loss: bool = False, shard: Shard | None = None, factor_samples: int = 0,
         graph: bool = True):
    ext = AlsExt()
    ext.disable_graph = 0 if graph else 1
    ext.core_solver = int(core_solver)
    ext.fast_loss = int(fast_loss)
    ext.factor_samples = int(factor_samples)
    keep = []
    if shard is not None:
        fn = shard.allreduce

        def _cb(ptr, n, stream, user):
            try:
                fn(C.cast(ptr, C.c_void_p).value, int(n), int(stream or 0))
            except Exception as e:  # a callback cannot raise into C
                import traceback
                traceback.print_exc()
                raise SystemExit(f"allreduce callback failed: {e}")
        cb = _ALLREDUCE(_cb)
        keep.append(cb)
        ext.shard_rank = shard.rank
        ext.shard_count = shard.count
        ext.shard_rows_total = shard.rows_total
        ext.allreduce = cb
    if init_model is not None:
        core = _f64(init_model.core).ravel()
        fc = _f64(np.concatenate([_f64(f).ravel() for f in init_model.factors]))
        keep += [core, fc]
        ext.init_core = _p(core)
        ext.init_factors = _p(fc)
    ext.profile_kernels = int(profile)
    return ext, keep


def als_run(x: Tensor, ranks, opts: AlsOptions | None = None, init_model: Model | None = None,
            profile: bool = False, core_solver: int = 0, fast_loss: bool = False,
            shard: Shard | None = None, factor_samples: int = 0, graph: bool = True) -> Result:
    """rtucker_als_run (ref capi.cpp:176-201); extensions via rtucker_b200_als_run_ex.
    With `shard`, `x` holds only that shard's rows of mode 1 (see shard_rows).
    factor_samples > 0: sketched factor updates with that many draws (perf mode)."""
    opts = opts or options()
    ranks = _u64(ranks)
    r = _vp()
    shape = tuple(x.shape)
    if shard is not None:
        shape = (shard.rows_total,) + shape[1:]
    if (init_model is None and not profile and not core_solver and not fast_loss and shard is None
            and not factor_samples and graph):
        _check(lib.rtucker_als_run(x.h, _p(ranks), len(ranks), C.byref(opts), C.byref(r)))
    else:
        ext, keep = _ext(init_model, profile, core_solver, fast_loss, shard, factor_samples,
                         graph)
        _check(lib.rtucker_b200_als_run_ex(x.h, _p(ranks), len(ranks), C.byref(opts),
                                           C.byref(ext), C.byref(r)))
        del keep
    return Result(r, shape)


class Session:
    """Step-wise run (rtucker_b200_session_*): init at construction, sweeps on demand."""

    def __init__(self, x: Tensor, ranks, opts: AlsOptions | None = None,
                 init_model: Model | None = None, profile: bool = False, core_solver: int = 0,
                 shard: Shard | None = None, factor_samples: int = 0, graph: bool = True):
        self.shape = tuple(x.shape)
        if shard is not None:
            self.shape = (shard.rows_total,) + self.shape[1:]
        opts = opts or options()
        ranks = _u64(ranks)
        ext, self._keep = _ext(init_model, profile, core_solver, False, shard, factor_samples,
                               graph)
        self.h = _vp()
        _check(lib.rtucker_b200_session_create(x.h, _p(ranks), len(ranks), C.byref(opts),
                                               C.byref(ext), C.byref(self.h)))

    def sweeps(self, n: int) -> None:
        _check(lib.rtucker_b200_session_sweeps(self.h, n))

    def result(self) -> Result:
        r = _vp()
        _check(lib.rtucker_b200_session_result(self.h, C.byref(r)))
        return Result(r, self.shape)

    def free(self):
        if self.h:
            lib.rtucker_b200_session_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def variant_count(name: str) -> int:
    """Launches so far of a named headline kernel variant (e.g. "k_ttm_mid3")."""
    return int(lib.rtucker_b200_variant_count(name.encode()))


def set_stream(stream_ptr: int | None) -> None:
    _check(lib.rtucker_b200_set_stream(_vp(stream_ptr or 0)))


# ---- ridge toolkit (ref rtucker.h:104-122) ----

def solve_ridge(a, b, lam: float) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    x = np.zeros(a.shape[1])
    _check(lib.rtucker_solve_ridge(_p(a), a.shape[0], a.shape[1], _p(b), lam, _p(x)))
    return x


def ridge_scores(a, lam: float) -> np.ndarray:
    a = _f64(a)
    out = np.zeros(a.shape[0])
    _check(lib.rtucker_ridge_scores(_p(a), a.shape[0], a.shape[1], lam, _p(out)))
    return out


def sketched_ridge(a, b, candidate_scores, lam, d_eff_lower, epsilon, delta,
                   sample_count_override, seed):
    a, b = _f64(a), _f64(b)
    x = np.zeros(a.shape[1])
    s, bp = C.c_uint64(), C.c_double()
    cs = None if candidate_scores is None else _f64(candidate_scores)
    _check(lib.rtucker_sketched_ridge(_p(a), a.shape[0], a.shape[1], _p(b), _p(cs), lam,
                                      d_eff_lower, epsilon, delta, sample_count_override, seed,
                                      _p(x), C.byref(s), C.byref(bp)))
    return x, s.value, bp.value


# ---- parity-ladder entry points (include/rtucker_b200.h) ----

def factor_scores(f):
    f = _f64(f)
    rows, cols = f.shape
    sc, cdf = np.zeros(rows), np.zeros(rows)
    tot, rank = C.c_double(), C.c_uint64()
    _check(lib.rtucker_b200_factor_scores(_p(f), rows, cols, _p(sc), _p(cdf), C.byref(tot),
                                          C.byref(rank)))
    return sc, cdf, tot.value, rank.value


def kron_draw(rows, d, scores_list, cdf_list, sums, seed, s):
    rows = _u64(rows)
    sc = _f64(np.concatenate(scores_list))
    cdf = _f64(np.concatenate(cdf_list))
    sums = _f64(sums)
    idx, w = np.zeros(s, np.uint64), np.zeros(s)
    _check(lib.rtucker_b200_kron_draw(len(rows), _p(rows), d, _p(sc), _p(cdf), _p(sums), seed, s,
                                      _p(idx), _p(w)))
    return idx, w


def kron_normal_eq(shape, ranks, factors, x, lam, idx, w):
    shape, ranks = _u64(shape), _u64(ranks)
    fc = _f64(np.concatenate([_f64(f).ravel() for f in factors]))
    d = int(np.prod(ranks))
    g, rhs = np.zeros((d, d)), np.zeros(d)
    idx, w = _u64(idx), _f64(w)
    _check(lib.rtucker_b200_kron_normal_eq(len(shape), _p(shape), _p(ranks), _p(fc),
                                           _p(_f64(x).ravel()), lam, len(idx), _p(idx), _p(w),
                                           _p(g), _p(rhs)))
    return g, rhs


def kron_fiber_sketch(x_ptr, shape, a2_ptr, a3_ptr, r2, r3, lam, s, seed, gram_ptr=None,
                      rhs_ptr=None, want_draws=False, fiber_major=False, shard=(0, 1)):
    """BASELINE C4 microbench on device pointers (rtucker_b200_kron_fiber_sketch_shard):
    X (I1 x I2 x I3 FP32; canonical row-major, or fiber-major when fiber_major), A2 (I2 x r2),
    A3 (I3 x r3) FP64; gram (W x W) and rhs (W x I1) FP64 outputs, W = r2 r3. shard = (rank,
    count): this shard's partial sums (j2 range), to be summed over the shards.
    Returns {data_draws, unique_rows, phase_ms, [indices, weights]}."""
    shape = _u64(shape)
    idx = np.zeros(s, np.uint64) if want_draws else None
    w = np.zeros(s) if want_draws else None
    nd, nu = C.c_uint64(), C.c_uint64()
    ms = np.zeros(3)
    _check(lib.rtucker_b200_kron_fiber_sketch_shard(
        C.c_void_p(x_ptr or 0), _p(shape), 1 if fiber_major else 0, C.c_void_p(a2_ptr),
        C.c_void_p(a3_ptr), r2, r3, lam, s, seed, C.c_void_p(gram_ptr or 0),
        C.c_void_p(rhs_ptr or 0), _p(idx) if want_draws else None, _p(w) if want_draws else None,
        C.byref(nd), C.byref(nu), _p(ms), int(shard[0]), int(shard[1])))
    out = {"data_draws": nd.value, "unique_rows": nu.value, "phase_ms": ms.tolist()}
    if want_draws:
        out["indices"], out["weights"] = idx, w
    return out


def tensor_fiber_major(x_ptr, shape, out_ptr):
    """Fiber-major copy (mode 1 fastest) of a device FP32 I1 x I2 x I3 tensor
    (rtucker_b200_tensor_fiber_major)."""
    shape = _u64(shape)
    _check(lib.rtucker_b200_tensor_fiber_major(C.c_void_p(x_ptr), _p(shape), C.c_void_p(out_ptr)))


def aug_draw(candidate_scores, d, d_eff_lower, seed, s):
    """Dense-toolkit RowSketch (AugmentedSampler) drawn on the GPU."""
    cand = _f64(candidate_scores)
    idx, w = np.zeros(s, np.uint64), np.zeros(s)
    _check(lib.rtucker_b200_aug_draw(_p(cand), len(cand), d, d_eff_lower, seed, s, _p(idx),
                                     _p(w)))
    return idx, w


def dense_normal_eq(a, b, lam, idx, w):
    a, b = _f64(a), _f64(b)
    n, d = a.shape
    idx, w = _u64(idx), _f64(w)
    g, rhs = np.zeros((d, d)), np.zeros(d)
    _check(lib.rtucker_b200_dense_normal_eq(_p(a), n, d, _p(b), lam, len(idx), _p(idx), _p(w),
                                            _p(g), _p(rhs)))
    return g, rhs


def sample_count(beta_prime, d, epsilon, delta) -> int:
    out = np.zeros(1, np.uint64)
    _check(lib.rtucker_b200_sample_count(beta_prime, d, epsilon, delta, _p(out)))
    return int(out[0])


def sym_eig(a):
    """(evals non-increasing, evecs with eigenvector k in column k) on the GPU."""
    a = _f64(a)
    d = a.shape[0]
    ev, vec = np.zeros(d), np.zeros((d, d))
    _check(lib.rtucker_b200_sym_eig(_p(a), d, _p(ev), _p(vec)))
    return ev, vec


def spd_solve(g, rhs):
    g, rhs = _f64(g), _f64(rhs)
    x = np.zeros(len(rhs))
    rank, path = C.c_uint64(), C.c_int()
    _check(lib.rtucker_b200_spd_solve(_p(g), _p(rhs), len(rhs), _p(x), C.byref(rank),
                                      C.byref(path)))
    return x, rank.value, path.value


def update_core_sketched(x: Tensor, model: Model, s: int, seed: int):
    h = model.handle()
    try:
        core = np.zeros(int(np.prod(model.core.shape)))
        idx, w = np.zeros(s, np.uint64), np.zeros(s)
        _check(lib.rtucker_b200_update_core_sketched(x.h, h, s, seed, _p(core), _p(idx), _p(w)))
    finally:
        lib.rtucker_model_free(h)
    return core, idx, w


def update_factor(x: Tensor, model: Model, mode: int):
    h = model.handle()
    try:
        f = model.factors[mode - 1]
        out = np.zeros(f.shape)
        _check(lib.rtucker_b200_update_factor(x.h, h, mode, _p(out)))
    finally:
        lib.rtucker_model_free(h)
    return out


def update_core_exact(x: Tensor, model: Model):
    h = model.handle()
    try:
        core = np.zeros(int(np.prod(model.core.shape)))
        _check(lib.rtucker_b200_update_core_exact(x.h, h, _p(core)))
    finally:
        lib.rtucker_model_free(h)
    return core


def loss(x: Tensor, model: Model):
    h = model.handle()
    try:
        lo, rm = C.c_double(), C.c_double()
        _check(lib.rtucker_b200_loss(x.h, h, C.byref(lo), C.byref(rm)))
    finally:
        lib.rtucker_model_free(h)
    return lo.value, rm.value


class DeviceArray:
    """A raw device pointer viewed through __cuda_array_interface__ (float64, 1-D), so
    frameworks (torch.as_tensor) can wrap library buffers without a copy."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3, "stream": None}


def torch_allreduce(dist, group=None):
    """Shard.allreduce over torch.distributed for device buffers (NCCL): the library's
    buffer is wrapped without a copy and summed in place. Run the library on torch's
    current stream (set_stream) so the collective is ordered after its kernels."""
    import torch

    def fn(ptr, count, stream):
        t = torch.as_tensor(DeviceArray(ptr, count), device="cuda")
        dist.all_reduce(t, group=group)
    return fn


def host_allreduce(dist, group=None):
    """The same contract for host buffers (gloo): sums `count` doubles at host address
    `ptr` across the process group, in place."""
    import torch

    def fn(ptr, count, stream):
        arr = np.ctypeslib.as_array((C.c_double * count).from_address(ptr))
        dist.all_reduce(torch.from_numpy(arr), group=group)
    return fn
