"""Mode-1 sharded ALS (the multi-GPU path) on one GPU: P host threads, each driving
its own shard of X through the C ABI on the library's shared stream (so kernels of
different shards serialise and never wait on each other), with a host-side
allreduce callback standing in for NCCL. The sharded run must reproduce the
single-process run (same draws; sums regrouped across shards)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def planted(shape, ranks, noise=0.01, seed=0):
    """N(0,1) core and factors, dense noise at noise * ||X|| / sqrt(N)."""
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    factors = [rng.standard_normal((i, r)) for i, r in zip(shape, ranks)]
    x = core
    for n, f in enumerate(factors):
        x = np.moveaxis(np.tensordot(f, x, axes=(1, n)), 0, n)
    sigma = noise * np.linalg.norm(x) / np.sqrt(x.size)
    return x + sigma * rng.standard_normal(x.shape)


class HostAllreduce:
    """Sum `count` doubles at a device address across P threads, fixed shard order."""

    def __init__(self, n):
        import torch
        self.torch = torch
        self.n = n
        self.barrier = threading.Barrier(n)
        self.slots = [None] * n
        self.calls = [0] * n

    def fn(self, rank):
        torch = self.torch

        def allreduce(ptr, count, stream):
            from paper_2107_10654_b200 import rtucker as rt
            torch.cuda.ExternalStream(stream).synchronize() if stream else torch.cuda.synchronize()
            t = torch.as_tensor(rt.DeviceArray(ptr, count), device="cuda")
            self.slots[rank] = t.cpu()
            self.calls[rank] += 1
            self.barrier.wait()
            tot = self.slots[0].clone()
            for k in range(1, self.n):
                tot += self.slots[k]
            t.copy_(tot.to("cuda"))
            torch.cuda.synchronize()
            self.barrier.wait()
        return allreduce


def run_sharded(rt, x, ranks, kw, P, **extra):
    ar = HostAllreduce(P)
    out = [None] * P
    err = []

    def worker(r):
        try:
            lo, hi = rt.shard_rows(r, P, x.shape[0])
            xt = rt.Tensor.from_numpy(np.ascontiguousarray(x[lo:hi]))
            res = rt.als_run(xt, ranks, rt.options(**kw),
                             shard=rt.Shard(r, P, x.shape[0], ar.fn(r)), **extra)
            out[r] = (res.history(), res.model(), res.sketch_info())
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            ar.barrier.abort()
    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    assert len(set(ar.calls)) == 1, ar.calls  # every shard made the same collective calls
    return out


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("sketched", [1, 0])
def test_sharded_als_matches_single_process(rt, P, sketched):
    shape, ranks = (36, 30, 28), (4, 3, 5)
    x = planted(shape, ranks, seed=41)
    kw = dict(lam=1e-2, sketched_core=sketched, sample_count_override=6000, max_iterations=3,
              tolerance=0.0, record_history=1, seed=6)
    ref = rt.als_run(rt.Tensor.from_numpy(x), ranks, rt.options(**kw))
    outs = run_sharded(rt, x, ranks, kw, P)
    rh = ref.history()
    rm = ref.model()
    # exact: 1e-9; sketched: the regrouped Gram sums pass through the ill-conditioned
    # early-sweep solves (kappa up to ~1e8 from the uniform init), ~1e-9..1e-8
    tol = 1e-9 if not sketched else 1e-7
    for hist, model, info in outs:
        assert [(h[0], h[1]) for h in hist] == [(h[0], h[1]) for h in rh]
        for (gi, gs, gl, grm), (_, _, fl, frm) in zip(hist, rh):
            assert abs(gl - fl) / fl < tol, (gi, gs, gl, fl)
        for a, b in zip(model.factors, rm.factors):
            assert np.linalg.norm(a - b) / np.linalg.norm(b) < 100 * tol
        assert np.linalg.norm(model.core - rm.core) / np.linalg.norm(rm.core) < 100 * tol
    # the shards' data draws partition the sketch's data draws
    if sketched:
        assert sum(o[2]["data_draws"] for o in outs) == ref.sketch_info()["data_draws"]


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_order4_bucketed_path(rt, P):
    """Order 4 with draws >> (i1, i2) pairs: the (i1, i2)-bucketed Gram (k_gram.cu,
    sketch_normal_eq_m4) restricted to this shard's i1 rows (BASELINE config 3 across GPUs)."""
    shape, ranks = (20, 18, 16, 14), (3, 3, 2, 2)
    x = planted(shape, ranks, seed=43)
    kw = dict(lam=0.1, sketched_core=1, sample_count_override=20000, max_iterations=3,
              tolerance=0.0, record_history=1, seed=7)
    ref = rt.als_run(rt.Tensor.from_numpy(x), ranks, rt.options(**kw))
    outs = run_sharded(rt, x, ranks, kw, P)
    rh, rm = ref.history(), ref.model()
    for hist, model, info in outs:
        assert [(h[0], h[1]) for h in hist] == [(h[0], h[1]) for h in rh]
        for (gi, gs, gl, grm), (_, _, fl, frm) in zip(hist, rh):
            assert abs(gl - fl) / fl < 1e-7, (gi, gs, gl, fl)
        assert np.linalg.norm(model.core - rm.core) / np.linalg.norm(rm.core) < 1e-5
    assert sum(o[2]["data_draws"] for o in outs) == ref.sketch_info()["data_draws"]


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("order", [3, 4])
def test_sharded_factor_sketch_matches_single_process(rt, P, order):
    """Sketched factor updates (perf mode) across shards: mode 1's sampled fibers are split
    into the shards' segments (own rows of A_1, stitched), the other modes' fibers are
    gathered by the shard owning their i_1 and the partial Gram / M all-reduced; augmented rows
    count on shard 0 only. Same draws on every shard, so the result is the single-process one
    up to the regrouped sums."""
    if order == 3:
        shape, ranks, fs = (36, 30, 28), (4, 3, 5), 3000
    else:
        shape, ranks, fs = (20, 18, 16, 14), (3, 3, 2, 2), 4000
    x = planted(shape, ranks, seed=44)
    kw = dict(lam=1e-2, sketched_core=1, sample_count_override=8000, max_iterations=3,
              tolerance=0.0, record_history=1, seed=9)
    ref = rt.als_run(rt.Tensor.from_numpy(x), ranks, rt.options(**kw), factor_samples=fs)
    outs = run_sharded(rt, x, ranks, kw, P, factor_samples=fs)
    rh, rm = ref.history(), ref.model()
    for hist, model, info in outs:
        assert [(h[0], h[1]) for h in hist] == [(h[0], h[1]) for h in rh]
        for (gi, gs, gl, grm), (_, _, fl, frm) in zip(hist, rh):
            assert abs(gl - fl) / fl < 1e-7, (gi, gs, gl, fl)
        for a, b in zip(model.factors, rm.factors):
            assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-5
        assert np.linalg.norm(model.core - rm.core) / np.linalg.norm(rm.core) < 1e-5


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("shape,ranks,s", [((40, 36, 34), (8, 32, 32), 400000),
                                           ((24, 22, 20, 18), (10, 10, 10, 10), 500000)])
def test_sharded_distributed_core_solve(rt, P, shape, ranks, s):
    """Large d under sharding: the core solve is distributed by mode-1 slices
    (pcg_solve_dist: each shard expands and multiplies its own slices' blocks -- the tiled
    rank-32 matvec at d = 8192, the order-4 one at d = 10^4 -- and the matvec shares are
    all-reduced every iteration); every shard ends with the single-process core up to the
    regrouped sums."""
    x = planted(shape, ranks, seed=45)
    kw = dict(lam=1e-2, sketched_core=1, sample_count_override=s, max_iterations=2,
              tolerance=0.0, record_history=1, seed=10)
    before = rt.variant_count("k_pcg_dist")
    ref = rt.als_run(rt.Tensor.from_numpy(x), ranks, rt.options(**kw))
    outs = run_sharded(rt, x, ranks, kw, P)
    assert rt.variant_count("k_pcg_dist") >= before + P, "sharded solve was not distributed"
    rh, rm = ref.history(), ref.model()
    for hist, model, info in outs:
        assert info["solver_path"] == 2  # the CG answer was accepted
        for (gi, gs, gl, grm), (_, _, fl, frm) in zip(hist, rh):
            assert abs(gl - fl) / fl < 1e-8, (gi, gs, gl, fl)
        assert np.linalg.norm(model.core - rm.core) / np.linalg.norm(rm.core) < 1e-7
    # every shard holds the same model
    for o in outs[1:]:
        assert np.array_equal(o[1].core, outs[0][1].core)


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_c2_rank16_split_pcg(rt, P):
    """Rank (16,16,16) under sharding (the C2 shape class): the replicated core solve is the
    split-role PCG on the all-reduced compact Gram (k_pcg_split, no block expansion), as in
    the single-process run."""
    shape, ranks = (48, 40, 36), (16, 16, 16)
    x = planted(shape, ranks, seed=47)
    kw = dict(lam=1e-2, sketched_core=1, sample_count_override=120000, max_iterations=2,
              tolerance=0.0, record_history=1, seed=12)
    ref = rt.als_run(rt.Tensor.from_numpy(x), ranks, rt.options(**kw))
    before = rt.variant_count("k_pcg_split")
    outs = run_sharded(rt, x, ranks, kw, P)
    assert rt.variant_count("k_pcg_split") >= before + P, "sharded C2 solve did not take k_pcg_split"
    rh, rm = ref.history(), ref.model()
    assert ref.sketch_info()["solver_path"] == 2
    for hist, model, info in outs:
        assert info["solver_path"] == 2  # the CG answer was accepted
        for (gi, gs, gl, grm), (_, _, fl, frm) in zip(hist, rh):
            assert abs(gl - fl) / fl < 1e-8, (gi, gs, gl, fl)
        assert np.linalg.norm(model.core - rm.core) / np.linalg.norm(rm.core) < 1e-7
    for o in outs[1:]:
        assert np.array_equal(o[1].core, outs[0][1].core)


def test_sharded_rejects_bad_split(rt):
    x = planted((20, 10, 8), (2, 2, 2), seed=1)
    with pytest.raises(rt.RtuckerError):
        rt.als_run(rt.Tensor.from_numpy(x[:7]), (2, 2, 2), rt.options(max_iterations=1),
                   shard=rt.Shard(0, 2, 20, lambda p, n, s: None))


_NCCL_CB = r"""
import os, sys
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["RTB_ROOT"])
from paper_2107_10654_b200 import rtucker as rt
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % int(os.environ["RTB_PORT"]),
                        rank=0, world_size=1, device_id=torch.device("cuda", 0))
fn = rt.torch_allreduce(dist)
stream = torch.cuda.current_stream()
rt.set_stream(stream.cuda_stream)
buf = torch.arange(1000, dtype=torch.float64, device="cuda") * 0.5
want = buf.clone()
# the library hands the callback a raw device address, a count and its stream
fn(buf.data_ptr() + 8 * 10, 900, stream.cuda_stream)
torch.cuda.synchronize()
assert torch.equal(buf, want), "a one-rank NCCL sum must leave the buffer unchanged"
# and through the C ABI: with the callback installed the library takes its sharded path (one
# shard: every partial sum goes through the NCCL all-reduce) and must reproduce the plain run
import numpy as np
rng = np.random.default_rng(3)
x = rng.standard_normal((20, 18, 16))
kw = dict(lam=1e-2, sketched_core=1, sample_count_override=3000, max_iterations=2,
          tolerance=0.0, record_history=1, seed=5)
a = rt.als_run(rt.Tensor.from_numpy(x), (3, 3, 3), rt.options(**kw))
b = rt.als_run(rt.Tensor.from_numpy(x), (3, 3, 3), rt.options(**kw),
               shard=rt.Shard(0, 1, 20, fn))
ha, hb = a.history(), b.history()
assert len(ha) == len(hb) and len(ha) > 0
for p, q in zip(ha, hb):
    assert p[:2] == q[:2]
    assert abs(p[2] - q[2]) <= 1e-9 * abs(p[2]), (p, q)
assert b.graph_sweeps == 0  # the sharded path runs kernel by kernel
dist.destroy_process_group()
print("nccl-callback-ok")
"""


def test_nccl_allreduce_callback_one_rank(rt):
    """bench.py's N > 1 plumbing (rt.torch_allreduce: raw device pointer -> torch view ->
    NCCL all-reduce in place on the library's stream) run for real on a one-rank NCCL group,
    in a child process so the process group does not outlive the test."""
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RTB_ROOT=root, RTB_PORT=str(port))
    p = subprocess.run([sys.executable, "-c", _NCCL_CB], env=env, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0 and "nccl-callback-ok" in p.stdout, p.stdout + p.stderr
