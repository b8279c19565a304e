"""World-size-2 gloo tests of the multi-GPU decomposition (runs on CPU).

The sharded engine splits X along mode 1 with
rtucker.shard_rows and meets every partial sum in a Shard.allreduce callback.
Here two gloo processes check the identities it relies on, with the reference
restatement as the arithmetic and the library's own host_allreduce callable as
the collective: (1) the row split partitions [0, I_1); (2) the mode-1
contraction of the X slabs sums to the full X x_1 A_1^T; (3) the normal
equations of the shard-local data draws plus the (replicated) augmented draws
sum to the full sketched normal equations; (4) the stitched A_1 rows (zero
elsewhere) sum to the full factor; (5) the perf-mode sketched factor update across shards:
mode 1's fibers split into the shards' row segments, the other modes' draws owned by the
shard of their i_1 (augmented rows on shard 0), partial Gram / M summed."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _planted(shape, ranks, seed):
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    fs = [rng.standard_normal((i, r)) for i, r in zip(shape, ranks)]
    x = core
    for n, f in enumerate(fs):
        x = np.moveaxis(np.tensordot(f, x, axes=(1, n)), 0, n)
    return x + 0.01 * rng.standard_normal(x.shape), core, fs


CASES = [((13, 9, 7), (3, 2, 2)), ((12, 9, 7, 6), (2, 3, 2, 2))]


def _worker(rank, world, port, q, case=0):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.oracle import Oracle
        from paper_2107_10654_b200 import rtucker as rt
        ar = rt.host_allreduce(dist)
        shape, ranks = CASES[case]
        x, core, fs = _planted(shape, ranks, 5)
        I1 = shape[0]
        lo, hi = rt.shard_rows(rank, world, I1)
        # (1) partition
        cov = np.zeros(I1)
        cov[lo:hi] = 1.0
        ar(cov.ctypes.data, cov.size, 0)
        assert np.array_equal(cov, np.ones(I1)), cov
        # (2) mode-1 projection from the slab with this shard's rows of A_1
        part = np.ascontiguousarray(np.tensordot(fs[0][lo:hi].T, x[lo:hi], axes=(1, 0)))
        ar(part.ctypes.data, part.size, 0)
        full = np.tensordot(fs[0].T, x, axes=(1, 0))
        assert np.allclose(part, full, rtol=1e-13, atol=1e-12)
        # (3) sketched normal equations: data draws split by i1, augmented draws once
        o = Oracle()
        # order 4: s above 2 I1 I2 (the library's (i1, i2)-bucketed path, whose shard split
        # is the same i1 ownership of the data draws)
        lam, s, seed = 0.05, 900 if len(shape) == 3 else 2500, 17
        _, idx, w, _ = o.update_core_fast(shape, ranks, core, fs, lam, x, s, seed)
        total = int(np.prod(shape))
        inner = total // I1
        data = idx < total
        own = data & (idx // inner >= lo) & (idx // inner < hi)
        g_own, r_own = o.kron_normal_eq(shape, ranks, fs, x, lam, idx[own], w[own])
        g_own = np.ascontiguousarray(g_own)
        r_own = np.ascontiguousarray(r_own)
        ar(g_own.ctypes.data, g_own.size, 0)
        ar(r_own.ctypes.data, r_own.size, 0)
        g_aug, _ = o.kron_normal_eq(shape, ranks, fs, x, lam, idx[~data], w[~data])
        g_all, r_all = o.kron_normal_eq(shape, ranks, fs, x, lam, idx, w)
        dg = np.sqrt(np.outer(np.diag(g_all), np.diag(g_all)))
        assert np.max(np.abs(g_own + g_aug - g_all) / dg) < 1e-12
        assert np.linalg.norm(r_own - r_all) / np.linalg.norm(r_all) < 1e-12
        # (4) A_1 stitched from shard rows
        a1 = np.zeros_like(fs[0])
        a1[lo:hi] = fs[0][lo:hi]
        ar(a1.ctypes.data, a1.size, 0)
        assert np.array_equal(a1, fs[0])
        # (5) sketched factor updates (perf mode) across shards, with the oracle's draws
        for mode in range(len(shape)):
            _fsk_decomposition(o, ar, rank, shape, ranks, core, fs, x, lo, hi, mode)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


def _fsk_normal_eq(shape, ranks, core, fs, x, lam, mode, idx, w, keep, rows=None):
    """Gram (R_n x R_n) and M (I_n x R_n) of the perf-mode factor sketch (k_fsketch.cu) over
    the draws selected by `keep`; `rows` restricts the fibers to mode-1 rows [lo, hi) (mode 1
    sharded)."""
    other = [m for m in range(len(shape)) if m != mode]
    total_o = int(np.prod([shape[m] for m in other]))
    gn = np.moveaxis(core, mode, 0).reshape(ranks[mode], -1)  # G_(n), other modes ascending
    rn = ranks[mode]
    G = np.zeros((rn, rn))
    M = np.zeros((shape[mode] if rows is None else rows[1] - rows[0], rn))
    for t in np.nonzero(keep)[0]:
        i = int(idx[t])
        if i >= total_o:
            j = i - total_o
            G[j, j] += lam * w[t] ** 2
            continue
        js, rem = [], i
        for m in reversed(other):
            js.append(rem % shape[m])
            rem //= shape[m]
        js = js[::-1]
        z = np.ones(1)
        for m, jm in zip(other, js):
            z = np.kron(z, fs[m][jm])
        k = gn @ z
        G += w[t] ** 2 * np.outer(k, k)
        sl = [slice(None)] * len(shape)
        for m, jm in zip(other, js):
            sl[m] = jm
        fib = x[tuple(sl)]
        if rows is not None:
            fib = fib[rows[0]:rows[1]]
        M += w[t] ** 2 * np.outer(fib, k)
    return G, M


def _fsk_decomposition(o, ar, rank, shape, ranks, core, fs, x, lo, hi, mode):
    lam, s, seed = 0.05, 600, 23
    new, idx, w = o.update_factor_sketched(shape, ranks, core, fs, lam, x, mode + 1, s, seed)
    allk = np.ones(s, bool)
    Gf, Mf = _fsk_normal_eq(shape, ranks, core, fs, x, lam, mode, idx, w, allk)
    # the restatement reproduces the oracle's update: A_n = M Gram^-1
    assert np.linalg.norm(Mf @ np.linalg.inv(Gf) - new) / np.linalg.norm(new) < 1e-10
    other = [m for m in range(len(shape)) if m != mode]
    total_o = int(np.prod([shape[m] for m in other]))
    if mode == 0:
        # fibers along the sharded mode: this shard's segments, the whole Gram everywhere
        G, M = _fsk_normal_eq(shape, ranks, core, fs, x, lam, 0, idx, w, allk, rows=(lo, hi))
        assert np.allclose(G, Gf, rtol=1e-13, atol=0)
        full = np.zeros_like(Mf)
        full[lo:hi] = M
        ar(full.ctypes.data, full.size, 0)
        assert np.allclose(full, Mf, rtol=1e-12, atol=1e-12 * np.abs(Mf).max())
    else:
        # the data draws of this shard's i_1 rows, the augmented rows on shard 0
        inner = total_o // shape[0]
        data = idx < total_o
        i1 = np.where(data, idx // inner, -1)
        keep = (data & (i1 >= lo) & (i1 < hi)) | (~data & (rank == 0))
        G, M = _fsk_normal_eq(shape, ranks, core, fs, x, lam, mode, idx, w, keep)
        G, M = np.ascontiguousarray(G), np.ascontiguousarray(M)
        ar(G.ctypes.data, G.size, 0)
        ar(M.ctypes.data, M.size, 0)
        assert np.allclose(G, Gf, rtol=1e-12, atol=1e-12 * np.abs(Gf).max())
        assert np.allclose(M, Mf, rtol=1e-12, atol=1e-12 * np.abs(Mf).max())


@pytest.mark.parametrize("world", [2])
@pytest.mark.parametrize("case", [0, 1])
def test_sharding_decomposition_gloo(oracle, world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def _c4_worker(rank, world, port, q):
    """BASELINE C4 sharding (rtucker_b200_kron_fiber_sketch_shard): every shard takes the
    same draws, keeps the data draws with j2 in its range (rt.shard_rows over I2) and adds
    the augmented diagonal on shard 0 only; the sum over shards is the full Gram and RHS."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.oracle import Oracle
        from paper_2107_10654_b200 import rtucker as rt
        ar = rt.host_allreduce(dist)
        o = Oracle()
        rng = np.random.default_rng(8)
        I1, I2, I3, R2, R3, lam, s = 12, 17, 15, 3, 4, 1e-2, 4000
        X = rng.standard_normal((I1, I2, I3))
        A2, A3 = rng.standard_normal((I2, R2)), rng.standard_normal((I3, R3))
        sc, cdf, sums = [], [], []
        for f in (A2, A3):
            a, b, c, _ = o.factor_scores(f)
            sc.append(a)
            cdf.append(b)
            sums.append(c)
        W, total = R2 * R3, I2 * I3
        idx, w, _ = o.kron_draw([I2, I3], W, sc, cdf, sums, 11, s)

        def normal_eq(sel, with_aug):
            d = idx < total
            m = d & sel
            j2, j3 = idx[m] // I3, idx[m] % I3
            Z = np.einsum("tp,tq->tpq", A2[j2], A3[j3]).reshape(-1, W) * (w[m] ** 2)[:, None]
            G = Z.T @ np.einsum("tp,tq->tpq", A2[j2], A3[j3]).reshape(-1, W)
            Rh = Z.T @ X[:, j2, j3].T
            if with_aug:
                for j, wt in zip(idx[~d] - total, w[~d]):
                    G[j, j] += wt * wt * lam
            return np.ascontiguousarray(G), np.ascontiguousarray(Rh)

        lo, hi = rt.shard_rows(rank, world, I2)
        j2all = np.where(idx < total, idx // I3, -1)
        g, r = normal_eq((j2all >= lo) & (j2all < hi), rank == 0)
        ar(g.ctypes.data, g.size, 0)
        ar(r.ctypes.data, r.size, 0)
        gf, rf = normal_eq(np.ones(s, bool), True)
        dg = np.sqrt(np.outer(np.diag(gf), np.diag(gf)))
        assert np.max(np.abs(g - gf) / dg) < 1e-12
        assert np.linalg.norm(r - rf) / np.linalg.norm(rf) < 1e-12
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2])
def test_c4_sharding_decomposition_gloo(oracle, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_c4_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"
