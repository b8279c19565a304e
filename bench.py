#!/usr/bin/env python
"""bench.py -- sketched Tucker-ALS sweeps/s on B200 (BASELINE.json configs[1], "C2").

Workload (one "step" = one ALS sweep over a device-resident tensor):
  X = 512^3 FP64 (1.07 GB, larger than the 126 MB L2), planted rank (16,16,16)
  with N(0,1) core/factors plus dense Gaussian noise at 1% of ||X||/sqrt(N),
  Tucker rank (16,16,16), lambda = 1e-2, 200,000 sketch rows for the core
  update (d = 4096), exact factor updates (the reference's semantics,
  ref tucker.cpp:241-248; the reference has no sketched factor update),
  reference uniform init (ref tucker.cpp:168-190). Synthetic data, seed 0.

Arms:
  default            our librtucker_b200.so (hand-written sm_100a kernels)
  --impl reference   the reference's own CPU code (oracle/_ref, compiled from
                     /root/reference/proj sources), single-threaded, timed on
                     bounded samples of each sweep phase and extrapolated.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPE = (512, 512, 512)
RANKS = (16, 16, 16)
LAM = 1e-2
S_CORE = 200_000
S_FACTOR = 20_000  # BASELINE configs[1]: samples per factor update (perf mode line)
NOISE = 0.01
E2E_SWEEPS = 10  # the C2 protocol
METRIC = "sketched Tucker-ALS sweeps/s"
WORKLOAD = ("C2: dense 3-way FP64 512^3 (1.07 GB), planted rank (16,16,16) N(0,1) + 1% "
            "noise; Tucker rank (16,16,16), lambda=1e-2, 200,000 sampled rows for the core "
            "update (d=4096); exact factor updates (reference semantics)")


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ---------------------------------------------------------------------------
# reference CPU arm (oracle/_ref = the reference compiled from its sources)

SVD_GROWTH = 11.3  # the reference's Jacobi SVD, d = 512 -> 1024, measured
SVD_ANCHOR_R = 7   # the reference's own update_core_fast timed at d = 7^3 = 343


def reference_sweep_estimate(ref, np, x_full, core, factors, slab=64, gram_samples=100,
                             seed=12345):
    """One bounded sample of every phase of a C2 sweep, timed with the reference's own
    routines (oracle/_ref), extrapolated to C2 (labelled "extrapolated": a C2 sweep takes
    hours on the reference). Returns (seconds per sweep, detail dict)."""
    # update_factor(mode) and the loss are linear in prod(I_n) when the tensor is
    # cut along a mode other than the updated one (the Kronecker of the other
    # factors shrinks with the slab); mode 1 is timed on a mode-3 slab, modes 2
    # and 3 and the loss on a mode-1 slab.
    t_factor = 0.0
    t_loss = 0.0
    xa = x_full[:slab]
    fa = [factors[0][:slab], factors[1], factors[2]]
    xc = np.ascontiguousarray(x_full[:, :, :slab])
    fc = [factors[0], factors[1], factors[2][:slab]]
    for mode in (1, 2, 3):
        if mode == 1:
            shp, xs, fs = (SHAPE[0], SHAPE[1], slab), xc, fc
        else:
            shp, xs, fs = (slab, SHAPE[1], SHAPE[2]), xa, fa
        out = ref.time_sweep_phases(shp, RANKS, core, fs, LAM, xs, 16, seed, mode,
                                    gram_samples=0, svd_dim=0, do_factor=True,
                                    do_loss=(mode == 2))
        t_factor += out[0]
        t_loss += out[1]
    scale = SHAPE[0] / slab
    # the Gram/RHS stream at C2 (d = 4096, the 67 MB upper triangle streamed per data row):
    # the loop of sketch_ridge.cpp:105-128 over the reference's KroneckerRowSource on 100
    # real C2 data rows (ref_time_sweep_phases)
    out = ref.time_sweep_phases(SHAPE, RANKS, core, factors, LAM, x_full, S_CORE, seed, 1,
                                gram_samples=gram_samples, svd_dim=0, do_factor=False,
                                do_loss=False)
    t_gram_sample, t_setup, n_data = out[2], out[3], out[5]
    # the solve: the reference's own update_core_fast (setup + draws + Gram stream + Jacobi
    # compact_svd + pinv apply) on the C2 tensor at core rank 7 (d = 343), s = 2,000 (its
    # Gram stream is ~1% of it), then the SVD grown to d = 4096 by the reference's measured
    # growth per doubling of d (x11.3)
    ra = (SVD_ANCHOR_R,) * 3
    core_a, fac_a = ref.random_model(SHAPE, ra, 0)
    ta = ref.time_core_fast(SHAPE, ra, core_a, fac_a, LAM, x_full, 2000, seed)
    d_a = SVD_ANCHOR_R ** 3
    d = int(np.prod(RANKS))
    t_svd_full = ta[4] * SVD_GROWTH ** np.log2(d / d_a)
    total = scale * (t_factor + t_loss) + t_setup + n_data * t_gram_sample + t_svd_full
    detail = {"factor_updates_s": scale * t_factor, "loss_s": scale * t_loss,
              "kron_setup_s": t_setup, "gram_stream_s": n_data * t_gram_sample,
              "gram_s_per_data_row": t_gram_sample, "data_rows": int(n_data),
              "svd_solve_s_extrapolated": t_svd_full,
              "anchor_update_core_fast": {"d": d_a, "s": 2000, "total_s": ta[0],
                                          "solve_s": ta[4], "setup_s": ta[1]},
              "svd_growth_per_doubling": SVD_GROWTH}
    return total, detail


def reference_inputs(np):
    from oracle.oracle import Reference
    ref = Reference()
    rng = np.random.default_rng(0)
    x = rng.standard_normal(SHAPE)
    core, factors = ref.random_model(SHAPE, RANKS, 0)
    return ref, x, core, factors


REF_SAMPLE = ("EXTRAPOLATED C2 sweep from bounded samples of the reference's own routines: "
              "update_factor (3 modes) and tucker_loss on 64-wide slabs cut along a mode other "
              "than the updated one (x8, linear in prod I_n); the Gram/RHS stream of "
              "sketch_ridge.cpp:105-128 on 100 real C2 data rows at d=4096 (x s_data); "
              "ImplicitKronecker setup at C2; the reference's update_core_fast at d=343 (its "
              "Jacobi SVD solve) grown to d=4096 by the measured x11.3 per doubling of d")


# ---------------------------------------------------------------------------
# C1 head to head (BASELINE configs[0]): the same C-API job through either library

C1_SHAPE, C1_RANKS, C1_LAM, C1_S, C1_SWEEPS = (100, 100, 100), (5, 5, 5), 1e-3, 20000, 10
C1_WORKLOAD = ("C1: dense 3-way FP64 100^3, planted rank (5,5,5) N(0,1) core/factors + 1% "
               "Gaussian noise (seed 0); Tucker rank (5,5,5), lambda=1e-3, 20,000 sampled rows "
               "for the core update, exact factor updates, 10 sweeps, the reference's uniform init")


def c1_input(np):
    rng = np.random.default_rng(0)
    core = rng.standard_normal(C1_RANKS)
    x = core
    for n, (i, r) in enumerate(zip(C1_SHAPE, C1_RANKS)):
        x = np.moveaxis(np.tensordot(rng.standard_normal((i, r)), x, axes=(1, n)), 0, n)
    x = x + NOISE * np.linalg.norm(x) / np.sqrt(x.size) * rng.standard_normal(x.shape)
    return np.ascontiguousarray(x)


def capi_als_job(lib, opts, x, ranks):
    """One C1 job through the reference's C API (include/rtucker.h, identical in both
    libraries): rtucker_tensor_create(host X) + rtucker_als_run + rtucker_result_model.
    Returns (wall seconds, final loss)."""
    import ctypes as C
    import numpy as np
    shape = np.ascontiguousarray(x.shape, dtype=np.uint64)
    rk = np.ascontiguousarray(ranks, dtype=np.uint64)
    u64p = C.POINTER(C.c_uint64)
    f64p = C.POINTER(C.c_double)
    t, r, m = C.c_void_p(), C.c_void_p(), C.c_void_p()
    lib.rtucker_result_final_loss.restype = C.c_double
    t0 = time.perf_counter()
    rc = lib.rtucker_tensor_create(shape.ctypes.data_as(u64p), len(shape),
                                   x.ctypes.data_as(f64p), C.byref(t))
    rc = rc or lib.rtucker_als_run(t, rk.ctypes.data_as(u64p), len(rk), C.byref(opts), C.byref(r))
    rc = rc or lib.rtucker_result_model(r, C.byref(m))
    loss = lib.rtucker_result_final_loss(r) if not rc else float("nan")
    t1 = time.perf_counter()
    if m:
        lib.rtucker_model_free(m)
    if r:
        lib.rtucker_result_free(r)
    if t:
        lib.rtucker_tensor_free(t)
    if rc:
        raise RuntimeError(f"C1 job failed: status {rc}")
    return t1 - t0, loss


def c1_head_to_head(lib, opts, jobs):
    import numpy as np
    x = c1_input(np)
    capi_als_job(lib, opts, x, C1_RANKS)  # warm-up job
    secs, loss = [], None
    for _ in range(jobs):
        t, loss = capi_als_job(lib, opts, x, C1_RANKS)
        secs.append(t)
    med = statistics.median(secs)
    return {"workload": C1_WORKLOAD, "sweeps_per_s": C1_SWEEPS / med, "seconds_per_job": med,
            "jobs": jobs, "final_loss": loss, "measured": True,
            "step": "one job = rtucker_tensor_create(host X) + rtucker_als_run(10 sweeps) + "
                    "rtucker_result_model, wall clock, median over jobs"}


def run_reference_arm(args):
    import numpy as np
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    ref, x, core, factors = reference_inputs(np)
    # C1 head to head: the same C-API job our arm runs, on the reference's own library
    from oracle.oracle import AlsOptions as RefOpts
    c1 = c1_head_to_head(ref.lib, RefOpts(C1_LAM, 1, 0.1, 0.1, 0, C1_SWEEPS, 0.0, C1_S, 0), 3)
    c1["library"] = "oracle/_ref/librtucker_ref.so (the reference compiled from its sources)"
    # each estimate is a bounded sample of one C2 sweep (~8 s of CPU); the run is capped at
    # one warm-up and 8 timed estimates so that --steps K --warmup W ends within minutes
    n_warm, n_timed = min(args.warmup, 1), max(1, min(args.steps, 8))
    vals = []
    for i in range(n_warm + n_timed):
        t, detail = reference_sweep_estimate(ref, np, x, core, factors)
        if i >= n_warm:
            vals.append(t)
    sec = statistics.mean(vals)
    value = 1.0 / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sweeps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": REF_SAMPLE,
                   "timed_estimates": n_timed, "warmup_estimates": n_warm},
        "extrapolated": True,
        "cpu_baseline": {"value": value, "unit": "sweeps/s", "cores": 1, "kind": "reference",
                         "sample": REF_SAMPLE, "phases": detail, "extrapolated": True,
                         "host_cores": os.cpu_count()},
        "c1_head_to_head": c1,
        "e2e": {"value": value, "unit": "sweeps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class Clocks:
    """nvidia-smi sampler (100 ms period) on a reader thread that timestamps every line;
    only samples taken inside [mark_start, stop] are reported."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        import threading
        self.p = None
        self.lines = []
        self.t0 = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
            return

        def reader():
            for line in self.p.stdout:
                self.lines.append((time.perf_counter(), line))
        self.th = threading.Thread(target=reader, daemon=True)
        self.th.start()

    def wait_first(self, timeout=10.0):
        t = time.perf_counter()
        while self.p is not None and not self.lines and time.perf_counter() - t < timeout:
            time.sleep(0.01)

    def mark_start(self):
        self.t0 = time.perf_counter()

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.perf_counter()
        time.sleep(0.15)  # let the sample straddling the end arrive
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            pass
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0 = self.t0 if self.t0 is not None else 0.0
        for ts, line in list(self.lines):
            if ts < t0 or ts > t1 + 0.1:
                continue
            f = [v.strip() for v in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for name, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm

def make_input(torch, device, seed=0):
    g = torch.Generator(device=device).manual_seed(seed)
    core = torch.randn(RANKS, dtype=torch.float64, device=device, generator=g)
    x = core
    for n, I in enumerate(SHAPE):
        f = torch.randn(I, RANKS[n], dtype=torch.float64, device=device, generator=g)
        x = torch.movedim(torch.tensordot(f, x, dims=([1], [n])), 0, n)
    sigma = NOISE * x.norm() / x.numel() ** 0.5
    x = x + sigma * torch.randn(x.shape, dtype=torch.float64, device=device, generator=g)
    return x.contiguous()


def family_table(fam, steps, n_data, n_buckets, pcg_iters, peaks, hbm_peak):
    """Per-sweep time and roofline fraction of every major kernel family (DESIGN.md s.3).
    Work is algorithmic: flops of the DMMA contractions, bytes of the X passes."""
    total = SHAPE[0] * SHAPE[1] * SHAPE[2]
    R3 = RANKS[2]
    v = [r * (r + 1) // 2 for r in RANKS]
    dmma = peaks["dmma_m8n8k4_tflops"]
    rows = {}
    def add(name, sec, flops=None, hbm_bytes=None, note=None):
        row = {"ms_per_sweep": sec * 1e3}
        if flops:
            row["tflops"] = flops / sec / 1e12
            row["frac_dmma"] = row["tflops"] / dmma
        if hbm_bytes:
            row["gbs"] = hbm_bytes / sec / 1e9
            row["frac_hbm"] = row["gbs"] / hbm_peak
        if note:
            row["note"] = note
        rows[name] = row
    per = {k: v_[0] / steps for k, v_ in fam.items()}
    if "gram" in per:
        add("gram", per["gram"], flops=2.0 * (n_data * v[1] * v[2] + n_buckets * v[0] * v[1] * v[2]),
            note="vech Gram: draw records + tables, H_b GEMMs (k_vech_bucket5), contraction over "
                 "buckets (k_vech_contract3)")
    if "gram_sort" in per:
        add("gram_sort", per["gram_sort"],
            note="bucket keys from A_1's CDF, stable key sort, bucket table and order; a side "
                 "branch after F1 in the timed (graph) sweeps, off the critical path")
    if "ttm_last_loss" in per:
        add("ttm_last_loss", per["ttm_last_loss"], flops=4.0 * total * R3, hbm_bytes=8.0 * total,
            note="one X pass: T = X A_3 and the direct residual (X - P A_3^T)^2")
    if "ttm_mid" in per:
        add("ttm_mid", per["ttm_mid"], flops=2.0 * total * RANKS[0], hbm_bytes=8.0 * total,
            note="X x_1 A_1^T (F3 projection) + three 32 MB T-based products")
    if "pcg" in per:
        d = RANKS[0] * RANKS[1] * RANKS[2]
        add("pcg", per["pcg"], note=f"{pcg_iters} CG iterations on the compact Gram "
            f"({v[0] * v[1] * v[2] * 8 / 1e6:.0f} MB, slices resident in shared memory, "
            f"k_pcg_split), d={d}")
    if "chol" in per:
        d = RANKS[0] * RANKS[1] * RANKS[2]
        add("chol", per["chol"], flops=d ** 3 / 3 + 2 * d * d)
    return rows


PCG_ITERS = [0]


def kernel_work(family, n_data, n_buckets):
    """Algorithmic work per launch of a kernel family."""
    d = 1
    for r in RANKS:
        d *= r
    total = SHAPE[0] * SHAPE[1] * SHAPE[2]
    if family == "chol":
        return "tensor", "TFLOP/s", d ** 3 / 3 + 2 * d * d
    if family == "pcg":
        # per solve: every CG iteration (+1 residual check) reads the compact Gram once
        # (shared-memory resident in k_pcg_split, counted against the HBM roofline)
        v = [r * (r + 1) // 2 for r in RANKS]
        blk = v[0] * v[1] * v[2] * 8
        return "hbm", "GB/s", (PCG_ITERS[0] + 1) * blk
    if family == "gram":
        # vech-factored Gram: per data draw one rank-1 update of
        # the i1-bucket's H_b (vech(R2) x vech(R3)), then S = V1^T H over buckets.
        v = [r * (r + 1) // 2 for r in RANKS]
        return "tensor", "TFLOP/s", 2.0 * (n_data * v[1] * v[2] + n_buckets * v[0] * v[1] * v[2])
    if family == "ttm_last_loss":
        # one launch per sweep: T = X A_3 plus the direct residual, 4 * total * R3 flops
        return "tensor", "TFLOP/s", 4.0 * total * RANKS[2]
    if family in ("ttm_last", "ttm_mid"):
        return "hbm", "GB/s", 8.0 * total
    return None, None, None


def run_our_arm(args):
    import numpy as np
    import torch
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif args.nccl_p1:
        # diagnostic: the sharded code path (kernel-by-kernel sweeps, partial sums through the
        # NCCL all-reduce callback) with ONE shard on one GPU -- the collective plumbing run for
        # real, and its cost before any scaling
        import socket
        import torch.distributed as dist
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                world_size=1, device_id=torch.device("cuda", local))
    from paper_2107_10654_b200 import rtucker as rt
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    rt.set_stream(stream.cuda_stream)

    # N > 1: one C2 job split across the GPUs along mode 1 (strong scaling); every
    # rank builds the same seeded X and keeps its rows; partial sums meet in NCCL
    # all-reduces issued by the library through the Shard callback.
    x = make_input(torch, dev)
    shard = None
    lshape = SHAPE
    if world > 1:
        lo, hi = rt.shard_rows(rank, world, SHAPE[0])
        x = x[lo:hi].contiguous()
        lshape = (hi - lo,) + tuple(SHAPE[1:])
        shard = rt.Shard(rank, world, SHAPE[0], rt.torch_allreduce(dist))
    elif args.nccl_p1:
        shard = rt.Shard(0, 1, SHAPE[0], rt.torch_allreduce(dist))
    torch.cuda.synchronize()
    t = rt.Tensor.from_device(x.data_ptr(), lshape)
    torch.cuda.synchronize()
    xh = torch.empty(lshape, dtype=torch.float64, pin_memory=True)
    xh.copy_(x)
    del x
    torch.cuda.empty_cache()

    opts = rt.options(lam=LAM, sketched_core=1, sample_count_override=S_CORE, tolerance=0.0,
                      max_iterations=args.warmup + args.steps, seed=0)
    # headline: K sweeps of one session, kernel by kernel for the first sweep and one CUDA
    # graph launch per sweep after that (no host round trip inside a sweep)
    sess = rt.Session(t, RANKS, opts, shard=shard)
    sess.sweeps(args.warmup)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.wait_first()
    launches0 = rt.lib.rtucker_b200_launch_count()
    clocks.mark_start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sess.sweeps(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    launches = rt.lib.rtucker_b200_launch_count() - launches0
    ms = e0.elapsed_time(e1)
    if dist:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    res = sess.result()
    info = res.sketch_info()
    graph_sweeps = res.graph_sweeps
    hist = res.history()
    sess.free()

    # per-kernel-family device times for the roofline: the same workload re-run kernel by
    # kernel with CUDA events around every family on the library's stream (the headline
    # region runs as graph launches, where no per-kernel events are recorded)
    prof_steps = min(args.steps, 50)
    sp = rt.Session(t, RANKS, rt.options(lam=LAM, sketched_core=1, sample_count_override=S_CORE,
                                         tolerance=0.0, max_iterations=args.warmup + prof_steps,
                                         seed=0), profile=True, shard=shard)
    sp.sweeps(args.warmup)
    torch.cuda.synchronize()
    k0 = {k[0]: k for k in sp.result().kernels()}
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    sp.sweeps(prof_steps)
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1) / prof_steps
    fam = {}
    for name, secs, n in sp.result().kernels():
        p = k0.get(name, (name, 0.0, 0))
        fam[name] = (secs - p[1], n - p[2])
    sp.free()

    # BASELINE configs[1] as written also samples the factor updates (20,000 draws per mode,
    # design width 256): the library's perf mode (ext.factor_samples; the reference has no
    # such update, so the headline keeps its exact factor updates). Timed the same way.
    fsk = None
    if world == 1 and not args.c2_only:
        fs_steps = min(args.steps, 50)
        opts_f = rt.options(lam=LAM, sketched_core=1, sample_count_override=S_CORE,
                            tolerance=0.0, max_iterations=args.warmup + fs_steps, seed=0)
        sf = rt.Session(t, RANKS, opts_f, factor_samples=S_FACTOR)
        sf.sweeps(args.warmup)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        sf.sweeps(fs_steps)
        f1.record(stream)
        torch.cuda.synchronize()
        fh = sf.result().history()
        sf.free()
        fsk = {"sweeps_per_s": fs_steps / (f0.elapsed_time(f1) / 1e3), "steps": fs_steps,
               "factor_samples": S_FACTOR, "final_loss": fh[-1][2] if fh else None,
               "note": "perf mode (sketched factor updates, BASELINE configs[1] literally); "
                       "not the reference's semantics. At C2 it stays slower than the exact "
                       "updates: those reuse T = X x3 A3 from the loss pass, while every sketched "
                       "mode pays a latency-bound scores + draw-decode chain (~0.1 ms); the fiber "
                       "gathers read mode-n-last copies of X (contiguous, 1.05x useful bytes)"}

    # roofline of the dominant kernel: the largest single kernel of the step, which in
    # the ncu launch list of this command (profiles/r01_launches_bench_v6.txt) is
    # k_ttm_last5, the whole of the ttm_last_loss family. The library's other families
    # group several kernels (gram: 8 launches, largest k_vech_bucket2; pcg: 5, largest
    # k_pcg); their own rooflines are in "families".
    dom = "ttm_last_loss" if "ttm_last_loss" in fam else max(fam, key=lambda k: fam[k][0])
    PCG_ITERS[0] = info.get("pcg_iterations", 0) or 0
    n_data = info["data_draws"]
    n_buckets = SHAPE[0]
    bound, unit, work = kernel_work(dom, n_data, n_buckets)
    peaks = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
    mp = {}
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    roofline = None
    if bound:
        secs, n = fam[dom]
        per_launch = secs / max(n, 1)
        if bound == "tensor":
            achieved = work / per_launch / 1e12
            peak = peaks["dmma_m8n8k4_tflops"]
            peak_src = "measured FP64 DMMA.8x8x4 microbench (profiles/fp64_peak.json)"
        else:
            achieved = work / per_launch / 1e9
            peak = mp.get("hbm_gbs", 6553.3)
            peak_src = "MEASURED_PEAKS.json hbm_gbs"
        traffic = None
        tf = os.path.join(ROOT, "profiles", "r02_traffic.json")
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get(dom)
        roofline = {"kernel": dom + (" (k_ttm_last5)" if dom == "ttm_last_loss" else " (family)"),
                    "bound": bound, "achieved": achieved, "peak": peak,
                    "unit": unit, "frac": achieved / peak, "traffic": traffic,
                    "peak_source": peak_src, "work_per_launch": work,
                    "launch_ms": per_launch * 1e3, "launches": n}

    # e2e through the public C API with host buffers (rank 0 timing, max over ranks)
    e2e_vals = []
    xnp = xh.numpy()
    h2d_bytes = int(xnp.nbytes)
    rt.set_stream(stream.cuda_stream)
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = rt.Tensor.from_numpy(xnp)  # host -> library (rtucker_tensor_create)
        r = rt.als_run(th, RANKS, rt.options(lam=LAM, sketched_core=1,
                                             sample_count_override=S_CORE, tolerance=0.0,
                                             max_iterations=E2E_SWEEPS, seed=0), shard=shard)
        m = r.model()  # device -> host result
        fl = r.final_loss
        t1 = time.perf_counter()
        r.free()
        th.free()
        if i > 0:
            e2e_vals.append(t1 - t0)
    e2e_s = statistics.mean(e2e_vals)
    if dist:
        tt = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    d2h = (m.core.size + sum(f.size for f in m.factors)) * 8 + 8

    # C1 head to head (BASELINE configs[0]): the same C-API job as the reference arm's, on
    # (before the CPU baseline: its host-side numpy work leaves BLAS threads spinning, which
    # slowed these wall-clocked millisecond jobs)
    # this library; plus the device-only C1 sweep rate (resident X, graph launches)
    c1 = None
    if rank == 0 and world == 1 and not args.c2_only:
        c1 = c1_head_to_head(rt.lib, rt.options(lam=C1_LAM, sketched_core=1, tolerance=0.0,
                                                sample_count_override=C1_S,
                                                max_iterations=C1_SWEEPS, seed=0), 20)
        c1["library"] = "paper_2107_10654_b200/lib/librtucker_b200.so"
        xc = rt.Tensor.from_numpy(c1_input(np))
        n1 = 200
        sc = rt.Session(xc, C1_RANKS, rt.options(lam=C1_LAM, sketched_core=1, tolerance=0.0,
                                                 sample_count_override=C1_S,
                                                 max_iterations=args.warmup + n1, seed=0))
        sc.sweeps(args.warmup)
        torch.cuda.synchronize()
        c0e, c1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0e.record(stream)
        sc.sweeps(n1)
        c1e.record(stream)
        torch.cuda.synchronize()
        c1["device_sweeps_per_s"] = n1 / (c0e.elapsed_time(c1e) / 1e3)
        c1["device_ms_per_sweep"] = c0e.elapsed_time(c1e) / n1
        c1["device_cuda_graph_sweeps"] = sc.result().graph_sweeps
        sc.free()
        xc.free()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ref, xr, core, factors = reference_inputs(np)
            sec, detail = reference_sweep_estimate(ref, np, xr, core, factors)
            cpu = {"value": 1.0 / sec, "unit": "sweeps/s", "cores": 1, "kind": "reference",
                   "sample": REF_SAMPLE, "host_cores": os.cpu_count(), "phases": detail}
        except Exception as e:  # oracle/_ref missing on this box
            cpu = {"value": None, "unit": "sweeps/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    # BASELINE configs 3 and 4, measured in the same run (their own clocks samples)
    extra = {}
    if rank == 0 and world == 1 and not args.no_extra:
        t.free()
        del xh, xnp
        torch.cuda.empty_cache()
        extra["c3"] = c3_lines(args, steps=min(args.steps, 20))
        extra["c4"] = c4_lines(args, steps=min(args.steps, 5), s_list=[100000, 1000000, 10000000])
        extra["c5"] = c5_lines(args, steps=min(args.steps, 5))

    if rank == 0:
        sweeps_per_s = args.steps / (ms / 1e3)  # one job across all GPUs
        line = {
            "metric": METRIC, "value": sweeps_per_s, "unit": "sweeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": ("strong" if world > 1 else "weak"),
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded torch N(0,1) planted model + 1% noise)",
            "config": {"workload": WORKLOAD, "shape": list(SHAPE), "ranks": list(RANKS),
                       "lambda": LAM, "s_core": S_CORE, "factor_updates": "exact",
                       "l2": "inputs larger than L2 (X = 1.07 GB > 126 MB)",
                       "step": "one ALS sweep (3 factor updates + sketched core + loss)",
                       "parallelism": (f"X sharded along mode 1 over {world} GPUs, NCCL all-reduce"
                                       " of partial sums" if world > 1 else
                                       "single GPU, sharded code path with one shard (one-rank NCCL "
                                       "all-reduce behind every partial sum)" if args.nccl_p1
                                       else "single GPU"),
                       "final_loss": hist[-1][2] if hist else None},
            "clocks": clk,
            "e2e": {"value": E2E_SWEEPS / e2e_s, "unit": "sweeps/s",
                    "h2d_bytes_per_step": h2d_bytes * world, "d2h_bytes_per_step": int(d2h),
                    "step": "one job: rtucker_tensor_create(host X) + rtucker_als_run(10 sweeps)"
                            " + rtucker_result_model", "seconds_per_job": e2e_s},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "kernels_ms_per_sweep": {k: v[0] * 1e3 / prof_steps for k, v in fam.items()},
            "families": family_table(fam, prof_steps, n_data, n_buckets,
                                     info.get("pcg_iterations"), peaks, mp.get("hbm_gbs", 6553.3)),
            "profiled_region": {"sweeps": prof_steps, "ms_per_step": prof_ms,
                                "note": "kernel-by-kernel re-run with CUDA events around every "
                                        "kernel family; source of kernels_ms_per_sweep, "
                                        "families and roofline"},
            "cuda_graph_sweeps": graph_sweeps,
            "sketch": info,
            "sketched_factor_updates": fsk,
            "cpu_baseline": cpu,
            "c1_head_to_head": c1,
            "other_configs": extra or None,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def c4_lines(args, steps=None, s_list=None):
    """BASELINE config 4 microbench (--workload c4): Kronecker-product sampling + fused fiber
    gather/SYRK. 3 factors 2048 x 32 N(0,1) FP64 (A1 unused by the microbench), X 2048^3 FP32
    N(0,1) (34 GB, resident, replicated per GPU), lambda = 1e-2; for each s: draws of
    [A2 (x) A3; sqrt(lambda) I] (W = 1024), the W x W Gram and the W x 2048 mode-1 fiber RHS.
    N > 1 (torchrun): shard r accumulates the draws of its j2 range and an NCCL all-reduce sums
    the Gram and RHS inside the timed step (device time, max over ranks). One JSON line per s."""
    import numpy as np
    import torch
    from paper_2107_10654_b200 import rtucker as rt
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rt.set_stream(torch.cuda.current_stream().cuda_stream)
    I, R, lam = 2048, 32, 1e-2
    g = torch.Generator(device="cuda").manual_seed(0)
    a2 = torch.randn(I, R, dtype=torch.float64, device="cuda", generator=g)
    a3 = torch.randn(I, R, dtype=torch.float64, device="cuda", generator=g)
    x = torch.empty((I, I, I), dtype=torch.float32, device="cuda")
    for k in range(0, I, 128):  # seeded N(0,1) in slabs (bounded temporaries)
        x[k:k + 128].normal_(generator=g)
    W = R * R
    gram = torch.empty(W, W, dtype=torch.float64, device="cuda")
    rhs = torch.empty(W, I, dtype=torch.float64, device="cuda")
    # fiber-major copy (mode 1 fastest, every mode-1 fiber one contiguous 8 KB run): a one-time
    # layout conversion of the resident tensor, timed and reported, not part of a step
    xf = torch.empty_like(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rt.tensor_fiber_major(x.data_ptr(), (I, I, I), xf.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    fm_ms = e0.elapsed_time(e1)
    peaks = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
    mp = {}
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = mp.get("hbm_gbs", 6553.3)
    fp64 = peaks["dmma_m8n8k4_tflops"]

    def step(xp, fm, s, seed):
        out = rt.kron_fiber_sketch(xp, (I, I, I), a2.data_ptr(), a3.data_ptr(), R, R, lam, s, seed,
                                   gram.data_ptr(), rhs.data_ptr(), fiber_major=fm,
                                   shard=(rank, world))
        if dist is not None:
            dist.all_reduce(gram)
            dist.all_reduce(rhs)
        return out

    steps = steps or args.steps
    clk_all = {}

    def run(xp, fm, s):
        for _ in range(args.warmup):
            step(xp, fm, s, 1)
        ph, nd, nu = np.zeros(3), 0, 0
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = Clocks(local)
        clocks.wait_first()
        clocks.mark_start()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for k in range(steps):
            out = step(xp, fm, s, 2 + k)
            ph += np.array(out["phase_ms"])
            nd += out["data_draws"]
            nu += out["unique_rows"]
        t1.record()
        torch.cuda.synchronize()
        clk_all[(s, fm)] = clocks.stop()
        ms = t0.elapsed_time(t1) / steps
        if dist is not None:
            tt = torch.tensor([ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms, ph / steps, nd / steps, nu / steps

    lines = []
    for s in s_list or [int(float(v)) for v in args.c4_s.split(",")]:
        step_ms, (draw_ms, gram_ms, rhs_ms), nd, nu = run(xf.data_ptr(), True, s)
        c_ms, (_, _, rhs_c_ms), _, _ = run(x.data_ptr(), False, s) if world == 1 else (0, (0, 0, 0), 0, 0)
        # Gram: two DMMA GEMMs over vech Khatri-Rao row products (T = C KA3, G' = KA2^T T,
        # m = R (R + 1) / 2 pair columns); the phase also holds the shared sort / merge
        m = R * (R + 1) // 2
        gram_flops = (2.0 * I * I * m + 2.0 * m * m * I) / world
        # RHS: per distinct sampled row 2 R I1 (D_b accumulation), per bucket the a2 (x) D_b fold
        rhs_flops = (2.0 * nu * R * I + 2.0 * I * R * R * I) / world
        fiber_bytes = 4.0 * I * nu / world        # each distinct FP32 fiber read once
        line = {
            "metric": "C4 sketched Kronecker samples/s (Gram+RHS)",
            "value": s / (step_ms / 1e3),
            "unit": "samples/s", "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "dtype": "f64 (FP32 tensor upcast)", "data": "synthetic",
            "config": {"workload": "C4: factors 2048 x 32 N(0,1), X 2048^3 FP32 N(0,1) (34 GB), "
                                   "design A2 (x) A3 (4,194,304 x 1024), lambda 1e-2",
                       "s": s, "data_draws": nd, "distinct_rows": nu,
                       "x_layout": "fiber-major (mode 1 fastest), converted once on device",
                       "fiber_major_convert_ms": fm_ms,
                       "parallelism": f"j2-bucket shards x {world}, NCCL all-reduce of Gram + RHS"
                       if world > 1 else "single GPU"},
            "phases_ms": {"scores_and_draws": draw_ms, "sort_merge_and_gram": gram_ms,
                          "fiber_rhs": rhs_ms},
            "gram_only_samples_per_s": s / ((draw_ms + gram_ms) / 1e3),
            "fiber_rhs": {"useful_gbs": fiber_bytes / (rhs_ms / 1e3) / 1e9,
                          "useful_frac_hbm": fiber_bytes / (rhs_ms / 1e3) / 1e9 / hbm,
                          "tflops": rhs_flops / (rhs_ms / 1e3) / 1e12,
                          "frac_fp64": rhs_flops / (rhs_ms / 1e3) / 1e12 / fp64},
            "gram": {"tflops": gram_flops / (gram_ms / 1e3) / 1e12,
                     "frac_fp64": gram_flops / (gram_ms / 1e3) / 1e12 / fp64},
        }
        if world == 1:
            line["canonical_layout"] = {"fiber_rhs_ms": rhs_c_ms, "samples_per_s": s / (c_ms / 1e3)}
        line["clocks"] = clk_all.get((s, True))
        if rank == 0:
            lines.append(line)
    del x, xf
    torch.cuda.empty_cache()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return lines


def run_c4(args):
    for line in c4_lines(args):
        print(json.dumps(line), flush=True)
    return 0


def c3_lines(args, steps=None):
    """BASELINE config 3 (--workload c3): dense 4-way FP64 160^4 (5.2 GB), planted rank
    (10,10,10,10) with coherent factors (rows scaled by i.i.d. Pareto(1.5) weights), 5% noise,
    lambda = 0.1, s_core = 500,000; one line with exact factor updates (reference semantics)
    and one with sketched factor updates (50,000 samples, perf mode). Seeded synthetic data on
    the device; K sweeps timed with CUDA events after the warm-up sweeps."""
    import torch
    from paper_2107_10654_b200 import rtucker as rt
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:  # N > 1: X split along mode 1, NCCL all-reduce of every partial sum
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rt.set_stream(torch.cuda.current_stream().cuda_stream)
    I, R, lam, s = 160, 10, 0.1, 500000
    shape, ranks = (I,) * 4, (R,) * 4
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(ranks, dtype=torch.float64, device="cuda", generator=g)
    for n in range(4):
        f = torch.randn(I, R, dtype=torch.float64, device="cuda", generator=g)
        u = torch.rand(I, 1, dtype=torch.float64, device="cuda", generator=g)
        f = f * (1.0 - u) ** (-1.0 / 1.5)  # Pareto(alpha = 1.5) row weights
        x = torch.movedim(torch.tensordot(f, x, dims=([1], [n])), 0, n)
    x = x + 0.05 * x.norm() / x.numel() ** 0.5 * torch.randn(x.shape, dtype=torch.float64,
                                                               device="cuda", generator=g)
    shard, lshape = None, shape
    if world > 1:
        lo, hi = rt.shard_rows(rank, world, I)
        x = x[lo:hi]
        lshape = (hi - lo,) + shape[1:]
        shard = rt.Shard(rank, world, I, rt.torch_allreduce(dist))
    x = x.contiguous()
    torch.cuda.synchronize()
    t = rt.Tensor.from_device(x.data_ptr(), lshape)
    del x
    steps = steps or args.steps
    lines = []
    # exact (reference semantics) and sketched (perf mode) factor updates, sharded alike
    for fs in (0, 50000):
        opts = rt.options(lam=lam, sketched_core=1, sample_count_override=s, tolerance=0.0,
                          max_iterations=args.warmup + steps + 1)
        sess = rt.Session(t, ranks, opts, factor_samples=fs, shard=shard)
        sess.sweeps(args.warmup)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        clocks = Clocks(local)
        clocks.wait_first()
        clocks.mark_start()
        e0.record()
        sess.sweeps(steps)
        e1.record()
        torch.cuda.synchronize()
        clk = clocks.stop()
        ms = e0.elapsed_time(e1) / steps
        if dist:
            tt = torch.tensor([ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        r = sess.result()
        graph_sweeps = r.graph_sweeps
        sess.free()
        # kernel shares from a kernel-by-kernel re-run with per-family CUDA events
        sp = rt.Session(t, ranks, rt.options(lam=lam, sketched_core=1, sample_count_override=s,
                                             tolerance=0.0, max_iterations=args.warmup + 5),
                        profile=True, factor_samples=fs, shard=shard)
        sp.sweeps(args.warmup + 5)
        fam = {}
        for name, secs, n in sp.result().kernels():
            fam[name] = fam.get(name, 0.0) + secs
        sp.free()
        tot = sum(fam.values()) or 1.0
        line = {
            "metric": "sketched Tucker-ALS sweeps/s (C3)", "value": 1e3 / ms, "unit": "sweeps/s",
            "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
            "scaling": "strong" if world > 1 else "weak",
            "clocks": clk, "cuda_graph_sweeps": graph_sweeps,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic (seeded torch)",
            "config": {"workload": "C3: dense 4-way FP64 160^4 (5.2 GB), planted rank (10,10,10,10), "
                                   "Pareto(1.5)-scaled factor rows, 5% noise, lambda=0.1, "
                                   "s_core=500,000",
                       "factor_updates": "exact" if fs == 0 else f"sketched ({fs} samples)",
                       "final_loss": r.final_loss},
            "sketch": r.sketch_info(),
            "kernel_share": {k: round(v / tot, 4) for k, v in sorted(fam.items(),
                                                                    key=lambda kv: -kv[1])[:8]},
        }
        line["config"]["parallelism"] = (f"X sharded along mode 1 over {world} GPUs, NCCL "
                                         "all-reduce of partial sums" if world > 1 else "single GPU")
        if rank == 0:
            lines.append(line)
    t.free()
    torch.cuda.empty_cache()
    return lines


def c5_lines(args, steps=None):
    """BASELINE config 5 (--workload c5): 3-way FP64 planted rank (32,32,32), 1% noise,
    lambda = 1e-2, s_core = 1e6, X sharded along mode 1 with 34.4 GB (512 x 4096 x 2048) per
    GPU: at N GPUs the tensor is (512 N) x 4096 x 2048, so N = 8 is BASELINE's 4096 x 4096 x 2048
    (275 GB) and N = 1 is the one-GPU share of it run as a whole ALS problem (weak scaling).
    Generated on the device shard by shard (rtucker_b200_tensor_generate_device); exact factor
    updates (reference semantics) and a sketched-factor line (1e5 samples, perf mode)."""
    import torch
    from paper_2107_10654_b200 import rtucker as rt
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rt.set_stream(torch.cuda.current_stream().cuda_stream)
    I1, lam, s = 512 * world, 1e-2, 1000000
    shape, ranks = (I1, 4096, 2048), (32, 32, 32)
    t = rt.Tensor.generate_device(shape, ranks, 0.01, 0, shard=(rank, world))
    shard = rt.Shard(rank, world, I1, rt.torch_allreduce(dist)) if world > 1 else None
    torch.cuda.synchronize()
    steps = steps or args.steps
    lines = []
    for fs in (0, 100000):
        opts = rt.options(lam=lam, sketched_core=1, sample_count_override=s, tolerance=0.0,
                          max_iterations=args.warmup + steps + 1)
        sess = rt.Session(t, ranks, opts, factor_samples=fs, shard=shard)
        sess.sweeps(args.warmup)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        clocks = Clocks(local)
        clocks.wait_first()
        clocks.mark_start()
        e0.record()
        sess.sweeps(steps)
        e1.record()
        torch.cuda.synchronize()
        clk = clocks.stop()
        ms = e0.elapsed_time(e1) / steps
        if dist:
            tt = torch.tensor([ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        r = sess.result()
        graph_sweeps = r.graph_sweeps
        sess.free()
        sp = rt.Session(t, ranks, rt.options(lam=lam, sketched_core=1, sample_count_override=s,
                                             tolerance=0.0, max_iterations=args.warmup + 3),
                        profile=True, factor_samples=fs, shard=shard)
        sp.sweeps(args.warmup + 2)
        fam = {}
        for name, secs, n in sp.result().kernels():
            fam[name] = fam.get(name, 0.0) + secs
        sp.free()
        tot = sum(fam.values()) or 1.0
        line = {
            "metric": "sketched Tucker-ALS sweeps/s (C5)", "value": 1e3 / ms, "unit": "sweeps/s",
            "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
            "scaling": "weak", "clocks": clk, "cuda_graph_sweeps": graph_sweeps,
            "higher_is_better": True, "dtype": "f64",
            "data": "synthetic (generated on the device from seed 0)",
            "config": {"workload": f"C5 weak-scaling unit: 3-way FP64 {I1}x4096x2048 "
                                   f"({8 * I1 * 4096 * 2048 / 1e9:.1f} GB, 34.4 GB per GPU; "
                                   "N = 8 is BASELINE's 275 GB), planted rank (32,32,32) N(0,1) "
                                   "+ 1% noise, lambda=1e-2, s_core=1,000,000 (d = 32768)",
                       "factor_updates": "exact" if fs == 0 else f"sketched ({fs} samples)",
                       "final_loss": r.final_loss,
                       "parallelism": (f"X sharded along mode 1 over {world} GPUs, NCCL "
                                       "all-reduce of partial sums" if world > 1
                                       else "single GPU")},
            "sketch": r.sketch_info(),
            "kernel_share": {k: round(v / tot, 4) for k, v in sorted(fam.items(),
                                                                    key=lambda kv: -kv[1])[:8]},
        }
        if rank == 0:
            lines.append(line)
    t.free()
    torch.cuda.empty_cache()
    return lines


def run_c5(args):
    for line in c5_lines(args):
        print(json.dumps(line), flush=True)
    if env_int("WORLD_SIZE", 1) > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_c3(args):
    for line in c3_lines(args):
        print(json.dumps(line), flush=True)
    if env_int("WORLD_SIZE", 1) > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the BASELINE config 3 / 4 measurements of the default run")
    ap.add_argument("--c2-only", action="store_true",
                    help="only the C2 headline and its profiled re-run (for ncu launch lists): "
                         "implies --no-extra, skips the C1 head-to-head and the perf-mode line")
    ap.add_argument("--nccl-p1", action="store_true",
                    help="diagnostic (N = 1): run the sharded code path with one shard and a "
                         "one-rank NCCL group behind the all-reduce callback")
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"],
                    help="c2 (default): the headline ALS sweep; c3: the BASELINE config-3 "
                         "4-way Pareto-factor sweep; c4: the BASELINE config-4 sampling + "
                         "fiber gather/SYRK microbench; c5: the BASELINE config-5 rank-32 "
                         "sweep, 34.4 GB of X per GPU (N = 8: the 275 GB tensor)")
    ap.add_argument("--c4-s", default="1e5,1e6,1e7", help="sample counts for --workload c4")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.nccl_p1:
        args.c2_only = args.no_cpu_baseline = True
    if args.c2_only:
        args.no_extra = True
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.workload == "c4":
        return run_c4(args)
    if args.workload == "c3":
        return run_c3(args)
    if args.workload == "c5":
        return run_c5(args)
    return run_our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
