/*
 * rtucker_b200.h -- additive extensions of the B200 build (librtucker_b200.so).
 *
 * Nothing here changes the reference ABI in rtucker.h; these entry points
 * expose what the reference keeps internal (SURVEY.md section 8(b),
 * "Extensions the replacement must add"):
 *   - device-resident tensors (no host copy; for benchmarks and large runs),
 *   - initial-model injection (the reference can only self-initialise,
 *     ref tucker.cpp:168-190),
 *   - oracle/replay entry points for each rung of the parity ladder:
 *     the GPU sampler driven by caller-supplied CDFs (rung 1), the GPU
 *     normal-equation accumulation driven by a caller-supplied RowSketch
 *     (rung 3) and the GPU SPD solve of a caller-supplied Gram (rung 4),
 *   - per-kernel timing export and multi-GPU sample sharding hooks.
 * All pointers are host pointers unless the name says _device.
 */
#ifndef RTUCKER_B200_H
#define RTUCKER_B200_H

#include "rtucker.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Device ordinal used by this thread's calls (default 0). */
rtucker_status rtucker_b200_set_device(int device);
/* CUDA stream (cudaStream_t) for this thread's work; NULL restores the
 * library-owned stream. Lets a caller time the library with its own events. */
rtucker_status rtucker_b200_set_stream(void* stream);
/* Number of this library's kernel launches so far in the process. */
unsigned long long rtucker_b200_launch_count(void);
/* Launches so far of one named kernel variant of the headline path ("k_ttm_mid3",
 * "k_ttm_mid2", "k_ttm_last3", "k_ttm_last3_fused", "k_vech_bucket2<17>", "k_vech_bucket5",
 * "k_vech_contract2", "k_pcg<16,16>"): lets tests assert which kernel ran. */
unsigned long long rtucker_b200_variant_count(const char* name);

/* Wrap a tensor that already lives in device memory of the current device.
 * The data is copied (device to device) before the call returns, so the caller may
 * free or reuse data_device afterwards. There is no host mirror until one is asked
 * for: rtucker_tensor_data() then downloads a host copy (device to host) and
 * returns it (borrowed, valid for the tensor's lifetime). */
rtucker_status rtucker_b200_tensor_create_device(const uint64_t* shape, uint32_t order,
                                                 const double* data_device,
                                                 rtucker_tensor** out);
/* Planted synthetic tensor generated on the GPU (BASELINE configs; a large tensor never
 * exists on the host): core and factors i.i.d. N(0,1), factor rows scaled by i.i.d.
 * Pareto(pareto_alpha) weights when pareto_alpha > 0 (BASELINE config 3), X = the
 * reconstruction plus i.i.d. N(0, sigma^2) noise on every entry with sigma = noise_level *
 * ||X_planted||_F / sqrt(prod I_n). Counter-based SplitMix64 streams (one per role) and
 * Box-Muller, so shard r of P (rows [r I1 / P, (r + 1) I1 / P) of mode 1; shard_count 0 or
 * 1 = the whole tensor) is generated on its own and equals that slab of the unsharded
 * tensor. Not the reference generator's stream (rtucker_tensor_generate is). The result is
 * device-resident (no host mirror until rtucker_tensor_data asks for one). core_out
 * (prod ranks) / factors_out (sum I_n R_n, full A_1) optional, host. */
rtucker_status rtucker_b200_tensor_generate_device(const uint64_t* shape,
                                                   const uint64_t* planted_ranks, uint32_t order,
                                                   double noise_level, double pareto_alpha,
                                                   uint64_t seed, uint32_t shard_rank,
                                                   uint32_t shard_count, rtucker_tensor** out,
                                                   double* core_out, double* factors_out);

/* Device pointer of a tensor's resident copy (borrowed). */
const double* rtucker_b200_tensor_device_data(const rtucker_tensor* t);

/* Extended ALS options. Zero-initialise, then set what you need. */
typedef struct rtucker_b200_als_ext {
  /* If non-NULL: initial core (prod ranks, row-major) and factors (factor n is
   * I_n x R_n row-major, concatenated) replace the uniform init. */
  const double* init_core;
  const double* init_factors;
  /* Multi-GPU (shard_count > 1): X is split along mode 1; this process passes only
   * its rows [r*I1/P, (r+1)*I1/P) (r = shard_rank, P = shard_count, I1 =
   * shard_rows_total) as `x`. X passes, mode-1 factor rows and the sketch's data
   * draws stay local; every partial sum (projections, A_1 rows, compact Gram + rhs,
   * residual) goes through `allreduce` (in place, doubles, enqueued on the
   * library's stream, e.g. ncclAllReduce sum). shard_count 0/1 with a NULL
   * `allreduce` = no sharding; with a callback installed the sharded path runs
   * with one shard (every partial sum still goes through the callback). */
  uint32_t shard_rank;
  uint32_t shard_count;
  void (*allreduce)(double* device_buf, uint64_t count, void* stream, void* user);
  void* allreduce_user;
  /* Skip the per-sweep host sync when tolerance <= 0 (no early stop possible):
   * the whole run is enqueued back to back. Default 1. */
  int async_sweeps_when_no_tolerance;
  /* 1 = record per-kernel-family device time (CUDA events on the run's
   * stream), exported by rtucker_b200_result_kernel_row. */
  int profile_kernels;
  /* Sketched-core solver: 0 = auto (Kronecker-preconditioned CG when lambda > 0,
   * every augmented row was drawn and d fits, verified by its true residual;
   * Cholesky otherwise or on failure), 1 = always Cholesky. */
  int core_solver;
  /* 1 = loss by ||X||^2 - 2<Y,G> + <Q,G> (one cheaper X pass; ~1e-12 ||X||^2
   * absolute accuracy, falls back to the direct residual near an exact fit);
   * 0 (default) = the reference's direct residual pass. */
  int fast_loss;
  int shard_rows_total; /* global I_1 of a sharded run */
  /* Perf mode (not the reference's semantics): > 0 = sketched factor updates with this
   * many draws per mode from the product of the other modes' leverage distributions
   * plus the sqrt(lambda) augmentation (BASELINE "samples per factor update"; DESIGN.md
   * section 3). 0 (default) = the reference's exact factor updates. Not with sharding. */
  uint32_t factor_samples;
  /* 1 = enqueue every sweep kernel by kernel (no CUDA graph; results are identical) */
  int disable_graph;
  int reserved[2];
} rtucker_b200_als_ext;

rtucker_status rtucker_b200_als_run_ex(const rtucker_tensor* x, const uint64_t* ranks,
                                       uint32_t order, const rtucker_als_options* opts,
                                       const rtucker_b200_als_ext* ext,
                                       rtucker_als_result** out);

/* Sessions: the same run split into steps, so a caller can time exactly K
 * sweeps (bench.py). create = init + initial loss; sweeps ignore tolerance. */
typedef struct rtucker_b200_session rtucker_b200_session;
rtucker_status rtucker_b200_session_create(const rtucker_tensor* x, const uint64_t* ranks,
                                           uint32_t order, const rtucker_als_options* opts,
                                           const rtucker_b200_als_ext* ext,
                                           rtucker_b200_session** out);
rtucker_status rtucker_b200_session_sweeps(rtucker_b200_session* s, uint32_t n);
rtucker_status rtucker_b200_session_result(rtucker_b200_session* s, rtucker_als_result** out);
void rtucker_b200_session_free(rtucker_b200_session* s);

/* Sweeps of a result that ran as one CUDA graph launch (from the second sweep on, when
 * the path allows it: sketched core with the CG solve, no per-kernel profiling, no
 * sharding; RTB_NO_GRAPH=1 disables). */
uint64_t rtucker_b200_result_graph_sweeps(const rtucker_als_result* r);

/* Device seconds of the sweep loop of a result (CUDA events). */
double rtucker_b200_result_sweep_seconds(const rtucker_als_result* r);

/* Model contents (host copies). core_out: prod ranks; factors_out: sum I_n*R_n. */
rtucker_status rtucker_b200_model_data(const rtucker_model* m, double* core_out,
                                       double* factors_out);
/* Build a model from host arrays (shape I_n, ranks R_n). */
rtucker_status rtucker_b200_model_create(const uint64_t* shape, const uint64_t* ranks,
                                         uint32_t order, const double* core,
                                         const double* factors, double lambda,
                                         rtucker_model** out);

/* Sketch diagnostics of the last core update of a result:
 * sample count, data-row draws, rank-deficiency flag, solver path (0 =
 * Cholesky, 1 = eigen pinv fallback). */
rtucker_status rtucker_b200_result_sketch_info(const rtucker_als_result* r,
                                               uint64_t* sample_count,
                                               uint64_t* data_draws,
                                               int* rank_deficient, int* solver_path);
/* solver_path: 0 Cholesky, 1 eigen/pinv fallback (d <= 64), 2 preconditioned CG.
 * CG iterations of the last sketched core solve (0 if CG was not used). */
int rtucker_b200_result_pcg_iterations(const rtucker_als_result* r);

/* Per-kernel device time accumulated over a run (CUDA events on the run's
 * stream). name_buf receives the kernel family name. */
uint64_t rtucker_b200_result_kernel_count(const rtucker_als_result* r);
rtucker_status rtucker_b200_result_kernel_row(const rtucker_als_result* r, uint64_t i,
                                              char* name_buf, size_t name_len,
                                              double* total_seconds, uint64_t* launches);

/* ---- parity-ladder entry points ---- */

/* Per-mode classical leverage scores, CDF and score sum on the GPU
 * (ref kronecker.cpp:9-35 with ridge_scores(svd, n, 0), leverage.cpp:16-37). */
rtucker_status rtucker_b200_factor_scores(const double* factor, uint64_t rows,
                                          uint64_t cols, double* scores_out,
                                          double* cdf_out, double* sum_out,
                                          uint64_t* rank_out);

/* Rung 1: draws s rows of the augmented Kronecker design on the GPU from
 * caller-supplied per-mode scores/CDFs/sums (concatenated over modes) and the
 * SplitMix64 seed, exactly as ProductLeverageSampler + solve_sketched_ridge
 * (ref kronecker.cpp:125-181, sketch_ridge.cpp:80-90). indices_out/weights_out
 * have length s. */
rtucker_status rtucker_b200_kron_draw(uint32_t order, const uint64_t* rows, uint64_t d,
                                      const double* scores, const double* cdfs,
                                      const double* sums, uint64_t seed, uint64_t s,
                                      uint64_t* indices_out, double* weights_out);

/* BASELINE config 4 microbench (Kronecker-product sampling + fused fiber gather/SYRK), all
 * buffers on the device: draws s rows of [A2 (x) A3; sqrt(lambda) I_W] (W = r2 r3) with the
 * reference's ProductLeverageSampler stream, then gram_dev (W x W, if non-NULL) = the
 * sketched Gram and rhs_dev (W x I1, if x_dev and rhs_dev are non-NULL) = sum over data
 * draws of w^2 (a2 (x) a3) X[:, j2, j3]^T, X being an I1 x I2 x I3 FP32 tensor (upcast in
 * the kernel). x_layout: 0 = canonical row-major (last index fastest), 1 = fiber-major
 * (mode 1 fastest: element (i1,i2,i3) at (i2 I3 + i3) I1 + i1, every mode-1 fiber
 * contiguous; see rtucker_b200_tensor_fiber_major). indices_out / weights_out (host, s
 * entries, optional) receive the draws; data_draws_out / unique_rows_out (optional) the
 * number of data draws and of distinct sampled rows; phase_ms_out[3] (optional) =
 * scores+draws, Gram (including the shared sort/merge of the draws), RHS device times.
 * r2, r3 <= 32. */
rtucker_status rtucker_b200_kron_fiber_sketch(const float* x_dev, const uint64_t* shape,
                                              uint32_t x_layout, const double* a2_dev,
                                              const double* a3_dev, uint32_t r2, uint32_t r3,
                                              double lambda, uint64_t s, uint64_t seed,
                                              double* gram_dev, double* rhs_dev,
                                              uint64_t* indices_out, double* weights_out,
                                              uint64_t* data_draws_out, uint64_t* unique_rows_out,
                                              double* phase_ms_out);

/* Sharded variant (multi-GPU, one process per GPU, X replicated): every shard decodes the
 * same draws, and shard r of P accumulates only the data draws with j2 in
 * [I2 r / P, I2 (r + 1) / P) (the augmented diagonal on shard 0), so the caller's sum
 * all-reduce of gram_dev and rhs_dev over the P shards gives the full Gram and RHS.
 * data_draws_out / unique_rows_out are the global counts. */
rtucker_status rtucker_b200_kron_fiber_sketch_shard(
    const float* x_dev, const uint64_t* shape, uint32_t x_layout, const double* a2_dev,
    const double* a3_dev, uint32_t r2, uint32_t r3, double lambda, uint64_t s, uint64_t seed,
    double* gram_dev, double* rhs_dev, uint64_t* indices_out, double* weights_out,
    uint64_t* data_draws_out, uint64_t* unique_rows_out, double* phase_ms_out,
    uint32_t shard_rank, uint32_t shard_count);

/* Fiber-major copy of a device FP32 tensor (shape[3] = I1, I2, I3, canonical row-major in):
 * out_dev[(i2 I3 + i3) I1 + i1] = x_dev[(i1 I2 + i2) I3 + i3]. */
rtucker_status rtucker_b200_tensor_fiber_major(const float* x_dev, const uint64_t* shape,
                                               float* out_dev);

/* Rung 3: sketched normal equations (gram d x d full, rhs d) of the augmented
 * Kronecker design from a caller-supplied RowSketch (ref
 * sketch_ridge.cpp:105-128). x is the host tensor (prod rows values). */
rtucker_status rtucker_b200_kron_normal_eq(uint32_t order, const uint64_t* rows,
                                           const uint64_t* ranks, const double* factors,
                                           const double* x, double lambda, uint64_t s,
                                           const uint64_t* indices, const double* weights,
                                           double* gram_out, double* rhs_out);

/* Rung 4: x = gram^+ rhs for a symmetric PSD gram (d x d): Cholesky on the GPU
 * with the eigen/pinv fallback (rank cutoff d*eps*lambda_max as ref
 * svd.cpp:92-97). *rank_out = numerical rank, *path_out = 0 Cholesky / 1 pinv. */
rtucker_status rtucker_b200_spd_solve(const double* gram, const double* rhs, uint64_t d,
                                      double* x_out, uint64_t* rank_out, int* path_out);

/* The dense toolkit's RowSketch (ref sampler.cpp:9-57, sketch_ridge.cpp:80-90): s draws of
 * AugmentedSampler(candidate_scores[n], d, d_eff_lower) from SplitMix64(seed) on the GPU;
 * indices in [0, n + d), weights sqrt((1/s)/prob). Bit-exact with the reference. */
rtucker_status rtucker_b200_aug_draw(const double* candidate_scores, uint64_t n, uint64_t d,
                                     double d_eff_lower, uint64_t seed, uint64_t s,
                                     uint64_t* indices_out, double* weights_out);
/* Sketched normal equations of [A; sqrt(lambda) I] (A n x d row-major, b n) from a given
 * RowSketch (ref sketch_ridge.cpp:105-128): gram_out d x d (full), rhs_out d. */
rtucker_status rtucker_b200_dense_normal_eq(const double* a, uint64_t n, uint64_t d,
                                            const double* b, double lambda, uint64_t s,
                                            const uint64_t* indices, const double* weights,
                                            double* gram_out, double* rhs_out);
/* The sample-count formula ceil(4 d / beta' max{420 ln(4 d / delta), 1 / (delta epsilon)})
 * (ref sketch_ridge.cpp:40-50); invalid arguments -> RTUCKER_ERR_INVALID_ARGUMENT. */
rtucker_status rtucker_b200_sample_count(double beta_prime, uint64_t d, double epsilon,
                                         double delta, uint64_t* out);

/* Symmetric eigendecomposition of a d x d matrix on the GPU: evals_out non-increasing,
 * evecs_out row-major with eigenvector k in column k. d <= 64: one-CTA cyclic Jacobi;
 * larger d: the parallel block Jacobi of the pinv fallback (k_eig.cu). */
rtucker_status rtucker_b200_sym_eig(const double* a, uint64_t d, double* evals_out,
                                    double* evecs_out);

/* One sketched core update on the GPU for a given model (ref tucker.cpp:141-166).
 * Optional outputs (NULL to skip): indices/weights of the drawn sketch. */
rtucker_status rtucker_b200_update_core_sketched(const rtucker_tensor* x,
                                                 const rtucker_model* m, uint64_t s,
                                                 uint64_t seed, double* core_out,
                                                 uint64_t* indices_out,
                                                 double* weights_out);
/* One exact factor update (ref tucker.cpp:70-89), mode 1-based. */
rtucker_status rtucker_b200_update_factor(const rtucker_tensor* x, const rtucker_model* m,
                                          uint32_t mode, double* factor_out);
/* Exact core update (ref tucker.cpp:91-129). */
rtucker_status rtucker_b200_update_core_exact(const rtucker_tensor* x,
                                              const rtucker_model* m, double* core_out);
/* Regularised loss and rmse of a model (ref tucker.cpp:47-68, 216-229). */
rtucker_status rtucker_b200_loss(const rtucker_tensor* x, const rtucker_model* m,
                                 double* loss_out, double* rmse_out);

#ifdef __cplusplus
}
#endif

#endif /* RTUCKER_B200_H */
