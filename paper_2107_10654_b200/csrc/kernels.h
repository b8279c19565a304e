// kernels.h -- host-side launchers of the sm_100a kernels (namespace rtb).
#pragma once
#include <functional>

#include <cstdint>
#include <cuda_runtime.h>

namespace rtb {

// Factor matrices of one model, passed by value to kernels.
struct FactorSet {
  const double* ptr[8];
  int rows[8];
  int cols[8];
  int order;
};

// ---- k_small.cu ----
__global__ void k_factor_gram(const FactorSet fs, double* grams, int r_max);
__global__ void k_sym_eigen(const double* in, const int* ns, int stride, double* evals,
                            double* evecs, int* status);
__global__ void k_sym_eigen_warp(const double* in, const int* ns, int stride, double* evals,
                                 double* evecs, int* status, int nmat, const int* skip);
// symmetric eigensolver dispatch: warp-per-matrix for n <= 32, else CTA (n <= 64)
void sym_eigen(const double* in, const int* ns_dev, int nmax, int stride, double* evals,
               double* evecs, int* status, int nmat, cudaStream_t st, const int* skip = nullptr);
__global__ void k_leverage_rows(const FactorSet fs, const double* evals, const double* evecs,
                                int stride, double lambda, double* scores,
                                const long long* score_off, int* ranks, const int* skip);
void leverage_chol(const FactorSet& fs, const double* linv, int stride, const int* ok,
                   double* scores, const long long* score_off, int* ranks, int max_rows,
                   int nmodes, int rmax, cudaStream_t st);
// batched small SPD Cholesky (n <= 32): Linv (+ optional P = M^-1), ok flags
void spd_small(const double* in, const int* ns_dev, int stride, double tolrel, double* linv,
               double* pinv, int* ok, int nmat, cudaStream_t st, int nmax = 32);
// one-sided Jacobi SVD scores of each matrix b of fs with n <= 32 columns (k_hjsvd.cu),
// skipped where skip[b]; one CTA of 512 threads per matrix, workspace work_stride doubles each
__global__ void k_hj_cta(const FactorSet fs, double* work, long long work_stride, double lambda,
                         double* scores, const long long* score_off, int* ranks, const int* skip,
                         int* status);
size_t hj_work_bytes(long long rows, int cols);
void hj_ridge_scores(const double* A, long long rows, int cols, double lambda, double* scores,
                     int* rank, void* work, cudaStream_t st);
__global__ void k_score_cdf(const double* scores, const long long* off, const int* rows,
                            int order, double* cdf, double* sums);
__global__ void k_sym_pinv(const double* evals, const double* evecs, const int* ns, int stride,
                           double* out, int* ranks, const int* skip);
__global__ void k_rows_times_small(const double* M, const double* P, int I, int R, double* out);

// ---- k_ttm.cu ----
// While a guard is set (non-null), ttm_last / ttm_generic / ttm_expand / sum_partials
// kernels do nothing unless *need != 0 at run time (nullptr clears the guard).
void set_ttm_guard(const int* need);
// partial count of the last ttm_last / ttm_last_resid launch of this host thread
long long ttm_last_blocks(long long O, int I, int R);
// upper bound on that count for any path (workspace sizing)
long long ttm_last_parts_bound(long long O, int I, int R);
// T (O x R) = X (O x I) A (I x R); if P != null also partial[block] = sum (X - P A^T)^2
// With W != nullptr (3-way), P is not read but generated per row: P[(i1,i2),:] =
// A2[i2,:] W[i1] with W = G x_1 A_1 (I1 x R2 x R3) -- saves writing / reading P.
void ttm_last(const double* X, long long O, int I, const double* A, int R, double* T,
              const double* P, double* partial, cudaStream_t st, const double* W = nullptr,
              const double* A2 = nullptr, int I2 = 0, int R2 = 0);
bool ttm_last_pgen_ok(int I, int R);
// partial[block] = sum (X - P A^T)^2 alone (no T), when the tensor-map kernel applies
// (R <= 16); false: not launched, use ttm_last. Same partial count as ttm_last_blocks.
bool ttm_last_resid(const double* X, long long O, int I, const double* A, int R, const double* P,
                    double* partial, cudaStream_t st);
// out[o,r,j] = sum_i A[i,r] X[o,i,j]
void ttm_mid(const double* X, long long O, int I, long long J, const double* A, int R, double* out,
             cudaStream_t st);
// out[o,r,j] = sum_i W[r*wr + i*wi] X[o,i,j]
void ttm_generic(const double* X, long long O, int I, long long J, const double* W, long long wr,
                 long long wi, int R, double* out, cudaStream_t st);
// out[o,r,j] = sum_i A[i,r] X[o,i,j], J <= 32 (returns false if not applicable)
bool ttm_smallj(const double* X, long long O, int I, int J, const double* A, int R, double* out,
                cudaStream_t st);
// out[o,i,j] = sum_r A[i,r] Y[o,r,j] (returns false if not applicable)
bool ttm_expand(const double* Y, long long O, int R, long long J, const double* A, int I,
                double* out, cudaStream_t st);
// M[i,r] = sum_{o,j} Y[o,i,j] G[o,r,j]
// F_1 / F_2 (n = 0 / 1) of an order-3 exact factor update straight from T (I1 x I2 x R3):
// M[u, :] = G_(n) vec(A_m^T T-slice_u) for every u of mode n; false if not applicable (R > 16)
bool fu_proj3(const double* T, int I1, int I2, int R3, const double* Am, int Rm, const double* G,
              int R1, int R2, int n, double* M, cudaStream_t st);
void contract_except(const double* Y, const double* G, long long O, int I, int R, long long J,
                     double* M, cudaStream_t st);
void sum_partials(const double* partial, long long n, double* out, cudaStream_t st);

// ---- k_draw.cu ----
struct DrawSpec {
  int order;
  long long rows[8];        // I_n
  long long cdf_off[8];     // offset of mode n in the concatenated score/CDF arrays
  unsigned long long total_rows;  // prod I_n
  unsigned long long d;     // prod R_n (augmented block size)
  unsigned long long seed;
  unsigned long long s;     // number of draws
  // non-null: the seed is read on the device at run time (a CUDA-graph-captured sweep
  // draws with a new seed every launch); `seed` is then ignored
  const unsigned long long* seed_dev;
};
struct DrawWork {          // device scratch, sized by draw_work_bytes
  void* base;
  size_t bytes;
};
size_t draw_work_bytes(const DrawSpec& spec);
// Decodes the sequential SplitMix64 draw stream in parallel and evaluates all
// s draws: indices (u64, reference format) and weights.
void draw_sketch(const DrawSpec& spec, const double* scores, const double* cdfs,
                 const double* sums, DrawWork work, unsigned long long* idx_out,
                 double* w_out, int* flag_dev, cudaStream_t st);
// the two halves of draw_sketch: stream positions (no CDFs needed), then evaluation
void draw_decode(const DrawSpec& spec, DrawWork work, cudaStream_t st);
// after draw_decode: the Gram's bucket keys from the first mode's CDF alone (k_draw_keys)
void draw_keys(const DrawSpec& spec, const double* scores, const double* cdfs, const double* sums,
               DrawWork work, int i1_lo, int i1_hi, unsigned* keys, unsigned* vals, int* counts,
               int* aug_count, unsigned long long* data_draws, cudaStream_t st);
void draw_evaluate(const DrawSpec& spec, const double* scores, const double* cdfs,
                   const double* sums, DrawWork work, unsigned long long* idx_out,
                   double* w_out, int* flag_dev, cudaStream_t st);

// ---- k_fsketch.cu: sketched factor update (perf mode) ----
struct FactorSketchSpec {
  int order;
  int mode;                 // 0-based
  int rows[8], ranks[8];
  const double* factors[8];
  const double* core;
  const double* x;
  double lambda;
  unsigned long long s;     // draws (indices over the other modes + R_n augmented rows)
  // 1: x is the mode-n-last copy of X (axes: the other modes ascending, then mode n;
  // move_axis_last), so every sampled fiber is one contiguous run of I_n values
  int x_mode_last = 0;
  // multi-GPU (X split along mode 1): x holds mode-1 rows [shard_lo, shard_lo + shard_rows)
  // (shard_rows = 0: the whole tensor). Draws are decoded with the global rows. For mode n > 0
  // only this shard's data draws contribute (partial Gram / M, to be summed over shards) and
  // the augmented rows only where count_aug; for n == 0 the fibers are this shard's segments
  // (M has shard_rows rows) and the Gram is the whole one on every shard.
  int shard_lo = 0, shard_rows = 0, count_aug = 1;
};
// out = X with axis of length In moved last: X viewed as [A][In][B] -> out [A][B][In]
void move_axis_last(const double* x, long long A, int In, long long B, double* out,
                    cudaStream_t st);
size_t factor_sketch_work_bytes(const FactorSketchSpec& spec);
// gram (R_n x R_n) and M (I_n x R_n) from the draws idx/w (k_draw.cu format with
// total_rows = prod_{m != n} I_m, d = R_n)
void factor_sketch_normal_eq(const FactorSketchSpec& spec, const unsigned long long* idx,
                             const double* w, void* work, double* gram, double* M,
                             cudaStream_t st);

// ---- FP64 DMMA GEMM (k_c4.cu): out[m][n] = sum_k A[k][m] B[k][n] (A: K x M, B: K x N,
// row-major with leading dims), optionally batched (blockIdx.z; strides sA, sB, sO) ----
void gemm_tn(const double* A, long long lda, const double* B, long long ldb, int M, long long N,
             int K, double* out, long long ldo, cudaStream_t st, int batch = 1, long long sA = 0,
             long long sB = 0, long long sO = 0);

// ---- k_c4.cu: BASELINE config-4 microbench (Kronecker sampling + fused fiber gather/SYRK) ----
size_t c4_work_bytes(unsigned long long s, int I1, int I2, int I3, int R2, int R3, bool gram);
// canonical row-major I1 x I2 x I3 -> fiber-major (mode 1 fastest: out[(i2 I3 + i3) I1 + i1])
void c4_to_fiber_major(const float* x, int I1, int I2, int I3, float* out, cudaStream_t st);
// From draws (idx, w) of [A2 (x) A3; sqrt(lambda) I]: gram (W x W, W = R2 R3, if non-null) and
// rhs (W x I1, if x and rhs are non-null) = sum over data draws of w^2 (a2 (x) a3) X[:, j2, j3]^T.
// Sharded (shard_count > 1): only the draws with j2 in this shard's range [I2 r / P, I2 (r+1) / P)
// contribute (the augmented diagonal on shard 0): the shards' gram / rhs sum to the full ones.
// X is FP32, canonical or fiber-major. *data_draws_dev / *unique_dev (optional): data draws and
// distinct sampled rows. ev_gram_done (optional) is recorded after the Gram.
void c4_sketch(const float* x, bool fiber_major, int I1, int I2, int I3, const double* A2, int R2,
               const double* A3, int R3, const unsigned long long* idx, const double* w,
               unsigned long long s, double lambda, void* work, size_t work_bytes, double* gram,
               double* rhs, unsigned long long* data_draws_dev, unsigned long long* unique_dev,
               cudaEvent_t ev_gram_done, cudaStream_t st, int shard_rank = 0, int shard_count = 1);

// ---- k_gram.cu ----
struct GramSpec {
  int order;
  int rows[8];
  int ranks[8];
  const double* factors[8];
  unsigned long long total_rows;
  int d;          // prod R_n
  int dprime;     // prod_{n>=1} R_n (z width)
  double lambda;
  unsigned long long s;
  // multi-GPU: only data draws with i1 in [i1_lo, i1_hi) contribute (this shard's X
  // slab; x points at the slab minus i1_lo * prod_{n>=2} I_n). Augmented draws are
  // counted by every shard. i1_hi == 0 means no sharding.
  int i1_lo, i1_hi;
};
size_t gram_work_bytes(const GramSpec& spec);
// keys ahead (order 3): the workspace's key buffers, their reset, and the sort + bucket table
// + bucket order that sketch_normal_eq(..., keys_ready = true) then skips
struct GramKeyBufs {
  unsigned* keys;
  unsigned* vals;
  int* counts;
  int* aug_count;
};
GramKeyBufs gram_key_buffers(const GramSpec& spec, void* work);
void gram_keys_reset(const GramSpec& spec, void* work, unsigned long long* data_draws_dev,
                     cudaStream_t st);
void gram_sort_keys(const GramSpec& spec, void* work, cudaStream_t st);
// the compact (vech) Gram S [m_1][Hsz] inside the workspace (sum it across shards)
double* gram_compact(const GramSpec& spec, void* work, size_t* count);
// Sketched normal equations from (idx, w): rhs, the compact (vech) Gram in the
// workspace and, if gram != nullptr, the full d x d Gram. With blocks != nullptr the last-mode
// blocks (gram_expand_blocks' output) may be written by the same pass: returns true if so.
bool sketch_normal_eq(const GramSpec& spec, const double* x, const unsigned long long* idx,
                      const double* w, void* work, size_t work_bytes, double* gram,
                      double* rhs, unsigned long long* data_draws_dev, cudaStream_t st,
                      double* blocks = nullptr, bool keys_ready = false);

// augmented-row draw counts [d] inside a gram workspace (valid after sketch_normal_eq)
const int* gram_aug_counts(const GramSpec& spec, void* work);
// diagonal term each augmented draw adds
double gram_aug_term(const GramSpec& spec);
// full Gram / last-mode blocks (data part only) from the workspace's compact Gram
void gram_expand_full(const GramSpec& spec, void* work, double* gram, cudaStream_t st);
long long gram_block_elems(const GramSpec& spec);
void gram_expand_blocks(const GramSpec& spec, void* work, double* blocks, cudaStream_t st);
// the blocks of the mode-1 slices u1 in [u_lo, u_hi) only (a distributed solve's share)
void gram_expand_blocks_range(const GramSpec& spec, void* work, double* blocks, int u_lo, int u_hi,
                              cudaStream_t st);

// ---- k_pcg.cu ----
struct PcgSpec {
  int order;
  int ranks[8];
  int d;
  double lambda;
  const double* pinv;   // per mode (stride linv_stride): (A_n^T A_n)^-1 (k_spd_small)
  int linv_stride;
  const int* linv_ok;   // per mode: Cholesky succeeded (any 0 -> status 3)
  const double* grams;  // per mode (same stride): A_n^T A_n
  const double* evals;  // per mode (same stride): eigenpairs of A_n^T A_n (eigen-form
  const double* evecs;  //   preconditioner when lambda is not small against mu_min)
  const double* prep;   // [3] from pcg_prepare
  const int* aug_count; // [d] augmented draws per column (any 0 -> status 3)
  double aug_term;      // diagonal added per augmented draw
  int max_iter;
  double tol;           // stop when ||r_k|| <= tol max(||b||, ||G||~ ||x_k||)
  double check_tol;     // accept when ||b - G x|| <= check_tol (||G||~ ||x|| + ||b||)
  int warm = 0;         // 1: x holds a starting guess (kept if ||b - G x0|| < ||b||)
  const int* warm_dev = nullptr;  // non-null: the warm flag is read on the device
};
size_t pcg_work_bytes(int d, int r1);
// with the per-CTA vector slices of the large-d form (vectors beyond shared memory)
size_t pcg_work_bytes(int d, int order, const int* ranks);
// norm estimates and preconditioner form (prep_dev[3]); skip_dev[order] = 1 where the
// factor-Gram eigenpairs are not needed (feed to sym_eigen as skip flags)
void pcg_prepare(const PcgSpec& spec, double* prep_dev, int* skip_dev, cudaStream_t st);
bool pcg_supported(int d, int order, const int* ranks);
// x = G^-1 b by Kronecker-preconditioned CG; status_dev[0] = 0 ok, 1 residual check
// failed, 2 breakdown (non-SPD), 3 not applicable; status_dev[1] = iterations.
// G is given as its last-mode blocks (gram_expand_blocks) + augmented diagonal.
// the split-role form (order 3, R_3 = 16): the compact vech Gram S [m_1][m_2 * 136] is held
// in shared memory across the solve (k_pcg_split); same contract as pcg_solve
bool pcg_split_ok(int d, int order, const int* ranks);
void pcg_solve_compact(const PcgSpec& spec, const double* S, const double* b, double* x,
                       void* work, int* status_dev, cudaStream_t st);
// Distributed large-d solve (multi-GPU): rank `rank` of `count` holds the blocks of its mode-1
// slices only (pcg_dist_slices; gram_expand_blocks_range) and the ranks' matvec shares are
// summed by `allreduce(q, d)` between launches; every rank ends with the same x and status.
// 16 ints of pinned host memory from a per-process pool (engine.cu), and their return
int* pinned_slot();
void pinned_slot_free(int* p);
bool pcg_dist_ok(int d, int order, const int* ranks);
void pcg_dist_slices(int m1, int rank, int count, int* u_lo, int* u_hi);
void pcg_solve_dist(const PcgSpec& spec, const double* blocks_local, int rank, int count,
                    const double* b, double* x, void* work, int* status_dev, cudaStream_t st,
                    const std::function<void(double*, size_t)>& allreduce);
void pcg_solve(const PcgSpec& spec, const double* blocks, const double* b, double* x, void* work,
               int* status_dev, cudaStream_t st);

// ---- k_eig.cu: symmetric eigendecomposition (parallel block Jacobi, d > 64) and
// x = G^+ b with the reference cutoff d eps max|mu| ----
size_t eig_large_work_bytes(int d);
// evals[d] (unsorted) and evecs (d x d row-major, column k = eigenvector k; optional)
void sym_eig_large(const double* A, int d, double* evals, double* evecs, void* work,
                   cudaStream_t st);
size_t pinv_large_work_bytes(int d);
// G (d x d symmetric, device) is left unchanged; *rank_dev = number of kept eigenpairs
void pinv_solve_large(double* G, int d, const double* b, double* x, int* rank_dev, void* work,
                      size_t work_bytes, cudaStream_t st);

// ---- k_chol.cu ----
size_t chol_work_bytes(int d);
// In-place Cholesky of the lower triangle of a (d x d, row-major) and solve
// a x = b (x overwrites b). *status_dev = 0 ok, k+1 = non-positive pivot at k.
void chol_solve(double* a, int d, double* b, int* status_dev, void* work, cudaStream_t st);
// profiling hooks: per-task (grab, ready, end, smid) into a device buffer
void chol_set_trace(unsigned long long* trace);
void chol_set_progress(volatile int* p);
void chol_debug(int d, void* work, int* out4);  // abort flag, flag index, value, wanted
int chol_task_count(int d);
void chol_task_table(int d, int* out4);

}  // namespace rtb
