// toolkit.cu -- the reference's dense ridge toolkit on the GPU (ref capi.cpp:299-362):
//   rtucker_ridge_scores   ridge leverage scores of a dense A (leverage.cpp:39-52) by the
//                          one-sided Jacobi SVD of A (k_hjsvd.cu), any shape, any lambda >= 0
//   rtucker_solve_ridge    x = pinv(A^T A + lambda I) A^T b (linalg.cpp:28-41): the Gram by
//                          split-K DMMA GEMMs, Cholesky, the block-Jacobi pinv behind it
//   rtucker_sketched_ridge AugmentedSampler draws (sampler.cpp:9-57, bit-exact given the
//                          scores), the sketched normal equations (sketch_ridge.cpp:105-128)
//                          as one DMMA GEMM over the gathered weighted rows, then the solve
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <vector>

#include "engine.h"
#include "kernels.h"

namespace rtb {

size_t hj_work_bytes(long long rows, int cols);
void hj_ridge_scores(const double* A, long long rows, int cols, double lambda, double* scores,
                     int* rank, void* work, cudaStream_t st);
void solve_sym_device(double* G, double* rhs, int d, double* x_dev, int* rank, int* path,
                      cudaStream_t st);

namespace {

__global__ void k_any_nonzero(const double* a, long long n, int* flag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && a[i] != 0.0) atomicExch(flag, 1);
}

__global__ void k_add_diag_t(double* a, int n, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[(size_t)i * n + i] += v;
}

// out[j] = sum_i a[i][j] b[i] (one block per column, fixed-order partials + tree)
__global__ void k_atb(const double* a, long long n, int d, const double* b, double* out) {
  __shared__ double red[32];
  const int j = blockIdx.x;
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s = fma(a[i * d + j], b[i], s);
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) out[j] = s;
}

// sum of `parts` partial d x d blocks in index order (+ optional accumulate into out)
__global__ void k_sum_parts(const double* __restrict__ part, long long elems, int parts,
                            double* __restrict__ out, int accumulate) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= elems) return;
  double s = accumulate ? out[e] : 0.0;
  for (int p = 0; p < parts; ++p) s += part[(long long)p * elems + e];
  out[e] = s;
}

// AugmentedSampler tables, sequential like the reference (sampler.cpp:9-40):
// out[0] = data_mass, out[1] = aug_mass_per_row, out[2] = total_mass; flag on bad input.
__global__ void k_aug_tables(const double* cand, long long n, int d, double d_eff_lower,
                             double* norm, double* cum, double* out, int* flag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double l1 = 0.0;
  for (long long i = 0; i < n; ++i) {
    const double s = cand[i];
    if (!(s >= 0.0) || !isfinite(s)) {
      *flag = 1;
      return;
    }
    l1 = __dadd_rn(l1, s);
  }
  if (l1 <= 0.0) {
    *flag = 2;
    return;
  }
  const double scale = __ddiv_rn((double)d, l1);
  double running = 0.0;
  for (long long i = 0; i < n; ++i) {
    norm[i] = __dmul_rn(cand[i], scale);
    running = __dadd_rn(running, norm[i]);
    cum[i] = running;
  }
  const double m = __dadd_rn((double)d, -d_eff_lower);
  const double aug = m < 1.0 ? m : 1.0;
  out[0] = running;
  out[1] = aug;
  out[2] = __dadd_rn(running, __dmul_rn((double)d, aug));
}

// one u64 per draw: draw t uses stream output t (sampler.cpp:42-57); the reference's IEEE
// operation sequence, so indices and weights are bitwise those of the reference
__global__ void k_aug_draw(const double* norm, const double* cum, long long n, int d,
                           const double* tab, unsigned long long seed, long long s,
                           unsigned long long* idx, double* w) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  const double data_mass = tab[0], aug = tab[1], total = tab[2];
  const double inv_s = __ddiv_rn(1.0, (double)s);
  const double u = __dmul_rn(u64_to_unit(sm_at(seed, (uint64_t)t)), total);
  double prob;
  unsigned long long index;
  if (u < data_mass || aug == 0.0) {
    const double key = u < data_mass ? u : data_mass;
    long long lo = 0, len = n;
    while (len > 0) {
      const long long half = len >> 1;
      if (!(key < cum[lo + half])) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    long long i = lo >= n ? n - 1 : lo;
    while (i > 0 && norm[i] == 0.0) --i;
    index = (unsigned long long)i;
    prob = __ddiv_rn(norm[i], total);
  } else {
    long long k = (long long)__ddiv_rn(__dadd_rn(u, -data_mass), aug);
    if (k >= d) k = d - 1;
    index = (unsigned long long)(n + k);
    prob = __ddiv_rn(aug, total);
  }
  idx[t] = index;
  w[t] = __dsqrt_rn(__ddiv_rn(inv_s, prob));
}

// weighted rows of the data draws [t0, t0 + rows): B[t - t0] = w_t a_{j_t}, wb[t - t0] =
// w_t b_{j_t}; augmented draws give zero rows and are counted per column instead
__global__ void k_dense_gather(const double* __restrict__ a, long long n, int d,
                               const double* __restrict__ b, const unsigned long long* __restrict__ idx,
                               const double* __restrict__ w, long long t0, long long rows,
                               double* __restrict__ B, double* __restrict__ wb,
                               int* __restrict__ aug_cnt, double* aug_w2) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * d) return;
  const long long r = e / d;
  const int c = (int)(e % d);
  const unsigned long long j = idx[t0 + r];
  const double wt = w[t0 + r];
  if (j < (unsigned long long)n) {
    B[e] = wt * a[(long long)j * d + c];
    if (c == 0) wb[r] = wt * b[j];
  } else {
    B[e] = 0.0;
    if (c == 0) {
      wb[r] = 0.0;
      atomicAdd(aug_cnt + (j - n), 1);
      *aug_w2 = wt * wt;  // every augmented draw has the same probability, so the same weight
    }
  }
}

// G[k][k] += count_k w_aug^2 lambda (the sqrt(lambda) e_k rows, sketch_ridge.cpp:18-36)
__global__ void k_aug_diag(double* G, int d, const int* cnt, const double* aug_w2, double lambda) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d || cnt[k] == 0) return;
  G[(size_t)k * d + k] += (double)cnt[k] * (*aug_w2 * lambda);
}

}  // namespace

// G (d x d) = X^T X (+= if accumulate) for X (rows x d, device): split-K DMMA GEMMs
// (k_gemm_tn) into partial blocks summed in a fixed order.
static void gram_splitk(const double* X, long long rows, int d, double* G, bool accumulate,
                        cudaStream_t st) {
  const long long dd = (long long)d * d;
  const long long max_parts = std::max<long long>(1, (1LL << 24) / std::max<long long>(dd, 1));
  long long parts = std::min<long long>(std::max<long long>(1, rows / 256), max_parts);
  parts = std::min<long long>(parts, 4096);
  const long long kc = (rows + parts - 1) / parts;
  parts = (rows + kc - 1) / kc;
  DevBuf pb((size_t)parts * dd * 8, st);
  const long long full = rows / kc;  // batches with exactly kc rows
  if (full > 0)
    gemm_tn(X, d, X, d, d, d, (int)kc, pb.as<double>(), d, st, (int)full, kc * d, kc * d, dd);
  if (full < parts) {
    const long long r0 = full * kc;
    gemm_tn(X + r0 * d, d, X + r0 * d, d, d, d, (int)(rows - r0), pb.as<double>() + full * dd, d,
            st);
  }
  k_sum_parts<<<(unsigned)ceil_div<long long>(dd, 256), 256, 0, st>>>(pb.as<double>(), dd,
                                                                      (int)parts, G, accumulate);
  RTB_LAUNCH_CHECK();
}

void dense_ridge_scores(const double* a, uint64_t n, uint64_t d, double lambda, double* out) {
  if (lambda < 0.0) throw Error(1, "ridge_scores: lambda must be non-negative");
  if (n == 0 || d == 0) throw Error(1, "compact_svd: empty matrix");
  if (d > (uint64_t)INT32_MAX || n > (uint64_t)INT32_MAX) throw Error(1, "ridge_scores: too large");
  cudaStream_t st = current_stream();
  DevBuf ad(n * d * 8, st), sc(n * 8, st), nz(4, st);
  RTB_CUDA(cudaMemcpyAsync(ad.p, a, n * d * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemsetAsync(nz.p, 0, 4, st));
  k_any_nonzero<<<(unsigned)ceil_div<uint64_t>(n * d, 256), 256, 0, st>>>(ad.as<double>(),
                                                                        (long long)(n * d),
                                                                        nz.as<int>());
  RTB_LAUNCH_CHECK();
  int any = 0;
  RTB_CUDA(cudaMemcpyAsync(&any, nz.p, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (!any) {  // zero rows score zero (ref leverage.cpp:40-50)
    std::memset(out, 0, n * 8);
    return;
  }
  DevBuf work(hj_work_bytes((long long)n, (int)d), st);
  int rank = 0;
  hj_ridge_scores(ad.as<double>(), (long long)n, (int)d, lambda, sc.as<double>(), &rank, work.p,
                  st);
  RTB_CUDA(cudaMemcpyAsync(out, sc.p, n * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
}

void dense_solve_ridge(const double* a, uint64_t n, uint64_t d, const double* b, double lambda,
                       double* x) {
  if (lambda < 0.0) throw Error(1, "solve_ridge_exact: lambda must be non-negative");
  if (d == 0) throw Error(1, "compact_svd: empty matrix");
  cudaStream_t st = current_stream();
  DevBuf ad(n * d * 8 + 8, st), bd(n * 8 + 8, st), g(d * d * 8, st), atb(d * 8, st),
      xd(d * 8, st);
  RTB_CUDA(cudaMemcpyAsync(ad.p, a, n * d * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(bd.p, b, n * 8, cudaMemcpyHostToDevice, st));
  if (n > 0) {
    gram_splitk(ad.as<double>(), (long long)n, (int)d, g.as<double>(), false, st);
  } else {
    RTB_CUDA(cudaMemsetAsync(g.p, 0, d * d * 8, st));
  }
  k_add_diag_t<<<(unsigned)ceil_div<uint64_t>(d, 64), 64, 0, st>>>(g.as<double>(), (int)d, lambda);
  RTB_LAUNCH_CHECK();
  k_atb<<<(unsigned)d, 256, 0, st>>>(ad.as<double>(), (long long)n, (int)d, bd.as<double>(),
                                     atb.as<double>());
  RTB_LAUNCH_CHECK();
  int rk = 0, path = 0;
  solve_sym_device(g.as<double>(), atb.as<double>(), (int)d, xd.as<double>(), &rk, &path, st);
  RTB_CUDA(cudaMemcpyAsync(x, xd.p, d * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
}

// AugmentedSampler tables + draws on the device buffers (cand: n scores)
static void aug_draw_dev(const double* cand_dev, uint64_t n, uint64_t d, double d_eff_lower,
                         uint64_t s, uint64_t seed, unsigned long long* idx, double* w,
                         double* norm, double* cum, double* tab, int* flag, cudaStream_t st) {
  RTB_CUDA(cudaMemsetAsync(flag, 0, 4, st));
  k_aug_tables<<<1, 1, 0, st>>>(cand_dev, (long long)n, (int)d, d_eff_lower, norm, cum, tab, flag);
  RTB_LAUNCH_CHECK();
  int f = 0;
  RTB_CUDA(cudaMemcpyAsync(&f, flag, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (f == 1) throw Error(1, "AugmentedSampler: scores must be finite and non-negative");
  if (f == 2) throw Error(1, "AugmentedSampler: scores must not all be zero");
  k_aug_draw<<<(unsigned)ceil_div<uint64_t>(s, 256), 256, 0, st>>>(norm, cum, (long long)n, (int)d,
                                                                  tab, seed, (long long)s, idx, w);
  RTB_LAUNCH_CHECK();
}

static void check_aug_args(uint64_t d, double d_eff_lower) {
  if (d == 0) throw Error(1, "AugmentedSampler: d must be positive");
  if (d_eff_lower < 0.0 || d_eff_lower > (double)d)
    throw Error(1, "AugmentedSampler: d_eff_lower outside [0, d]");
}

void aug_draw(const double* cand, uint64_t n, uint64_t d, double d_eff_lower, uint64_t seed,
              uint64_t s, uint64_t* idx_out, double* w_out) {
  check_aug_args(d, d_eff_lower);
  if (n == 0) throw Error(1, "AugmentedSampler: scores must not all be zero");
  if (s == 0) throw Error(1, "solve_sketched_ridge: sample count must be >= 1");
  cudaStream_t st = current_stream();
  DevBuf sc(n * 8, st), nm(n * 8, st), cm(n * 8, st), tab(32, st), fl(4, st), ix(s * 8, st),
      ww(s * 8, st);
  RTB_CUDA(cudaMemcpyAsync(sc.p, cand, n * 8, cudaMemcpyHostToDevice, st));
  aug_draw_dev(sc.as<double>(), n, d, d_eff_lower, s, seed, (unsigned long long*)ix.p,
               ww.as<double>(), nm.as<double>(), cm.as<double>(), tab.as<double>(), fl.as<int>(),
               st);
  RTB_CUDA(cudaMemcpyAsync(idx_out, ix.p, s * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(w_out, ww.p, s * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
}

// sketched normal equations of [A; sqrt(lambda) I] from device draws: gathered weighted data
// rows (in chunks of at most ~1 GB) -> one split-K DMMA Gram each, rhs by a column
// reduction, the augmented draws as per-column counts on the diagonal
static void dense_normal_eq_dev(const double* a, uint64_t n, uint64_t d, const double* b,
                                double lambda, const unsigned long long* idx, const double* w,
                                uint64_t s, double* G, double* rhs, cudaStream_t st) {
  const long long chunk =
      std::max<long long>(1, std::min<long long>((long long)s, (1LL << 27) / (long long)d));
  DevBuf B((size_t)chunk * d * 8, st), wb((size_t)chunk * 8, st), cnt(d * 4 + 8, st),
      w2(8, st), rp(d * 8, st);
  RTB_CUDA(cudaMemsetAsync(cnt.p, 0, d * 4, st));
  RTB_CUDA(cudaMemsetAsync(w2.p, 0, 8, st));
  RTB_CUDA(cudaMemsetAsync(rhs, 0, d * 8, st));
  bool first = true;
  for (long long t0 = 0; t0 < (long long)s; t0 += chunk) {
    const long long rows = std::min<long long>(chunk, (long long)s - t0);
    k_dense_gather<<<(unsigned)ceil_div<long long>(rows * (long long)d, 256), 256, 0, st>>>(
        a, (long long)n, (int)d, b, idx, w, t0, rows, B.as<double>(), wb.as<double>(),
        cnt.as<int>(), w2.as<double>());
    RTB_LAUNCH_CHECK();
    gram_splitk(B.as<double>(), rows, (int)d, G, !first, st);
    k_atb<<<(unsigned)d, 256, 0, st>>>(B.as<double>(), rows, (int)d, wb.as<double>(),
                                       rp.as<double>());
    RTB_LAUNCH_CHECK();
    k_sum_parts<<<(unsigned)ceil_div<uint64_t>(d, 256), 256, 0, st>>>(rp.as<double>(), (long long)d,
                                                                     1, rhs, 1);
    RTB_LAUNCH_CHECK();
    first = false;
  }
  k_aug_diag<<<(unsigned)ceil_div<uint64_t>(d, 256), 256, 0, st>>>(G, (int)d, cnt.as<int>(),
                                                                  w2.as<double>(), lambda);
  RTB_LAUNCH_CHECK();
}

void dense_normal_eq(const double* a, uint64_t n, uint64_t d, const double* b, double lambda,
                     uint64_t s, const uint64_t* idx, const double* w, double* gram, double* rhs) {
  if (d == 0 || s == 0) throw Error(1, "dense_normal_eq: d and s must be positive");
  for (uint64_t t = 0; t < s; ++t)
    if (idx[t] >= n + d) throw Error(1, "dense_normal_eq: row index out of range");
  cudaStream_t st = current_stream();
  DevBuf ad(n * d * 8 + 8, st), bd(n * 8 + 8, st), ix(s * 8, st), ww(s * 8, st), G(d * d * 8, st),
      r(d * 8, st);
  RTB_CUDA(cudaMemcpyAsync(ad.p, a, n * d * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(bd.p, b, n * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(ix.p, idx, s * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(ww.p, w, s * 8, cudaMemcpyHostToDevice, st));
  dense_normal_eq_dev(ad.as<double>(), n, d, bd.as<double>(), lambda,
                      (const unsigned long long*)ix.p, ww.as<double>(), s, G.as<double>(),
                      r.as<double>(), st);
  RTB_CUDA(cudaMemcpyAsync(gram, G.p, d * d * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(rhs, r.p, d * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
}

void dense_sketched_ridge(const double* a, uint64_t n, uint64_t d, const double* b,
                          const double* cand, double lambda, double d_eff_lower, double eps,
                          double delta, uint64_t s_override, uint64_t seed, double* x,
                          uint64_t* s_out, double* beta_out) {
  check_aug_args(d, d_eff_lower);
  if (lambda < 0.0) throw Error(1, "solve_sketched_ridge: lambda must be non-negative");
  std::vector<double> scores(n);
  if (cand) std::memcpy(scores.data(), cand, n * 8);
  else dense_ridge_scores(a, n, d, 0.0, scores.data());  // classical_scores
  cudaStream_t st = current_stream();
  const double m = std::min(1.0, (double)d - d_eff_lower);
  const double beta_prime = 1.0 / (1.0 + m);
  const uint64_t s = s_override ? s_override : sample_count_formula(beta_prime, d, eps, delta);
  DevBuf ad(n * d * 8 + 8, st), bd(n * 8 + 8, st), sc(n * 8 + 8, st), nm(n * 8 + 8, st),
      cm(n * 8 + 8, st), tab(32, st), fl(4, st), ix(s * 8, st), ww(s * 8, st), G(d * d * 8, st),
      r(d * 8, st), xd(d * 8, st);
  RTB_CUDA(cudaMemcpyAsync(ad.p, a, n * d * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(bd.p, b, n * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(sc.p, scores.data(), n * 8, cudaMemcpyHostToDevice, st));
  aug_draw_dev(sc.as<double>(), n, d, d_eff_lower, s, seed, (unsigned long long*)ix.p,
               ww.as<double>(), nm.as<double>(), cm.as<double>(), tab.as<double>(), fl.as<int>(),
               st);
  dense_normal_eq_dev(ad.as<double>(), n, d, bd.as<double>(), lambda,
                      (const unsigned long long*)ix.p, ww.as<double>(), s, G.as<double>(),
                      r.as<double>(), st);
  int rk = 0, path = 0;
  solve_sym_device(G.as<double>(), r.as<double>(), (int)d, xd.as<double>(), &rk, &path, st);
  RTB_CUDA(cudaMemcpyAsync(x, xd.p, d * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (s_out) *s_out = s;
  if (beta_out) *beta_out = beta_prime;
}

}  // namespace rtb
