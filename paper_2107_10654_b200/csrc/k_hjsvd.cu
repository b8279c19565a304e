// k_hjsvd.cu -- one-sided (Hestenes) Jacobi SVD of a tall matrix and the ridge leverage
// scores built on it, with the reference's exact semantics (ref svd.cpp:21-111,
// leverage.cpp:16-52): rotate the column pair (p, q) unless |gamma| <= 1e-14 ||A||_F^2 and
// |gamma| <= max(16, m, n) eps sqrt(alpha beta); sigma_j = ||w_j|| sorted non-increasing
// (stable); rank = #{sigma_j > max(m, n) eps sigma_max, sigma_j > 0}; scores
// l_i = sum_{k < rank} sigma_k^2 / (sigma_k^2 + lambda) u_ik^2.
//
// The rank cut is on singular values of A itself, not on eigenvalues of A^T A: a factor
// with kappa(A) between ~1e6.5 and ~1e13 keeps every direction, exactly as the reference
// does, where a Gram route would have to drop the directions below its eps * mu_max noise.
//
// Columns are rotated in parallel (round-robin ordering, one warp per pair, the three dot
// products as a fixed-order lane-strided sum + xor tree), instead of the reference's
// sequential row-cyclic order: singular values agree to high relative accuracy, and the
// scores are basis-invariant sums over the kept subspace.
//   k_hj_cta     n <= 32: the whole iteration in one CTA per matrix (columns in a global
//                column-major copy, V in shared memory); guarded by a skip flag so the
//                ALS sweep can enqueue it unconditionally behind the Cholesky route
//   k_hj_step    any n: one launch per round-robin step, one warp per pair (dense toolkit)
#include <algorithm>
#include <cfloat>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace rtb {

namespace {

// fixed-order warp sum
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// round-robin pair k of step r over n (even) indices
__device__ __forceinline__ void rr_pair(int k, int r, int n, int& p, int& q) {
  p = k == 0 ? 0 : 1 + (k - 1 + r) % (n - 1);
  q = 1 + (n - 2 - k + r) % (n - 1);
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

// One Jacobi rotation of columns p, q (length m, contiguous) by a warp; V (n x n, row-major,
// leading dimension ldv) gets the same right rotation. Returns true if it rotated.
__device__ bool hj_pair(double* __restrict__ W, long long ldw, double* __restrict__ V, int ldv,
                        int m, int n, int p, int q, double thr_abs, double tol_rel, int lane) {
  double* wp = W + (long long)p * ldw;
  double* wq = W + (long long)q * ldw;
  double alpha = 0.0, beta = 0.0, gamma = 0.0;
  for (int i = lane; i < m; i += 32) {
    const double a = wp[i], b = wq[i];
    alpha = fma(a, a, alpha);
    beta = fma(b, b, beta);
    gamma = fma(a, b, gamma);
  }
  alpha = warp_sum(alpha);
  beta = warp_sum(beta);
  gamma = warp_sum(gamma);
  if (fabs(gamma) <= thr_abs && fabs(gamma) <= tol_rel * sqrt(alpha * beta)) return false;
  const double zeta = (beta - alpha) / (2.0 * gamma);
  const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + t * t);
  const double s = c * t;
  for (int i = lane; i < m; i += 32) {
    const double a = wp[i], b = wq[i];
    wp[i] = c * a - s * b;
    wq[i] = s * a + c * b;
  }
  for (int i = lane; i < n; i += 32) {
    const double a = V[i * ldv + p], b = V[i * ldv + q];
    V[i * ldv + p] = c * a - s * b;
    V[i * ldv + q] = s * a + c * b;
  }
  return true;
}

// column norms, stable descending order, rank cut and the ridge scores of the rows
// (one CTA; n <= 32 columns; threads stride over the m rows)
__device__ void hj_finish(const double* __restrict__ W, long long ldw, int m, int n, double lambda,
                          double* __restrict__ scores, int* rank_out, double* sigma_out,
                          int* order_out) {
  __shared__ double nrm[64];
  __shared__ int ord[64];
  __shared__ double wgt[64];
  __shared__ int s_rank;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = warp; j < n; j += nw) {
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s = fma(W[(long long)j * ldw + i], W[(long long)j * ldw + i], s);
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < n; ++j) ord[j] = j;
    for (int a = 1; a < n; ++a) {  // stable insertion sort, non-increasing
      const int v = ord[a];
      int b = a - 1;
      while (b >= 0 && nrm[ord[b]] < nrm[v]) {
        ord[b + 1] = ord[b];
        --b;
      }
      ord[b + 1] = v;
    }
    const double smax = n ? nrm[ord[0]] : 0.0;
    const double cut = (double)(m > n ? m : n) * DBL_EPSILON * smax;
    int r = 0;
    while (r < n && nrm[ord[r]] > cut && nrm[ord[r]] > 0.0) ++r;
    s_rank = r;
    for (int k = 0; k < r; ++k) {
      const double s2 = nrm[ord[k]] * nrm[ord[k]];
      wgt[k] = s2 / (s2 + lambda);  // ref leverage.cpp:20-24
    }
    if (rank_out) *rank_out = r;
    if (sigma_out)
      for (int k = 0; k < n; ++k) sigma_out[k] = nrm[ord[k]];
    if (order_out)
      for (int k = 0; k < n; ++k) order_out[k] = ord[k];
  }
  __syncthreads();
  const int r = s_rank;
  if (!scores) return;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < r; ++k) {
      const int j = ord[k];
      // u_ik = w_ij / sigma_j (the reference divides first, then squares)
      const double u = W[(long long)j * ldw + i] / nrm[j];
      s += wgt[k] * u * u;
    }
    scores[i] = s;
  }
}

}  // namespace

// One CTA per matrix b (n <= 32 columns, m rows): A_b row-major (lda = n) copied into the
// column-major workspace W_b (m x n, ldw = m), Hestenes sweeps to convergence, then the
// ridge scores of its rows (scores_b, m entries) and *rank_b. Matrices with skip[b] != 0
// are left untouched (their scores come from the Cholesky route). status[b] = 3 if 100
// sweeps did not converge (ref svd.cpp:66).
__global__ void __launch_bounds__(512) k_hj_cta(const FactorSet fs, double* __restrict__ work,
                                                long long work_stride, double lambda,
                                                double* __restrict__ scores,
                                                const long long* __restrict__ score_off,
                                                int* __restrict__ ranks, const int* skip,
                                                int* status) {
  const int b = blockIdx.x;
  if (skip && skip[b]) return;
  const int m = fs.rows[b], n0 = fs.cols[b];
  const int n = n0 + (n0 & 1);  // even (a zero column never rotates)
  const double* A = fs.ptr[b];
  double* W = work + (long long)b * work_stride;
  __shared__ double V[32 * 33];
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double fro = 0.0;
  for (long long e = threadIdx.x; e < (long long)m * n; e += blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    const double v = j < n0 ? A[(long long)i * n0 + j] : 0.0;
    W[e] = v;
    fro = fma(v, v, fro);
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) V[(e / n) * 33 + e % n] = (e / n == e % n) ? 1.0 : 0.0;
  fro = block_sum<512>(fro, red);
  __shared__ double s_fro;
  if (threadIdx.x == 0) s_fro = fro;
  __syncthreads();
  const double thr = 1e-14 * s_fro;
  const double tol_rel = (double)(m > n0 ? (m > 16 ? m : 16) : (n0 > 16 ? n0 : 16)) * DBL_EPSILON;
  int st = 3;
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < n - 1; ++r) {
      int any = 0;
      if (warp < n / 2) {
        int p, q;
        rr_pair(warp, r, n, p, q);
        any = hj_pair(W, m, V, 33, m, n, p, q, thr, tol_rel, lane) ? 1 : 0;
      }
      rotated |= __syncthreads_or(any);
    }
    if (!rotated) {
      st = 0;
      break;
    }
  }
  if (threadIdx.x == 0 && status) status[b] = st;
  hj_finish(W, m, m, n0, lambda, scores + score_off[b], ranks + b, nullptr, nullptr);
}

namespace {
__global__ void k_hj_load(const double* __restrict__ A, int m, int n0, int n, double* __restrict__ W,
                          double* __restrict__ V) {
  const long long tot = (long long)m * n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    W[e] = j < n0 ? A[(long long)i * n0 + j] : 0.0;
  }
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x)
    V[e] = (e / n == e % n) ? 1.0 : 0.0;
}

__global__ void k_hj_fro(const double* __restrict__ W, long long tot, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long e = threadIdx.x; e < tot; e += blockDim.x) s = fma(W[e], W[e], s);
  s = block_sum<1024>(s, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_hj_step(double* __restrict__ W, double* __restrict__ V, int m, int n0, int n,
                          int r, const double* fro2, int* rotated) {
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (k >= n / 2) return;
  int p, q;
  rr_pair(k, r, n, p, q);
  const double tol_rel = (double)(m > n0 ? (m > 16 ? m : 16) : (n0 > 16 ? n0 : 16)) * DBL_EPSILON;
  if (hj_pair(W, m, V, n, m, n, p, q, 1e-14 * *fro2, tol_rel, lane) && lane == 0)
    atomicExch(rotated, 1);
}

// column norms (one warp per column)
__global__ void k_hj_norms(const double* __restrict__ W, int m, int n0, double* __restrict__ nrm) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (j >= n0) return;
  double s = 0.0;
  for (int i = lane; i < m; i += 32) s = fma(W[(long long)j * m + i], W[(long long)j * m + i], s);
  s = warp_sum(s);
  if (lane == 0) nrm[j] = sqrt(s);
}

// scores of the rows from the kept columns (ord[0..rank), weights wgt[k] on w_ij^2)
__global__ void k_hj_scores(const double* __restrict__ W, int m, const double* __restrict__ nrm,
                            const int* __restrict__ ord, const double* __restrict__ wgt, int rank,
                            double* __restrict__ scores) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int k = 0; k < rank; ++k) {
    const int j = ord[k];
    const double u = W[(long long)j * m + i] / nrm[j];
    s += wgt[k] * u * u;
  }
  scores[i] = s;
}
}  // namespace

namespace {
struct HjLayout {
  double *W, *V, *nrm, *fro2, *wgt;
  int *flag, *ord;
};
HjLayout hj_layout(long long m, int n, void* work) {
  HjLayout l;
  char* p = static_cast<char*>(work);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  l.W = reinterpret_cast<double*>(take((size_t)m * n * 8));
  l.V = reinterpret_cast<double*>(take((size_t)n * n * 8));
  l.nrm = reinterpret_cast<double*>(take((size_t)n * 8));
  l.wgt = reinterpret_cast<double*>(take((size_t)n * 8));
  l.fro2 = reinterpret_cast<double*>(take(8));
  l.flag = reinterpret_cast<int*>(take(8));
  l.ord = reinterpret_cast<int*>(take((size_t)n * 4));
  return l;
}

__global__ void k_hj_load_t(const double* __restrict__ A, int rows, int cols, int n,
                            double* __restrict__ W, double* __restrict__ V) {
  // W = the columns of A^T (A: rows x cols row-major): column j of A^T = row j of A
  const long long tot = (long long)cols * n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / cols), i = (int)(e % cols);
    W[e] = j < rows ? A[(long long)j * cols + i] : 0.0;
  }
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x)
    V[e] = (e / n == e % n) ? 1.0 : 0.0;
}

// wide A: u_ik = V[i][ord_k] (ref svd.cpp:122-129: the bases of the transpose swapped)
__global__ void k_hj_scores_v(const double* __restrict__ V, int n, const int* __restrict__ ord,
                              const double* __restrict__ wgt, int rank, int rows,
                              double* __restrict__ scores) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double s = 0.0;
  for (int k = 0; k < rank; ++k) {
    const double u = V[(long long)i * n + ord[k]];
    s += wgt[k] * u * u;
  }
  scores[i] = s;
}
}  // namespace

size_t hj_work_bytes(long long rows, int cols) {
  const long long m = std::max<long long>(rows, cols), n0 = std::min<long long>(rows, cols);
  const long long n = n0 + (n0 & 1);
  return (size_t)m * n * 8 + (size_t)n * n * 8 + 4 * (size_t)n * 8 + 8 * 256;
}

// Ridge scores of the rows of A (rows x cols, device, row-major) for any shape (dense
// toolkit, ref leverage.cpp:39-52): the one-sided Jacobi SVD of A (tall) or of A^T (wide,
// ref svd.cpp:115-129), one launch per round-robin step and one host check per sweep, then
// the reference's rank cut and scores; *rank = numerical rank.
void hj_ridge_scores(const double* A, long long rows, int cols, double lambda, double* scores,
                     int* rank, void* work, cudaStream_t st) {
  const bool wide = rows < cols;
  const long long m = wide ? cols : rows;  // length of the Jacobi columns
  const int n0 = wide ? (int)rows : cols;  // number of Jacobi columns
  const int n = n0 + (n0 & 1);
  HjLayout l = hj_layout(m, n, work);
  const unsigned g = (unsigned)std::min<long long>(ceil_div<long long>(m * n, 256), 8 * kNumSMs);
  if (wide) k_hj_load_t<<<g, 256, 0, st>>>(A, (int)rows, cols, n, l.W, l.V);
  else k_hj_load<<<g, 256, 0, st>>>(A, (int)m, n0, n, l.W, l.V);
  RTB_LAUNCH_CHECK();
  k_hj_fro<<<1, 1024, 0, st>>>(l.W, m * n, l.fro2);
  RTB_LAUNCH_CHECK();
  bool ok = false;
  for (int sweep = 0; sweep < 100; ++sweep) {
    RTB_CUDA(cudaMemsetAsync(l.flag, 0, 4, st));
    for (int r = 0; r < n - 1; ++r) {
      k_hj_step<<<ceil_div(n / 2 * 32, 256), 256, 0, st>>>(l.W, l.V, (int)m, n0, n, r, l.fro2,
                                                         l.flag);
      RTB_LAUNCH_CHECK();
    }
    int h = 0;
    RTB_CUDA(cudaMemcpyAsync(&h, l.flag, 4, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaStreamSynchronize(st));
    if (!h) {
      ok = true;
      break;
    }
  }
  if (!ok) throw Error(3, "compact_svd: Jacobi sweeps did not converge");
  k_hj_norms<<<ceil_div(n0 * 32, 256), 256, 0, st>>>(l.W, (int)m, n0, l.nrm);
  RTB_LAUNCH_CHECK();
  std::vector<double> hn(n0);
  RTB_CUDA(cudaMemcpyAsync(hn.data(), l.nrm, (size_t)n0 * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  std::vector<int> ord(n0);
  for (int j = 0; j < n0; ++j) ord[j] = j;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return hn[x] > hn[y]; });
  const double smax = n0 ? hn[ord[0]] : 0.0;
  const double cut = (double)std::max<long long>(m, n0) * DBL_EPSILON * smax;
  int r = 0;
  while (r < n0 && hn[ord[r]] > cut && hn[ord[r]] > 0.0) ++r;
  std::vector<double> wgt(std::max(r, 1));
  for (int k = 0; k < r; ++k) {
    const double s2 = hn[ord[k]] * hn[ord[k]];
    wgt[k] = s2 / (s2 + lambda);
  }
  RTB_CUDA(cudaMemcpyAsync(l.ord, ord.data(), (size_t)n0 * 4, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(l.wgt, wgt.data(), (size_t)std::max(r, 1) * 8, cudaMemcpyHostToDevice, st));
  if (wide)
    k_hj_scores_v<<<(unsigned)ceil_div<long long>(rows, 256), 256, 0, st>>>(l.V, n, l.ord, l.wgt,
                                                                        r, (int)rows, scores);
  else
    k_hj_scores<<<(unsigned)ceil_div<long long>(m, 256), 256, 0, st>>>(l.W, (int)m, l.nrm, l.ord,
                                                                    l.wgt, r, scores);
  RTB_LAUNCH_CHECK();
  RTB_CUDA(cudaStreamSynchronize(st));  // host vectors above go out of scope
  *rank = r;
}

}  // namespace rtb
