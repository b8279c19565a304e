// k_small.cu -- per-mode small dense linear algebra on the GPU.
//
//  * k_factor_gram      A_n^T A_n for every mode (R_n x R_n), deterministic.
//  * k_sym_eigen        batched cyclic Jacobi eigensolver, one CTA per matrix
//                       (n <= 64), round-robin parallel rotations.
//  * k_leverage_rows    classical leverage scores l_i = sum_k (a_i.v_k)^2/mu_k
//                       over the numerically nonzero eigenpairs of A^T A
//                       (ref leverage.cpp:16-37 at lambda = 0, kronecker.cpp:22).
//  * k_score_cdf        sequential left-to-right prefix sums, the same rounding
//                       as the reference CDF (ref kronecker.cpp:25-33).
//  * k_sym_pinv         pinv of a symmetric matrix from its eigenpairs with the
//                       reference rank cutoff n*eps*|mu|_max (ref svd.cpp:92-97,
//                       linalg.cpp:8-26).
//  * k_rows_times_small out = M * P for an I x R matrix M and R x R matrix P.
#include "common.cuh"
#include "kernels.h"

#include <cfloat>

namespace rtb {

// ---------------------------------------------------------------------------
// A^T A for each mode. grid = (entries, modes); each block reduces one (p,q)
// entry over all rows in a fixed order (per-thread strided partial sums, then a
// fixed-shape tree), so results are bitwise reproducible run to run.
__global__ void k_factor_gram(const FactorSet fs, double* grams /* [mode][Rmax*Rmax] */,
                              int r_max) {
  const int mode = blockIdx.y;
  const int R = fs.cols[mode];
  const int I = fs.rows[mode];
  const int e = blockIdx.x;
  const int p = e / r_max, q = e % r_max;
  __shared__ double red[32];
  if (p >= R || q >= R || q < p) return;
  const double* A = fs.ptr[mode];
  double acc = 0.0;
  for (int i = threadIdx.x; i < I; i += blockDim.x) acc += A[(size_t)i * R + p] * A[(size_t)i * R + q];
  const double s = block_sum<256>(acc, red);
  if (threadIdx.x == 0) {
    grams[(size_t)mode * r_max * r_max + p * R + q] = s;
    grams[(size_t)mode * r_max * r_max + q * R + p] = s;
  }
}

// ---------------------------------------------------------------------------
// Batched symmetric eigensolver. Matrix b is n_b x n_b at in + b*stride
// (row-major, dense n x n with leading dimension n). Outputs, per matrix:
//   evals[b*stride_v ...]   eigenvalues sorted non-increasing (stable)
//   evecs[b*stride ...]     n x n, column k pairs with evals[k]
//   status[b]               0 ok, 3 no convergence
__global__ void k_sym_eigen(const double* in, const int* ns, int stride, double* evals,
                            double* evecs, int* status) {
  extern __shared__ double sm[];
  const int b = blockIdx.x;
  const int n = ns[b];
  const int np = n + (n & 1);  // padded to even for the round-robin schedule
  double* A = sm;               // np x np
  double* V = A + np * np;      // np x np
  double* cs = V + np * np;     // 2 * np/2 rotation coefficients
  int* pair = reinterpret_cast<int*>(cs + np);  // np entries: partner schedule
  __shared__ int rotated;
  const double* src = in + (size_t)b * stride;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    const int i = e / np, j = e % np;
    A[e] = (i < n && j < n) ? src[i * n + j] : 0.0;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  __shared__ double red[32];
  double fro = 0.0;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) fro += A[e] * A[e];
  fro = block_sum<128>(fro, red);
  __shared__ double s_fro;
  if (threadIdx.x == 0) s_fro = fro;
  __syncthreads();
  fro = s_fro;
  const double tiny = 1e-300 + 1e-30 * fro * DBL_EPSILON;
  int st = 3;
  for (int sweep = 0; sweep < 100; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < np - 1; ++round) {
      // round-robin: position 0 fixed, others rotate
      if (threadIdx.x < np / 2) {
        const int k = threadIdx.x;
        auto at = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + round) % (np - 1); };
        int p = at(k), q = at(np - 1 - k);
        if (p > q) { int t = p; p = q; q = t; }
        pair[2 * k] = p;
        pair[2 * k + 1] = q;
        const double apq = A[p * np + q];
        const double app = A[p * np + p], aqq = A[q * np + q];
        double c = 1.0, s = 0.0;
        // rotate unless already negligible relative to the diagonal (high
        // relative accuracy criterion) or padding
        if (q < n && fabs(apq) > tiny &&
            fabs(apq) > DBL_EPSILON * 0.5 * sqrt(fabs(app) * fabs(aqq))) {
          const double theta = (aqq - app) / (2.0 * apq);
          const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = c * t;
          rotated = 1;
        }
        cs[2 * k] = c;
        cs[2 * k + 1] = s;
      }
      __syncthreads();
      // A <- A J (columns), V <- V J
      for (int e = threadIdx.x; e < (np / 2) * np; e += blockDim.x) {
        const int k = e / np, row = e % np;
        const int p = pair[2 * k], q = pair[2 * k + 1];
        const double c = cs[2 * k], s = cs[2 * k + 1];
        if (s == 0.0) continue;
        const double ap = A[row * np + p], aq = A[row * np + q];
        A[row * np + p] = c * ap - s * aq;
        A[row * np + q] = s * ap + c * aq;
        const double vp = V[row * np + p], vq = V[row * np + q];
        V[row * np + p] = c * vp - s * vq;
        V[row * np + q] = s * vp + c * vq;
      }
      __syncthreads();
      // A <- J^T A (rows)
      for (int e = threadIdx.x; e < (np / 2) * np; e += blockDim.x) {
        const int k = e / np, col = e % np;
        const int p = pair[2 * k], q = pair[2 * k + 1];
        const double c = cs[2 * k], s = cs[2 * k + 1];
        if (s == 0.0) continue;
        const double ap = A[p * np + col], aq = A[q * np + col];
        A[p * np + col] = c * ap - s * aq;
        A[q * np + col] = s * ap + c * aq;
      }
      __syncthreads();
    }
    if (!rotated) {
      st = 0;
      break;
    }
    __syncthreads();
  }
  // stable sort by eigenvalue, non-increasing
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double mk = A[k * np + k];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double mj = A[j * np + j];
      if (mj > mk || (mj == mk && j < k)) ++rank;
    }
    evals[(size_t)b * stride + rank] = mk;
    for (int i = 0; i < n; ++i) evecs[(size_t)b * stride * 1 + (size_t)i * n + rank] = V[i * np + k];
  }
  if (threadIdx.x == 0) status[b] = st;
}

// ---------------------------------------------------------------------------
// Leverage scores of every row of every factor from the eigenpairs of A^T A.
// rank cutoff (Gram form): mu_k > max(I,R) * eps * mu_max  and mu_k > 0.
// grid = (ceil(max I / 128), modes), block 128.
__global__ void k_leverage_rows(const FactorSet fs, const double* evals, const double* evecs,
                                int stride, double lambda, double* scores,
                                const long long* score_off, int* ranks) {
  const int mode = blockIdx.y;
  const int R = fs.cols[mode], I = fs.rows[mode];
  const double* mu = evals + (size_t)mode * stride;
  const double* V = evecs + (size_t)mode * stride;
  const double cut = (double)(I > R ? I : R) * DBL_EPSILON * mu[0];
  int rank = 0;
  while (rank < R && mu[rank] > cut && mu[rank] > 0.0) ++rank;
  if (blockIdx.x == 0 && threadIdx.x == 0) ranks[mode] = rank;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I) return;
  const double* a = fs.ptr[mode] + (size_t)i * R;
  double s = 0.0;
  for (int k = 0; k < rank; ++k) {
    double proj = 0.0;
    for (int j = 0; j < R; ++j) proj += a[j] * V[j * R + k];
    s += proj * proj / (mu[k] + lambda);  // = w_k u_ik^2, w_k = s^2/(s^2+lambda)
  }
  scores[score_off[mode] + i] = s;
}

// Left-to-right CDF per mode, one warp per mode: each lane loads 32 scores and
// every lane adds them in index order (shuffle broadcast), so the running sum
// is the same sequence of roundings as the reference's serial loop.
__global__ void k_score_cdf(const double* scores, const long long* off, const int* rows,
                            int order, double* cdf, double* sums) {
  const int mode = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (mode >= order) return;
  const double* s = scores + off[mode];
  double* c = cdf + off[mode];
  const int n = rows[mode];
  double running = 0.0;
  for (int base = 0; base < n; base += 32) {
    const double v = base + lane < n ? s[base + lane] : 0.0;
    double mine = 0.0;
    const int cnt = min(32, n - base);
    for (int k = 0; k < cnt; ++k) {
      running = __dadd_rn(running, __shfl_sync(0xffffffffu, v, k));
      if (lane == k) mine = running;
    }
    if (base + lane < n) c[base + lane] = mine;
  }
  if (lane == 0) sums[mode] = running;
}

// ---------------------------------------------------------------------------
// Symmetric pseudoinverse from eigenpairs: P = V diag(1/mu_k) V^T over
// |mu_k| > n*eps*max|mu| (singular values of a symmetric matrix are |mu|).
// grid = batch, block = 256. P stored row-major n x n at out + b*stride.
__global__ void k_sym_pinv(const double* evals, const double* evecs, const int* ns, int stride,
                           double* out, int* ranks) {
  const int b = blockIdx.x;
  const int n = ns[b];
  const double* mu = evals + (size_t)b * stride;
  const double* V = evecs + (size_t)b * stride;
  double amax = 0.0;
  for (int k = 0; k < n; ++k) amax = fmax(amax, fabs(mu[k]));
  const double cut = (double)n * DBL_EPSILON * amax;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    double s = 0.0;
    for (int k = 0; k < n; ++k) {
      const double m = mu[k];
      if (!(fabs(m) > cut) || m == 0.0) continue;
      s += V[i * n + k] * (V[j * n + k] / m);
    }
    out[(size_t)b * stride + e] = s;
  }
  if (threadIdx.x == 0 && ranks) {
    int r = 0;
    for (int k = 0; k < n; ++k)
      if (fabs(mu[k]) > cut && mu[k] != 0.0) ++r;
    ranks[b] = r;
  }
}

// out (I x R) = M (I x R) * P (R x R); one thread per output element.
__global__ void k_rows_times_small(const double* M, const double* P, int I, int R, double* out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)I * R) return;
  const int i = (int)(e / R), r = (int)(e % R);
  double s = 0.0;
  for (int k = 0; k < R; ++k) s += M[(size_t)i * R + k] * P[k * R + r];
  out[e] = s;
}

}  // namespace rtb
