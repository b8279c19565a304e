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

#include <algorithm>

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
  const int ld = np + 1;       // odd stride: column accesses hit distinct banks
  double* A = sm;               // np x ld
  double* V = A + np * ld;      // np x ld
  double* cs = V + np * ld;     // 2 * np/2 rotation coefficients
  int* pair = reinterpret_cast<int*>(cs + np);  // np entries: partner schedule
  __shared__ int rotated;
  const double* src = in + (size_t)b * stride;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    const int i = e / np, j = e % np;
    A[i * ld + j] = (i < n && j < n) ? src[i * n + j] : 0.0;
    V[i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  __shared__ double red[32];
  double fro = 0.0;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) fro += A[(e / np) * ld + e % np] * A[(e / np) * ld + e % np];
  fro = block_sum<128>(fro, red);
  __shared__ double s_fro;
  if (threadIdx.x == 0) s_fro = fro;
  __syncthreads();
  fro = s_fro;
  const double tiny = 1e-300;
  const double tol_abs = (double)n * DBL_EPSILON * sqrt(fro);
  int st = 3;
  for (int sweep = 0; sweep < 60; ++sweep) {
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
        const double apq = A[p * ld + q];
        const double app = A[p * ld + p], aqq = A[q * ld + q];
        double c = 1.0, s = 0.0;
        // rotate unless already negligible relative to the diagonal (high
        // relative accuracy criterion) or padding
        // absolute threshold n*eps*||A||_F (the rotated pair is zeroed explicitly
        // below): a relative test never settles when the diagonal spans many
        // orders of magnitude, since rotation rounding is ~eps*max|a_ii|
        if (q < n && fabs(apq) > tiny && fabs(apq) > tol_abs) {
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
        const double ap = A[row * ld + p], aq = A[row * ld + q];
        A[row * ld + p] = c * ap - s * aq;
        A[row * ld + q] = s * ap + c * aq;
        const double vp = V[row * ld + p], vq = V[row * ld + q];
        V[row * ld + p] = c * vp - s * vq;
        V[row * ld + q] = s * vp + c * vq;
      }
      __syncthreads();
      // A <- J^T A (rows)
      for (int e = threadIdx.x; e < (np / 2) * np; e += blockDim.x) {
        const int k = e / np, col = e % np;
        const int p = pair[2 * k], q = pair[2 * k + 1];
        const double c = cs[2 * k], s = cs[2 * k + 1];
        if (s == 0.0) continue;
        const double ap = A[p * ld + col], aq = A[q * ld + col];
        A[p * ld + col] = c * ap - s * aq;
        A[q * ld + col] = s * ap + c * aq;
      }
      __syncthreads();
      if (threadIdx.x < np / 2 && cs[2 * threadIdx.x + 1] != 0.0) {
        const int p = pair[2 * threadIdx.x], q = pair[2 * threadIdx.x + 1];
        A[p * ld + q] = 0.0;
        A[q * ld + p] = 0.0;
      }
      __syncthreads();
    }
    if (!rotated) {
#ifdef RTB_EIG_SWEEP_DEBUG
      st = -(sweep + 1);
#else
      st = 0;
#endif
      break;
    }
    __syncthreads();
  }
  // stable sort by eigenvalue, non-increasing
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double mk = A[k * ld + k];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double mj = A[j * ld + j];
      if (mj > mk || (mj == mk && j < k)) ++rank;
    }
    evals[(size_t)b * stride + rank] = mk;
    for (int i = 0; i < n; ++i) evecs[(size_t)b * stride * 1 + (size_t)i * n + rank] = V[i * ld + k];
  }
  if (threadIdx.x == 0) status[b] = st;
}

// ---------------------------------------------------------------------------
// Warp-per-matrix variant for n <= 32 (the factor Grams and the R_n x R_n
// factor-update systems): same rotations, only __syncwarp between phases.
__global__ void k_sym_eigen_warp(const double* in, const int* ns, int stride, double* evals,
                                 double* evecs, int* status, int nmat, const int* skip) {
  extern __shared__ double smw[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + wib;
  if (b >= nmat) return;
  if (skip && skip[b]) {  // a Cholesky already succeeded for this matrix
    if (lane == 0) status[b] = 0;
    return;
  }
  const int n = ns[b];
  const int np = n + (n & 1);
  const int ld = np + 1;  // odd stride: column accesses hit distinct banks
  double* A = smw + wib * (2 * 32 * 33 + 64);
  double* V = A + 32 * 33;
  double* cs = V + 32 * 33;
  int* pair = reinterpret_cast<int*>(cs + 32);
  const double* src = in + (size_t)b * stride;
  double fro = 0.0;
  for (int e = lane; e < np * np; e += 32) {
    const int i = e / np, j = e % np;
    const double v = (i < n && j < n) ? src[i * n + j] : 0.0;
    A[i * ld + j] = v;
    V[i * ld + j] = (i == j) ? 1.0 : 0.0;
    fro += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  const double tol_abs = (double)n * DBL_EPSILON * sqrt(fro);
  __syncwarp();
  int st = 3;
  // round-robin pairing: position 0 fixed, the others rotate by one per round
  int pos_p = 0, pos_q = 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < np - 1; ++round) {
      if (lane < np / 2) {
        // positions lane and np-1-lane; rotation offset without a division
        pos_p = lane == 0 ? 0 : 1 + ((lane - 1 + round) % (np - 1));
        pos_q = 1 + ((np - 2 - lane + round) % (np - 1));
        int p = min(pos_p, pos_q), q = max(pos_p, pos_q);
        pair[2 * lane] = p;
        pair[2 * lane + 1] = q;
        const double apq = A[p * ld + q], app = A[p * ld + p], aqq = A[q * ld + q];
        double c = 1.0, s = 0.0;
        if (q < n && fabs(apq) > 1e-300 && fabs(apq) > tol_abs) {
          // t = sign(theta) / (|theta| + sqrt(1 + theta^2)), theta = (aqq-app)/(2 apq)
          const double diff = aqq - app;
          const double den = fabs(diff) + sqrt(diff * diff + 4.0 * apq * apq);
          double t = 2.0 * apq / den;
          if (diff < 0.0) t = -t;
          c = rsqrt(1.0 + t * t);
          s = c * t;
        }
        cs[2 * lane] = c;
        cs[2 * lane + 1] = s;
      }
      rotated |= __any_sync(0xffffffffu, lane < np / 2 && cs[2 * lane + 1] != 0.0);
      __syncwarp();
      if (lane < np) {  // columns p, q of A and V: lane = row
        for (int k = 0; k < np / 2; ++k) {
          const double c = cs[2 * k], s = cs[2 * k + 1];
          if (s == 0.0) continue;
          const int p = pair[2 * k], q = pair[2 * k + 1];
          const double ap = A[lane * ld + p], aq = A[lane * ld + q];
          A[lane * ld + p] = c * ap - s * aq;
          A[lane * ld + q] = s * ap + c * aq;
          const double vp = V[lane * ld + p], vq = V[lane * ld + q];
          V[lane * ld + p] = c * vp - s * vq;
          V[lane * ld + q] = s * vp + c * vq;
        }
      }
      __syncwarp();
      if (lane < np) {  // rows p, q of A: lane = column
        for (int k = 0; k < np / 2; ++k) {
          const double c = cs[2 * k], s = cs[2 * k + 1];
          if (s == 0.0) continue;
          const int p = pair[2 * k], q = pair[2 * k + 1];
          const double ap = A[p * ld + lane], aq = A[q * ld + lane];
          A[p * ld + lane] = c * ap - s * aq;
          A[q * ld + lane] = s * ap + c * aq;
        }
      }
      __syncwarp();
      if (lane < np / 2 && cs[2 * lane + 1] != 0.0) {
        const int p = pair[2 * lane], q = pair[2 * lane + 1];
        A[p * ld + q] = 0.0;
        A[q * ld + p] = 0.0;
      }
      __syncwarp();
    }
    if (!rotated) {
#ifdef RTB_EIG_SWEEP_DEBUG
      st = -(sweep + 1);
#else
      st = 0;
#endif
      break;
    }
  }
  for (int k = lane; k < n; k += 32) {
    const double mk = A[k * ld + k];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double mj = A[j * ld + j];
      if (mj > mk || (mj == mk && j < k)) ++rank;
    }
    evals[(size_t)b * stride + rank] = mk;
    for (int i = 0; i < n; ++i) evecs[(size_t)b * stride + (size_t)i * n + rank] = V[i * ld + k];
  }
  if (lane == 0) status[b] = st;
}

// ---------------------------------------------------------------------------
// CTA-per-matrix parallel Jacobi for n <= 32: thread (i, j) owns A[i][j] and
// V[i][j]; every round applies the n/2 disjoint rotations of the round-robin
// tournament at once (they commute), A' = J^T A J and V' = V J, each thread
// reading the 4 (resp. 2) entries it needs from the previous buffer. Same
// rotation formula, absolute threshold and output order as k_sym_eigen_warp,
// ~2 barriers per round instead of a serial per-pair loop.
__global__ void __launch_bounds__(1024) k_sym_eigen_cta(const double* in, const int* ns, int stride,
                                                        double* evals, double* evecs, int* status,
                                                        const int* skip) {
  __shared__ double Ab[2][32][33];
  __shared__ double Vb[2][32][33];
  __shared__ double rc[32], rs[32];
  __shared__ int partner[32];
  __shared__ double red[32];
  const int b = blockIdx.x;
  if (skip && skip[b]) {
    if (threadIdx.x == 0) status[b] = 0;
    return;
  }
  const int n = ns[b];
  const int np = n + (n & 1);
  const int tid = threadIdx.x;
  const int i = tid / 32, j = tid % 32;
  const bool act = i < np && j < np;
  const double* src = in + (size_t)b * stride;
  double fro = 0.0;
  if (act) {
    const double v = (i < n && j < n) ? src[i * n + j] : 0.0;
    Ab[0][i][j] = v;
    Vb[0][i][j] = (i == j) ? 1.0 : 0.0;
    fro = v * v;
  }
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  if ((tid & 31) == 0) red[tid >> 5] = fro;
  __syncthreads();
  if (tid < 32) {
    double t = tid < (int)(blockDim.x >> 5) ? red[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (tid == 0) red[0] = t;
  }
  __syncthreads();
  const double tol_abs = (double)n * DBL_EPSILON * sqrt(red[0]);
  int cur = 0;
  int st = 3;
  for (int sweep = 0; sweep < 60; ++sweep) {
    for (int round = 0; round < np - 1; ++round) {
      if (tid < np / 2) {
        const int k = tid;
        const int pp = k == 0 ? 0 : 1 + ((k - 1 + round) % (np - 1));
        const int qq = 1 + ((np - 2 - k + round) % (np - 1));
        const int p = min(pp, qq), q = max(pp, qq);
        const double apq = Ab[cur][p][q], app = Ab[cur][p][p], aqq = Ab[cur][q][q];
        double c = 1.0, sn = 0.0;
        if (q < n && fabs(apq) > 1e-300 && fabs(apq) > tol_abs) {
          const double diff = aqq - app;
          const double den = fabs(diff) + sqrt(diff * diff + 4.0 * apq * apq);
          double t = 2.0 * apq / den;
          if (diff < 0.0) t = -t;
          c = rsqrt(1.0 + t * t);
          sn = c * t;
        }
        partner[p] = q;
        partner[q] = p;
        rc[p] = c;
        rc[q] = c;
        rs[p] = -sn;  // sigma_p s: column p' = c col_p - s col_q
        rs[q] = sn;   // sigma_q s: column q' = c col_q + s col_p
      }
      __syncthreads();
      if (act) {
        const int yi = partner[i], yj = partner[j];
        const double ci = rc[i], si = rs[i], cj = rc[j], sj = rs[j];
        const double (*A)[33] = Ab[cur];
        double v = ci * cj * A[i][j] + ci * sj * A[i][yj] + si * cj * A[yi][j] + si * sj * A[yi][yj];
        if (si != 0.0 && j == yi) v = 0.0;  // the annihilated pair
        Ab[cur ^ 1][i][j] = v;
        Vb[cur ^ 1][i][j] = cj * Vb[cur][i][j] + sj * Vb[cur][i][yj];
      }
      cur ^= 1;
      __syncthreads();
    }
    // converged when no rotation fired in the whole sweep
    int any = 0;
    if (act && i < j && j < n) any = fabs(Ab[cur][i][j]) > tol_abs && fabs(Ab[cur][i][j]) > 1e-300;
    if (!__syncthreads_or(any)) {
      st = 0;
      break;
    }
  }
  if (tid < n) {
    const int k = tid;
    const double mk = Ab[cur][k][k];
    int rank = 0;
    for (int jj = 0; jj < n; ++jj) {
      const double mj = Ab[cur][jj][jj];
      if (mj > mk || (mj == mk && jj < k)) ++rank;
    }
    evals[(size_t)b * stride + rank] = mk;
    for (int ii = 0; ii < n; ++ii) evecs[(size_t)b * stride + (size_t)ii * n + rank] = Vb[cur][ii][k];
  }
  if (tid == 0) status[b] = st;
}

// ---------------------------------------------------------------------------
// Batched small SPD factorization, one warp per matrix (n <= 32): Cholesky
// with row r in lane r's registers (column broadcasts through shuffles), then
// Linv (column per lane). ok[b] = 1 unless a pivot falls below
// tolrel * max diag (the caller then takes the eigen/pinv path for that
// matrix). Optionally also writes P = M^-1 = Linv^T Linv.
// Loops run to 32 with compile-time indices so row[] / x[] stay in registers;
// the matrix is padded with the identity beyond n.
template <int NM>
__global__ void __launch_bounds__(128) k_spd_small(const double* in, const int* ns, int stride,
                                                   double tolrel, double* linv, double* pinv,
                                                   int* ok, int nmat) {
  __shared__ double xs[4][32][33];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 4 + wib;
  if (b >= nmat) return;
  const int n = ns[b];
  const double* src = in + (size_t)b * stride;
  constexpr unsigned FULL = 0xffffffffu;
  double row[NM];
#pragma unroll
  for (int q = 0; q < NM; ++q)
    row[q] = (lane < n && q < n) ? src[lane * n + q] : (lane == q ? 1.0 : 0.0);
  double dmax = 0.0;
#pragma unroll
  for (int q = 0; q < NM; ++q)
    if (q == lane && lane < n) dmax = fabs(row[q]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(FULL, dmax, o));
  const double tol = tolrel * dmax;
  bool bad = false;
  double invd = 1.0;
#pragma unroll
  for (int c = 0; c < NM; ++c) {
    const double piv = __shfl_sync(FULL, row[c], c);
    bad |= (c < n) && !(piv > tol);
    const double rs = rsqrt(piv);
    row[c] = (lane == c) ? piv * rs : ((lane > c) ? row[c] * rs : row[c]);
    invd = (lane == c) ? rs : invd;
#pragma unroll
    for (int l = 1; l < NM; ++l) {
      if (l > c) {
        const double lc = __shfl_sync(FULL, row[c], l);
        row[l] = (lane >= l) ? row[l] - row[c] * lc : row[l];
      }
    }
  }
  bad = __any_sync(FULL, bad);
  if (lane == 0) ok[b] = bad ? 0 : 1;
  if (bad) return;
  // Linv: lane = column
  double x[NM];
#pragma unroll
  for (int rr = 0; rr < NM; ++rr) {
    double s0 = (rr == lane) ? 1.0 : 0.0, s1 = 0.0;
#pragma unroll
    for (int l = 0; l < NM - 1; ++l) {
      if (l < rr) {
        const double lv = __shfl_sync(FULL, row[l], rr);
        if (l & 1) s1 -= lv * x[l];
        else s0 -= lv * x[l];
      }
    }
    const double dinv = __shfl_sync(FULL, invd, rr);
    x[rr] = (rr >= lane) ? (s0 + s1) * dinv : 0.0;
  }
  double* lo = linv + (size_t)b * stride;
  if (lane < n) {
#pragma unroll
    for (int q = 0; q < NM; ++q)
      if (q < n) lo[q * n + lane] = x[q];  // Linv[q][lane]
  }
  if (pinv) {
    // P[i][j] = sum_k Linv[k][i] Linv[k][j]; lane j holds column j (x[k] = Linv[k][j])
#pragma unroll
    for (int q = 0; q < NM; ++q) xs[wib][q][lane] = x[q];
    __syncwarp();
    double* po = pinv + (size_t)b * stride;
    if (lane < n) {
      for (int i = 0; i < n; ++i) {
        double sacc = 0.0;
        for (int k = max(i, lane); k < n; ++k) sacc += xs[wib][k][i] * xs[wib][k][lane];
        po[i * n + lane] = sacc;
      }
    }
  }
}

// Leverage scores from a successful Cholesky: l_i = ||Linv a_i||^2.
// grid = (ceil(max I / 128), modes); modes with ok == 0 are left to
// k_leverage_rows (eigen path).
// Linv is staged in shared memory and the factor row held in registers (compile-time bounds):
// the previous form read both from global memory inside the dependent loops (one L2 latency
// per multiply-add, ~20 us at C2). Same arithmetic, same order.
template <int RM>
__global__ void __launch_bounds__(128) k_leverage_chol_t(const FactorSet fs, const double* linv,
                                                         int stride, const int* ok, double* scores,
                                                         const long long* score_off, int* ranks) {
  __shared__ double Ls[RM * RM];
  const int mode = blockIdx.y;
  if (!ok[mode]) return;
  const int R = fs.cols[mode], I = fs.rows[mode];
  if (blockIdx.x == 0 && threadIdx.x == 0) ranks[mode] = R;
  const double* L = linv + (size_t)mode * stride;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Ls[e] = L[e];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I) return;
  const double* ap = fs.ptr[mode] + (size_t)i * R;
  double a[RM];
#pragma unroll
  for (int k = 0; k < RM; ++k) a[k] = k < R ? ap[k] : 0.0;
  double s = 0.0;
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    if (r < R) {
      double y = 0.0;
#pragma unroll
      for (int k = 0; k < RM; ++k)
        if (k <= r) y += Ls[r * R + k] * a[k];
      s += y * y;
    }
  }
  scores[score_off[mode] + i] = s;
}

void leverage_chol(const FactorSet& fs, const double* linv, int stride, const int* ok,
                   double* scores, const long long* score_off, int* ranks, int max_rows,
                   int nmodes, int rmax, cudaStream_t st) {
  const dim3 grid(ceil_div(max_rows, 128), nmodes);
  if (rmax <= 8)
    k_leverage_chol_t<8><<<grid, 128, 0, st>>>(fs, linv, stride, ok, scores, score_off, ranks);
  else if (rmax <= 16)
    k_leverage_chol_t<16><<<grid, 128, 0, st>>>(fs, linv, stride, ok, scores, score_off, ranks);
  else
    k_leverage_chol_t<32><<<grid, 128, 0, st>>>(fs, linv, stride, ok, scores, score_off, ranks);
  RTB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Leverage scores of every row of every factor from the eigenpairs of A^T A.
// rank cutoff (Gram form): mu_k > max(I,R) * eps * mu_max  and mu_k > 0.
// grid = (ceil(max I / 128), modes), block 128.
__global__ void k_leverage_rows(const FactorSet fs, const double* evals, const double* evecs,
                                int stride, double lambda, double* scores,
                                const long long* score_off, int* ranks, const int* skip) {
  const int mode = blockIdx.y;
  if (skip && skip[mode]) return;
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
  // one block per mode: the scores are staged in shared memory by all threads (every load in
  // flight at once), then warp 0 runs the serial left-to-right sum from shared memory
  __shared__ double ss[4096];
  const int mode = blockIdx.x;
  if (mode >= order) return;
  const int lane = threadIdx.x & 31;
  const double* s = scores + off[mode];
  double* c = cdf + off[mode];
  const int n = rows[mode];
  double running = 0.0;
  for (int c0 = 0; c0 < n; c0 += 4096) {
    const int cn = min(4096, n - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < cn; e += blockDim.x) ss[e] = s[c0 + e];
    __syncthreads();
    if (threadIdx.x < 32) {
      for (int base = 0; base < cn; base += 32) {
        const double v = base + lane < cn ? ss[base + lane] : 0.0;
        double mine = 0.0;
        const int cnt = min(32, cn - base);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const double x = __shfl_sync(0xffffffffu, v, k);
          if (k < cnt) running = __dadd_rn(running, x);
          if (lane == k) mine = running;
        }
        if (base + lane < cn) c[c0 + base + lane] = mine;
      }
    }
  }
  if (threadIdx.x == 0) sums[mode] = running;
}

// ---------------------------------------------------------------------------
// Symmetric pseudoinverse from eigenpairs: P = V diag(1/mu_k) V^T over
// |mu_k| > n*eps*max|mu| (singular values of a symmetric matrix are |mu|).
// grid = batch, block = 256. P stored row-major n x n at out + b*stride.
__global__ void k_sym_pinv(const double* evals, const double* evecs, const int* ns, int stride,
                           double* out, int* ranks, const int* skip) {
  const int b = blockIdx.x;
  if (skip && skip[b]) return;
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

void sym_eigen(const double* in, const int* ns_dev, int nmax, int stride, double* evals,
               double* evecs, int* status, int nmat, cudaStream_t st, const int* skip) {
  if (nmax <= 32) {
    const int np = nmax + (nmax & 1);
    const int threads = std::max(64, ceil_div(np * 32, 32) * 32);
    k_sym_eigen_cta<<<nmat, threads, 0, st>>>(in, ns_dev, stride, evals, evecs, status, skip);
  } else {
    if (skip) throw Error(4, "eigen: skip flags need n <= 32");
    if (nmax > 64) throw Error(4, "eigen: n > 64 not supported");
    const int np = nmax + (nmax & 1);
    const size_t smem = (2 * (size_t)np * (np + 1) + 2 * np) * 8;
    set_max_smem(k_sym_eigen, (2 * 64 * 65 + 2 * 64) * 8);
    k_sym_eigen<<<nmat, 128, smem, st>>>(in, ns_dev, stride, evals, evecs, status);
  }
  RTB_LAUNCH_CHECK();
}

void spd_small(const double* in, const int* ns_dev, int stride, double tolrel, double* linv,
               double* pinv, int* ok, int nmat, cudaStream_t st, int nmax) {
  // rows beyond n are padded with the identity, so any NM >= n gives the same factor
  if (nmax <= 8)
    k_spd_small<8><<<ceil_div(nmat, 4), 128, 0, st>>>(in, ns_dev, stride, tolrel, linv, pinv, ok, nmat);
  else if (nmax <= 16)
    k_spd_small<16><<<ceil_div(nmat, 4), 128, 0, st>>>(in, ns_dev, stride, tolrel, linv, pinv, ok, nmat);
  else
    k_spd_small<32><<<ceil_div(nmat, 4), 128, 0, st>>>(in, ns_dev, stride, tolrel, linv, pinv, ok, nmat);
  RTB_LAUNCH_CHECK();
}

}  // namespace rtb
