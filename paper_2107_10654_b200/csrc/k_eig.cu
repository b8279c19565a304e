// k_eig.cu -- symmetric eigendecomposition for d > 64 (FP64): parallel two-sided block
// Jacobi, hand-written for the pinv fallback of the core solve and the dense ridge toolkit.
//
// Reference semantics: the reference pseudo-inverts the sketched Gram through its one-sided
// Jacobi SVD (ref svd.cpp:21-67, 87-97; linalg.cpp:8-26; sketch_ridge.cpp:130-139). For a
// symmetric G the singular triplets are (|mu_k|, v_k, sign(mu_k) v_k) of its eigenpairs, so
// G^+ b = sum_{|mu_k| > d eps max|mu|} v_k (v_k^T b) / mu_k. A Jacobi method is kept on purpose:
// like the reference's it computes small eigenvalues of graded PSD matrices to high relative
// accuracy, which is what decides the rank cut.
//
// Layout: A and V are Dp x Dp row-major (Dp = d rounded up to a multiple of 64; the padding
// rows/columns of A are zero and are never rotated, so V's first d columns are exactly the
// eigenvectors of the d x d input). Blocks of EB = 16 indices are paired by a round-robin
// tournament (nb - 1 rounds per sweep, nb = Dp / 16); per round:
//   k_bj_sub   one warp per block pair: one cyclic Jacobi sweep over the 32 x 32 subproblem
//              S = A[P, P] (P = the pair's 32 indices) in shared memory (round-robin rotations,
//              threshold max(eps ||A||_F, eps sqrt|a_pp a_qq|)); the accumulated rotation Q
//              (32 x 32, re-orthonormalised) is written out, or a skip flag when S is already
//              diagonal. One inner sweep per round measured as fast to converge (in outer
//              sweeps) as diagonalising S fully, at a third of the time (RTB_EIG_INNER)
//   k_bj_rows  A[P, :] <- Q^T A[P, :]        (DMMA m8n8k4, 32 x 64 output tiles)
//   k_bj_cols  A[:, P] <- A[:, P] Q and V[:, P] <- V[:, P] Q   (64 x 32 output tiles)
// A sweep in which no subproblem rotated ends the iteration (one host read per sweep: this
// is a rare fallback path, not the per-sweep hot path).
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace rtb {

namespace {
constexpr int EB = 16;       // indices per block
constexpr int ES = 2 * EB;   // subproblem size
constexpr int ELD = ES + 1;  // smem row stride of a subproblem
constexpr int kSubWarps = 4;
constexpr int kTile = 64;    // panel tile of the rotation GEMMs

struct EigLayout {
  double* A;
  double* V;
  double* Q;       // [npairs][32][32]
  int* flag;       // [npairs] 1 = the pair rotated this round
  int* count;      // [1] rotated pairs this sweep
  double* fro;     // [1] ||A||_F
  double* y;       // [d] pinv projection
  int Dp, nb;
};

EigLayout eig_layout(int d, void* work) {
  EigLayout l;
  l.Dp = ceil_div(d, kTile) * kTile;
  l.nb = l.Dp / EB;
  char* p = static_cast<char*>(work);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  const size_t dd = (size_t)l.Dp * l.Dp;
  l.A = reinterpret_cast<double*>(take(dd * 8));
  l.V = reinterpret_cast<double*>(take(dd * 8));
  l.Q = reinterpret_cast<double*>(take((size_t)(l.nb / 2) * ES * ES * 8));
  l.flag = reinterpret_cast<int*>(take((size_t)(l.nb / 2) * 4));
  l.count = reinterpret_cast<int*>(take(16));
  l.fro = reinterpret_cast<double*>(take(16));
  l.y = reinterpret_cast<double*>(take((size_t)d * 8));
  return l;
}

// block of tournament position `pos` in round r (position 0 fixed, the rest rotate)
__device__ __forceinline__ int bj_at(int pos, int r, int nb) {
  return pos == 0 ? 0 : 1 + (pos - 1 + r) % (nb - 1);
}
__device__ __forceinline__ void bj_pair(int k, int r, int nb, int& p, int& q) {
  p = bj_at(k, r, nb);
  q = bj_at(nb - 1 - k, r, nb);
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}
// global index of local subproblem index i (0..31) of the pair (p, q)
__device__ __forceinline__ int bj_idx(int i, int p, int q) {
  return i < EB ? p * EB + i : q * EB + (i - EB);
}

__global__ void k_bj_init(const double* __restrict__ in, int d, int Dp, double* __restrict__ A,
                          double* __restrict__ V, const int* guard) {
  if (guard && *guard == 0) return;
  const long long n = (long long)Dp * Dp;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / Dp), j = (int)(e % Dp);
    A[e] = (i < d && j < d) ? in[(size_t)i * d + j] : 0.0;
    V[e] = i == j ? 1.0 : 0.0;
  }
}

__global__ void k_bj_fro(const double* __restrict__ A, long long n, double* fro, const int* guard) {
  if (guard && *guard == 0) return;
  __shared__ double red[32];
  double s = 0.0;
  for (long long e = threadIdx.x; e < n; e += blockDim.x) s = fma(A[e], A[e], s);
  s = block_sum<1024>(s, red);
  if (threadIdx.x == 0) *fro = sqrt(s);
}

// one warp per block pair of round r
__global__ void __launch_bounds__(kSubWarps * 32)
    k_bj_sub(const double* __restrict__ A, int Dp, int nb, int r, const double* fro,
             double* __restrict__ Qout, int* __restrict__ flag, int* count, int max_inner,
             const int* guard) {
  if (guard && *guard == 0) return;
  extern __shared__ double esm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * kSubWarps + warp;
  if (k >= nb / 2) return;
  double* S = esm + (size_t)warp * (2 * ES * ELD + 3 * EB);
  double* Q = S + ES * ELD;
  double* cs = Q + ES * ELD;                          // [16] c, [16] s
  int* pq = reinterpret_cast<int*>(cs + 2 * EB);      // [16] p | q << 8
  int p, q;
  bj_pair(k, r, nb, p, q);
  // lane = row of the subproblem
  const int gi = bj_idx(lane, p, q);
  const double* arow = A + (size_t)gi * Dp;
  for (int j = 0; j < ES; ++j) {
    S[lane * ELD + j] = arow[bj_idx(j, p, q)];
    Q[lane * ELD + j] = lane == j ? 1.0 : 0.0;
  }
  __syncwarp();
  const double tol_abs = DBL_EPSILON * *fro;
  bool any = false;
  for (int sweep = 0; sweep < max_inner; ++sweep) {
    bool rot = false;
    for (int step = 0; step < ES - 1; ++step) {
      if (lane < EB) {
        int a = lane == 0 ? 0 : 1 + (lane - 1 + step) % (ES - 1);
        int b = 1 + (ES - 2 - lane + step) % (ES - 1);
        if (a > b) {
          const int t = a;
          a = b;
          b = t;
        }
        const double apq = S[a * ELD + b], app = S[a * ELD + a], aqq = S[b * ELD + b];
        double c = 1.0, s = 0.0;
        if (fabs(apq) > fmax(tol_abs, DBL_EPSILON * sqrt(fabs(app * aqq))) && apq != 0.0) {
          const double theta = (aqq - app) / (2.0 * apq);
          const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = c * t;
          rot = true;
        }
        cs[lane] = c;
        cs[EB + lane] = s;
        pq[lane] = a | (b << 8);
      }
      __syncwarp();
      // columns: S <- S J, Q <- Q J (lane = row)
      for (int m = 0; m < EB; ++m) {
        const double s = cs[EB + m];
        if (s == 0.0) continue;
        const double c = cs[m];
        const int a = pq[m] & 255, b = pq[m] >> 8;
        const double sa = S[lane * ELD + a], sb = S[lane * ELD + b];
        S[lane * ELD + a] = c * sa - s * sb;
        S[lane * ELD + b] = s * sa + c * sb;
        const double qa = Q[lane * ELD + a], qb = Q[lane * ELD + b];
        Q[lane * ELD + a] = c * qa - s * qb;
        Q[lane * ELD + b] = s * qa + c * qb;
      }
      __syncwarp();
      // rows: S <- J^T S (lane = column)
      for (int m = 0; m < EB; ++m) {
        const double s = cs[EB + m];
        if (s == 0.0) continue;
        const double c = cs[m];
        const int a = pq[m] & 255, b = pq[m] >> 8;
        const double sa = S[a * ELD + lane], sb = S[b * ELD + lane];
        S[a * ELD + lane] = c * sa - s * sb;
        S[b * ELD + lane] = s * sa + c * sb;
      }
      __syncwarp();
      if (lane < EB && cs[EB + lane] != 0.0) {
        const int a = pq[lane] & 255, b = pq[lane] >> 8;
        S[a * ELD + b] = 0.0;
        S[b * ELD + a] = 0.0;
      }
      __syncwarp();
    }
    rot = __any_sync(0xffffffffu, rot);
    any |= rot;
    if (!rot) break;
  }
  if (any) {
    // re-orthonormalise the accumulated rotation (modified Gram-Schmidt on its columns, lane =
    // row): hundreds of rotations leave ~1e-13 drift, which the V panels would otherwise
    // accumulate over every round that applies a Q
    for (int j = 0; j < ES; ++j) {
      double nrm = Q[lane * ELD + j] * Q[lane * ELD + j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      const double qj = Q[lane * ELD + j] / sqrt(nrm);
      Q[lane * ELD + j] = qj;
      for (int m = j + 1; m < ES; ++m) {
        double dot = qj * Q[lane * ELD + m];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        Q[lane * ELD + m] -= dot * qj;
      }
    }
  }
  double* qo = Qout + (size_t)k * ES * ES;
  for (int j = 0; j < ES; ++j) qo[lane * ES + j] = Q[lane * ELD + j];
  if (lane == 0) {
    flag[k] = any ? 1 : 0;
    if (any) atomicAdd(count, 1);
  }
}

// A[P, c0:c0+64] <- Q^T A[P, c0:c0+64]   (one CTA per (pair, column tile), 4 warps)
__global__ void __launch_bounds__(128)
    k_bj_rows(double* __restrict__ A, int Dp, int nb, int r, const double* __restrict__ Qg,
              const int* __restrict__ flag, const int* guard) {
  if (guard && *guard == 0) return;
  const int k = blockIdx.x;
  if (!flag[k]) return;
  __shared__ double Qs[ES][ES + 1];
  __shared__ double T[ES][kTile + 1];
  int p, q;
  bj_pair(k, r, nb, p, q);
  const int c0 = blockIdx.y * kTile;
  const double* qk = Qg + (size_t)k * ES * ES;
  for (int e = threadIdx.x; e < ES * ES; e += blockDim.x) Qs[e / ES][e % ES] = qk[e];
  for (int e = threadIdx.x; e < ES * kTile; e += blockDim.x) {
    const int i = e / kTile, j = e % kTile;
    T[i][j] = A[(size_t)bj_idx(i, p, q) * Dp + c0 + j];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double c[8][2];
#pragma unroll
  for (int ct = 0; ct < 8; ++ct) c[ct][0] = c[ct][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < ES / 4; ++kk) {
    const double a = Qs[4 * kk + t][8 * warp + g];  // (Q^T)[8w + g][4kk + t]
#pragma unroll
    for (int ct = 0; ct < 8; ++ct) dmma_8x8x4(c[ct][0], c[ct][1], a, T[4 * kk + t][8 * ct + g]);
  }
  // each output row 8w + g belongs to this warp only: write straight back
  double* out = A + (size_t)bj_idx(8 * warp + g, p, q) * Dp + c0;
#pragma unroll
  for (int ct = 0; ct < 8; ++ct) {
    out[8 * ct + 2 * t] = c[ct][0];
    out[8 * ct + 2 * t + 1] = c[ct][1];
  }
}

// X[r0:r0+64, P] <- X[r0:r0+64, P] Q for X = A (z = 0) and X = V (z = 1)
__global__ void __launch_bounds__(128)
    k_bj_cols(double* __restrict__ A, double* __restrict__ V, int Dp, int nb, int r,
              const double* __restrict__ Qg, const int* __restrict__ flag, const int* guard) {
  if (guard && *guard == 0) return;
  const int k = blockIdx.x;
  if (!flag[k]) return;
  __shared__ double Qs[ES][ES + 1];
  __shared__ double T[kTile][ES + 1];
  double* X = blockIdx.z ? V : A;
  int p, q;
  bj_pair(k, r, nb, p, q);
  const int r0 = blockIdx.y * kTile;
  const double* qk = Qg + (size_t)k * ES * ES;
  for (int e = threadIdx.x; e < ES * ES; e += blockDim.x) Qs[e / ES][e % ES] = qk[e];
  for (int e = threadIdx.x; e < kTile * ES; e += blockDim.x) {
    const int i = e / ES, j = e % ES;
    T[i][j] = X[(size_t)(r0 + i) * Dp + bj_idx(j, p, q)];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double c[2][4][2];
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) c[rt][ct][0] = c[rt][ct][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < ES / 4; ++kk) {
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) {
      const double a = T[16 * warp + 8 * rt + g][4 * kk + t];
#pragma unroll
      for (int ct = 0; ct < 4; ++ct)
        dmma_8x8x4(c[rt][ct][0], c[rt][ct][1], a, Qs[4 * kk + t][8 * ct + g]);
    }
  }
#pragma unroll
  for (int rt = 0; rt < 2; ++rt) {
    double* out = X + (size_t)(r0 + 16 * warp + 8 * rt + g) * Dp;
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      out[bj_idx(8 * ct + 2 * t, p, q)] = c[rt][ct][0];
      out[bj_idx(8 * ct + 2 * t + 1, p, q)] = c[rt][ct][1];
    }
  }
}

// eigenvalues = diag(A)[0:d], eigenvectors = V[0:d, 0:d] (column k)
__global__ void k_bj_extract(const double* __restrict__ A, const double* __restrict__ V, int d,
                             int Dp, double* __restrict__ evals, double* __restrict__ evecs,
                             const int* guard) {
  if (guard && *guard == 0) return;
  const long long n = (long long)d * d;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / d), j = (int)(e % d);
    if (evecs) evecs[e] = V[(size_t)i * Dp + j];
    if (i == 0) evals[j] = A[(size_t)j * Dp + j];
  }
}

// pinv apply: y_k = (v_k . b) / mu_k for |mu_k| > d eps max|mu| (and mu_k != 0), else 0;
// one warp per eigenvector (column k of V, stride Dp). rank_out = number kept.
__global__ void k_bj_pinv_project(const double* __restrict__ A, const double* __restrict__ V,
                                  int d, int Dp, const double* __restrict__ b,
                                  double* __restrict__ y, int* __restrict__ rank_out,
                                  const int* guard) {
  if (guard && *guard == 0) return;
  __shared__ double mmax_s;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < d; ++k) m = fmax(m, fabs(A[(size_t)k * Dp + k]));
    mmax_s = m;
  }
  __syncthreads();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= d) return;
  const double cutoff = (double)d * DBL_EPSILON * mmax_s;
  const double m = A[(size_t)warp * Dp + warp];
  const bool keep = fabs(m) > cutoff && m != 0.0;
  double acc = 0.0;
  if (keep)
    for (int j = lane; j < d; j += 32) acc = fma(V[(size_t)j * Dp + warp], b[j], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    y[warp] = keep ? acc / m : 0.0;
    if (keep) atomicAdd(rank_out, 1);
  }
}

// x[j] = sum_k V[j][k] y[k], one warp per row (fixed k order per lane + tree)
__global__ void k_bj_pinv_expand(const double* __restrict__ V, int d, int Dp,
                                 const double* __restrict__ y, double* __restrict__ x,
                                 const int* guard) {
  if (guard && *guard == 0) return;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= d) return;
  double acc = 0.0;
  for (int k = lane; k < d; k += 32) {
    const double yk = y[k];
    if (yk != 0.0) acc = fma(V[(size_t)warp * Dp + k], yk, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) x[warp] = acc;
}

}  // namespace

size_t eig_large_work_bytes(int d) {
  const size_t Dp = (size_t)ceil_div(d, kTile) * kTile, nb = Dp / EB;
  return 2 * (Dp * Dp * 8 + 256) + (nb / 2) * ES * ES * 8 + (nb / 2) * 4 + 3 * 256 +
         (size_t)d * 8 + 1024;
}

// Diagonalises the symmetric d x d A_in (device, unchanged). Returns the number of sweeps
// run, or -1 if 40 sweeps did not converge. The result stays in the workspace (A = diag,
// V = eigenvectors); evals/evecs (optional, device) receive it unsorted.
static int bj_run(const double* A_in, int d, void* work, cudaStream_t st) {
  EigLayout l = eig_layout(d, work);
  static const int max_inner = std::getenv("RTB_EIG_INNER") ? std::atoi(std::getenv("RTB_EIG_INNER")) : 1;
  const long long n = (long long)l.Dp * l.Dp;
  k_bj_init<<<(unsigned)std::min<long long>(ceil_div<long long>(n, 256), 4 * kNumSMs), 256, 0,
              st>>>(A_in, d, l.Dp, l.A, l.V, nullptr);
  RTB_LAUNCH_CHECK();
  k_bj_fro<<<1, 1024, 0, st>>>(l.A, n, l.fro, nullptr);
  RTB_LAUNCH_CHECK();
  const int npairs = l.nb / 2;
  const size_t sub_smem = (size_t)kSubWarps * (2 * ES * ELD + 3 * EB) * 8;
  set_max_smem(k_bj_sub, (int)sub_smem);
  const dim3 gr((unsigned)npairs, (unsigned)(l.Dp / kTile));
  const dim3 gc((unsigned)npairs, (unsigned)(l.Dp / kTile), 2);
  for (int sweep = 0; sweep < 40; ++sweep) {
    RTB_CUDA(cudaMemsetAsync(l.count, 0, 4, st));
    for (int r = 0; r < l.nb - 1; ++r) {
      k_bj_sub<<<ceil_div(npairs, kSubWarps), kSubWarps * 32, sub_smem, st>>>(
          l.A, l.Dp, l.nb, r, l.fro, l.Q, l.flag, l.count, max_inner, nullptr);
      RTB_LAUNCH_CHECK();
      k_bj_rows<<<gr, 128, 0, st>>>(l.A, l.Dp, l.nb, r, l.Q, l.flag, nullptr);
      RTB_LAUNCH_CHECK();
      k_bj_cols<<<gc, 128, 0, st>>>(l.A, l.V, l.Dp, l.nb, r, l.Q, l.flag, nullptr);
      RTB_LAUNCH_CHECK();
    }
    int cnt = 0;
    RTB_CUDA(cudaMemcpyAsync(&cnt, l.count, 4, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaStreamSynchronize(st));
    static const bool trace = std::getenv("RTB_EIG_TRACE") != nullptr;
    if (trace) std::fprintf(stderr, "[eig] d=%d sweep %d: %d of %d pairs x %d rounds rotated\n", d,
                            sweep + 1, cnt, npairs, l.nb - 1);
    if (cnt == 0) return sweep + 1;
  }
  return -1;
}

void sym_eig_large(const double* A_in, int d, double* evals, double* evecs, void* work,
                   cudaStream_t st) {
  if (d <= 0) throw Error(1, "compact_svd: empty matrix");
  if (bj_run(A_in, d, work, st) < 0)
    throw Error(3, "Jacobi SVD did not converge (block Jacobi eigensolver, 40 sweeps)");
  EigLayout l = eig_layout(d, work);
  k_bj_extract<<<(unsigned)std::min<long long>(ceil_div<long long>((long long)d * d, 256),
                                                4 * kNumSMs),
                 256, 0, st>>>(l.A, l.V, d, l.Dp, evals, evecs, nullptr);
  RTB_LAUNCH_CHECK();
}

size_t pinv_large_work_bytes(int d) { return eig_large_work_bytes(d); }

void pinv_solve_large(double* G, int d, const double* b, double* x, int* rank_dev, void* work,
                      size_t work_bytes, cudaStream_t st) {
  if (work_bytes < eig_large_work_bytes(d)) throw Error(4, "pinv_solve_large: workspace");
  if (bj_run(G, d, work, st) < 0)
    throw Error(3, "Jacobi SVD did not converge (block Jacobi eigensolver, 40 sweeps)");
  EigLayout l = eig_layout(d, work);
  double* y = l.y;
  RTB_CUDA(cudaMemsetAsync(rank_dev, 0, 4, st));
  k_bj_pinv_project<<<ceil_div(d * 32, 256), 256, 0, st>>>(l.A, l.V, d, l.Dp, b, y, rank_dev,
                                                          nullptr);
  RTB_LAUNCH_CHECK();
  k_bj_pinv_expand<<<ceil_div(d * 32, 256), 256, 0, st>>>(l.V, d, l.Dp, y, x, nullptr);
  RTB_LAUNCH_CHECK();
}

}  // namespace rtb
