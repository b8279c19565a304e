// k_pcg.cu -- the sketched core solve as Kronecker-preconditioned conjugate gradients.
//
// Reference: solve_sketched_ridge solves G x = b with a Jacobi-SVD pseudoinverse
// (ref sketch_ridge.cpp:130-139). G = K^T W K + lambda * diag(c) is SPD whenever
// lambda > 0 and every augmented row was drawn (c_j > 0), and it is a (1 +- eps)
// spectral approximation of the unsketched K^T K + lambda I (the point of ridge
// leverage-score sampling). For the Kronecker design K = A_1 (x) ... (x) A_N,
//     M = K^T K = (x)_n A_n^T A_n,   M^-1 = (x)_n P_n,  P_n = (A_n^T A_n)^-1,
// with the P_n from the score step's factor-Gram Cholesky (k_spd_small).
// Preconditioned by M, CG sees eigenvalues in [(1 - eps), (1 + eps)(1 + lambda /
// mu_min)] and converges in a few tens of iterations; M^-1 r costs N mode
// products on a d-vector.
//
// The matvec never touches the d x d Gram. G's entries depend only on the vech
// pairs of the first N-1 modes (k_gram.cu), so it is read from the "last-mode
// blocks" B[u_1..u_{N-1}][r][c] (C2: 38 MB, L2-resident across iterations):
//   q[i_1, im, r] = sum_{j_1} sum_{jm, c} B[v(i_1,j_1)][v(im,jm)][r][c] p[j_1, jm, c]
// CTA u owns the slice u_1 = v(a, b), a <= b, and produces both of its
// contributions (to q[a] with p[b], to q[b] with p[a]) from one read of the slice.
//
// One persistent cooperative kernel runs all iterations with two grid barriers
// per iteration: (A) slice partials -> barrier -> (B) each CTA sums the partials
// of its own rows in a fixed order (+ the augmented diagonal) -> barrier -> (C)
// every CTA redundantly and bit-identically updates the FULL r and x, applies
// M^-1, forms the dot products and the next p in shared memory.
// Iterations stop at a backward-stable residual, ||r|| <= tol max(||b||, ||G||~ ||x||)
// (||G||~ = lambda + prod_n ||A_n^T A_n||_F >= ||G||), and the result is accepted
// only if the true residual ||b - G x|| <= check_tol (||G||~ ||x|| + ||b||) (one
// extra matvec); otherwise status != 0 and the caller falls back to Cholesky.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <functional>
#include <cstdio>
#include <cstdlib>

namespace rtb {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

struct PcgShared {
  int d, order, rows_per_cta;
  int R[kMaxOrder], J[kMaxOrder], m[kMaxOrder];
  int dprime;     // d / R_1 (entries per first-mode index)
  int mid;        // prod_{1 <= n < N-1} R_n (middle modes)
  int last;       // R_N
  int mmid;       // prod_{1 <= n < N-1} m_n (middle vech blocks)
  int m1;         // vech pairs of mode 1 (slices)
  int jc;         // generic slice matvec: each slice split into jc chunks of the middle
                  // index jm (work units m1 * jc, partial sums per chunk); 1 for fast3
  int t32;        // tiled rank-32 matvec (slice_partials_t32): order 3, R_3 = 32, R_2 % 8 == 0
  int ng;         // t32: groups of 8 middle indices (R_2 / 8)
  int ntile;      // t32: tiles per slice, ng (ng + 1) / 2 (off-diagonal first)
  int t4;         // tiled order-4 matvec (slice_partials_t4)
  int t4h;        // t4: u3 ranges per (u1, u2) unit (finer work units for the tail)
  // distributed solve (k_pcg_dist_*): this rank holds and multiplies the slices u1 in
  // [u_lo, u_hi) only (blocks stored from u_lo on); aug_on: it also adds the augmented diagonal
  // (one rank). Single GPU: [0, m1), aug_on = 1.
  int u_lo, u_hi, aug_on;
};

struct PcgArgs {
  const double* B;        // last-mode blocks of the data Gram
  const double* b;
  double* x;
  double* q;              // [d]
  double* part;           // [m1][2][d']
  double* rpart;          // [grid] residual partials
  int warm;               // x holds a starting guess
  const int* warm_dev;    // non-null: the warm flag is read on the device
  unsigned* counter;
  int* status;            // [0] status, [1] iterations
  const double* pinv;     // per mode (stride): (A_n^T A_n)^-1, row-major
  int linv_stride;
  const int* linv_ok;     // per mode: Cholesky of A_n^T A_n succeeded
  const double* grams;    // per mode (stride): A_n^T A_n
  const double* evals;    // per mode (stride): eigenvalues of A_n^T A_n (descending)
  const double* evecs;    // per mode (stride): V[i*R+k], column k = eigenvector k
  const double* prep;     // k_pcg_prep: [0] ||G|| estimate, [1] 1/mu_min(K^T K), [2] eigen form
  const int* aug_count;
  double aug_term;
  double lambda;
  int max_iter;
  double tol;
  double check_tol;
  unsigned long long* prof;  // optional: per-phase ns accumulated by CTA 0 (RTB_PCG_PROF)
  double* vglobal;           // large d: each CTA's redundant vectors in global memory
                             // (6 dv doubles per CTA, L2-resident); nullptr: shared memory
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1u);
    while (ld_relaxed_u32(counter) < target) {
    }
    __threadfence();
  }
  __syncthreads();
}

// Deterministic block sum (fixed thread order, fixed tree): identical in every CTA.
__device__ __forceinline__ double block_sum_det(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (lane < kWarps) t = red[lane];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;  // every thread holds the total
}

// Two deterministic block sums with one pair of barriers.
__device__ __forceinline__ void block_sum2_det(double& v0, double& v1, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) {
    red[w] = v0;
    red[kWarps + w] = v1;
  }
  __syncthreads();
  double t0 = 0.0, t1 = 0.0;
  if (lane < kWarps) {
    t0 = red[lane];
    t1 = red[kWarps + lane];
  }
  for (int o = 16; o > 0; o >>= 1) {
    t0 += __shfl_xor_sync(0xffffffffu, t0, o);
    t1 += __shfl_xor_sync(0xffffffffu, t1, o);
  }
  v0 = t0;
  v1 = t1;
}

// out[o, j, k] = sum_i P[i * RM + j] X[o, i, k] (i, j < R <= RM; P symmetric) on
// a d-vector in shared memory. RX = R when every mode has exactly that rank
// (no guards: loops unroll into straight-line code), else 0 (guarded loops).
// J > 1: (fiber, 8-output group) per thread, X reads contiguous across threads,
//        P rows warp-uniform (broadcast LDS.128).
// J == 1: output j fixed per thread when kThreads % R == 0: column j of P is held
//        in registers and the fiber's inputs are broadcast reads.
template <int RM, int RX>
__device__ __forceinline__ void mode_product(const double* X, double* out, const double* P, int d,
                                             int Rrt, int J) {
  const int R = RX ? RX : Rrt;
  if (J == 1 && (kThreads % R) == 0) {
    const int j = threadIdx.x % R;
    double pc[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) pc[i] = (RX || i < R) ? P[i * RM + j] : 0.0;
    const int ostep = kThreads / R;
    for (int o = threadIdx.x / R; o < d / R; o += ostep) {
      const double* x = X + o * R;
      double acc0 = 0.0, acc1 = 0.0;
      if (RX && (RX % 2) == 0) {
#pragma unroll
        for (int i = 0; i < RM; i += 2) {
          const double2 xx = *reinterpret_cast<const double2*>(x + i);
          acc0 = fma(pc[i], xx.x, acc0);
          acc1 = fma(pc[i + 1], xx.y, acc1);
        }
      } else {
#pragma unroll
        for (int i = 0; i < RM; ++i)
          if (i < R) acc0 = fma(pc[i], x[i], acc0);
      }
      out[o * R + j] = acc0 + acc1;
    }
    return;
  }
  if (J == 1) {
    for (int e = threadIdx.x; e < d; e += kThreads) {
      const int o = e / R, j = e - o * R;
      const double* x = X + o * R;
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < RM; ++i)
        if (i < R) acc = fma(P[i * RM + j], x[i], acc);
      out[e] = acc;
    }
    return;
  }
  const int fibers = d / R;
  const int ngrp = (R + 7) / 8;
  const int work = fibers * ngrp;
  for (int w = threadIdx.x; w < work; w += kThreads) {
    const int g = w / fibers, f = w - g * fibers;
    const int o = f / J, k = f - o * J;
    const int base = o * R * J + k;
    const int j0 = 8 * g;
    double acc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] = 0.0;
#pragma unroll
    for (int i = 0; i < RM; ++i) {
      if (RX || i < R) {
        const double xi = X[base + i * J];
        const double2* wr = reinterpret_cast<const double2*>(P + i * RM + j0);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const double2 ww = wr[t];
          acc[2 * t] = fma(ww.x, xi, acc[2 * t]);
          acc[2 * t + 1] = fma(ww.y, xi, acc[2 * t + 1]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (RX ? (RX % 8 == 0 || j0 + t < R) : (j0 + t < R)) out[base + (j0 + t) * J] = acc[t];
  }
}

// Rank-16 modes on the FP64 tensor cores: out[o, j, k] = sum_i P[i][j] X[o, i, k] is
// C (16 x NN) = P^T (16 x 16) B (16 x NN) with column n = (o, k), NN = d / 16,
// B[i][n] = X[o*16*J + i*J + k]. m8n8k4 DMMAs: A = P^T fragments in registers
// (a = P[4 ks + t][8 mt + g]), one 8-column tile per warp iteration.
__device__ __forceinline__ void mode_product_dmma16(const double* X, double* out, const double* P,
                                                    int d, int J) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double a[2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) a[mt][ks] = P[(ks * 4 + t) * 16 + mt * 8 + g];
  const int ntiles = d / 128;
  for (int nt = warp; nt < ntiles; nt += kWarps) {
    const int n = nt * 8 + g;
    const int o = n / J, k = n - o * J;
    const double* xb = X + o * 16 * J + k;
    double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const double b = xb[(ks * 4 + t) * J];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) dmma_8x8x4(c[mt][0], c[mt][1], a[mt][ks], b);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n2 = nt * 8 + 2 * t + e;
      const int o2 = n2 / J, k2 = n2 - o2 * J;
      double* ob = out + o2 * 16 * J + k2;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) ob[(mt * 8 + g) * J] = c[mt][e];
    }
  }
}

// The 16 x 16 x 16 preconditioner below works on the FP64 pipe from fragment tables and
// XOR-swizzled shared layouts, so none of its shared-memory accesses is bank-conflicted
// beyond the 4-way read of the canonical r (the previous form, with its row stride of 16
// doubles on every fragment access, ran at 8-way conflicts: ~4.6k wavefronts per call).
// Fragment tables, Wf[set][mode][v][lane] (set 0 = W1, 1 = W2; v < 8; g = lane/4, t = lane%4):
//   modes 0, 1 (A operand W^T):      W[4 ks + t][8 mt + g],          v = 4 mt + ks
//   mode 2 (B operand, k permuted):  W[pi(ks, t)][8 nt + g],         v = 4 nt + ks
// pi(ks, t) = 8 (ks >> 1) + 2 t + (ks & 1) is the column a lane's C fragment of the previous
// GEMM holds, so the mode-3 GEMM takes that C fragment as its A operand without a round trip.
constexpr int kWfDoubles = 2 * 3 * 8 * 32;
__device__ __forceinline__ int pre16_pi(int ks, int t) { return 8 * (ks >> 1) + 2 * t + (ks & 1); }
__device__ void build_frags16(const double* W1, const double* W2, double* Wf) {
  for (int e = threadIdx.x; e < kWfDoubles; e += blockDim.x) {
    const int set = e / 768, n = (e / 256) % 3, v = (e / 32) & 7, lane = e & 31;
    const int g = lane >> 2, t = lane & 3, hi = v >> 2, ks = v & 3;
    const double* W = (set ? W2 : W1) + n * 256;
    Wf[e] = n < 2 ? W[(4 * ks + t) * 16 + 8 * hi + g] : W[pre16_pi(ks, t) * 16 + 8 * hi + g];
  }
}
// Layout of the preconditioner's output (and of its swizzled input in the eigen form):
// canonical element e lives at e ^ (8 * bit 8 of e), i.e. i3 ^ 8 (i1 & 1).
__device__ __forceinline__ int pre16_swz(int e) { return e ^ ((e >> 5) & 8); }

// One pass out = (W_1^T x W_2^T x W_3^T) src: warp w takes slab i1 = w through modes 2 and 3
// (two chained GEMMs, the intermediate in registers), writes it to scr in the exchange layout
// [i1][i2][i3 ^ (4 (i1 & 3) ^ 8 (i2 & 1))], one CTA barrier, then mode 1 (32 column tiles
// of 8, two per warp) into dst (pre16_swz layout). src_swz: src is in the pre16_swz layout.
// dst may alias src, not scr.
__device__ __forceinline__ void pre16_pass(const double* src, bool src_swz, double* scr,
                                           double* dst, const double* Wf) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const double* xs = src + w * 256;
  const int sx = src_swz ? 8 * (w & 1) : 0;
  double c[2][2][2], z[2][2][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) c[mt][nt][0] = c[mt][nt][1] = z[mt][nt][0] = z[mt][nt][1] = 0.0;
  // mode 2: Y[j2][i3] = sum_i2 W2[i2][j2] X[i2][i3]
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    double a[2], b[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) a[mt] = Wf[(256 + (4 * mt + ks) * 32) + lane];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) b[nt] = xs[(4 * ks + t) * 16 + ((8 * nt + g) ^ sx)];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) dmma_8x8x4(c[mt][nt][0], c[mt][nt][1], a[mt], b[nt]);
  }
  // mode 3: Z[j2][j3] = sum_i3 Y[j2][i3] W3[i3][j3], A = Y's C fragment (k = pi(ks, t))
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    double b[2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) b[nt] = Wf[(512 + (4 * nt + ks) * 32) + lane];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
        dmma_8x8x4(z[mt][nt][0], z[mt][nt][1], c[mt][ks >> 1][ks & 1], b[nt]);
  }
  {
    double* zs = scr + w * 256;
    const int fz = 4 * (w & 3) ^ 8 * (g & 1);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
        *reinterpret_cast<double2*>(zs + (8 * mt + g) * 16 + ((8 * nt + 2 * t) ^ fz)) =
            make_double2(z[mt][nt][0], z[mt][nt][1]);
  }
  __syncthreads();
  // mode 1: out[j1][n] = sum_i1 W1[i1][j1] Z[i1][n], n = 16 i2 + i3
  double a1[2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) a1[mt][ks] = Wf[(4 * mt + ks) * 32 + lane];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int nt = w + 16 * h, i2 = nt >> 1, b8 = 8 * (nt & 1);
    double o[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int i1 = 4 * ks + t;
      const double b = scr[i1 * 256 + i2 * 16 + ((b8 + g) ^ (4 * t ^ 8 * (i2 & 1)))];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) dmma_8x8x4(o[mt][0], o[mt][1], a1[mt][ks], b);
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
      *reinterpret_cast<double2*>(dst + (8 * mt + g) * 256 + i2 * 16 + ((b8 + 2 * t) ^ (8 * (g & 1)))) =
          make_double2(o[mt][0], o[mt][1]);
  }
}

// z = M^-1 r for 16 x 16 x 16 (order 3, all ranks 16, kWarps = 16 slabs) from the fragment
// tables Wf (build_frags16 of W1, W2). r is canonical and preserved; returns the buffer
// holding z in the pre16_swz layout.
__device__ double* precondition16(const double* r, double* a, double* b, const double* Wf,
                                  const double* dinv, bool eig, unsigned long long* pf = nullptr) {
  unsigned long long t0 = pf ? gtimer() : 0;
  auto mk = [&](int k) {
    if (pf) {
      const unsigned long long t1 = gtimer();
      pf[k] += t1 - t0;
      t0 = t1;
    }
  };
  pre16_pass(r, false, a, b, Wf);
  __syncthreads();
  mk(12);
  if (!eig) return b;
  for (int e = threadIdx.x; e < 4096; e += kThreads) b[pre16_swz(e)] *= dinv[e];
  __syncthreads();
  pre16_pass(b, true, a, b, Wf + 768);
  __syncthreads();
  mk(6);
  return b;
}

// z = M^-1 r with scratch a, b; returns the buffer holding z. Two forms:
//  * P form (eig == false): M = (x)_n A_n^T A_n, M^-1 = (x)_n P_n: N mode products.
//  * eigen form: M = (x)_n A_n^T A_n + lambda I = V diag(lambda + prod mu) V^T:
//    N products with V^T, a diagonal scaling, N products with V (2N + 1 passes).
template <int RM, int RX>
__device__ double* precondition(const PcgShared& sh, const double* r, double* a, double* b,
                                const double* W1, const double* W2, const double* dinv, bool eig,
                                unsigned long long* prof = nullptr) {
  const double* src = r;
  double* dst = a;
  unsigned long long t0 = prof ? gtimer() : 0;
  for (int n = 0; n < sh.order; ++n) {
    if constexpr (RX == 16 && RM == 16) mode_product_dmma16(src, dst, W1 + n * RM * RM, sh.d, sh.J[n]);
    else mode_product<RM, RX>(src, dst, W1 + n * RM * RM, sh.d, sh.R[n], sh.J[n]);
    __syncthreads();
    if (prof && n < 8) {
      const unsigned long long t1 = gtimer();
      prof[8 + n] += t1 - t0;
      t0 = t1;
    }
    src = dst;
    dst = (dst == a) ? b : a;
  }
  if (eig) {
    double* t = const_cast<double*>(src);
    for (int e = threadIdx.x; e < sh.d; e += kThreads) t[e] *= dinv[e];
    __syncthreads();
    for (int n = 0; n < sh.order; ++n) {
      if constexpr (RX == 16 && RM == 16) mode_product_dmma16(src, dst, W2 + n * RM * RM, sh.d, sh.J[n]);
      else mode_product<RM, RX>(src, dst, W2 + n * RM * RM, sh.d, sh.R[n], sh.J[n]);
      __syncthreads();
      src = dst;
      dst = (dst == a) ? b : a;
    }
  }
  return const_cast<double*>(src);
}

// (A) slice partials: for slice u1 = v(a, b), side 0 = q[a, :] from p[b, :],
// side 1 = q[b, :] from p[a, :] (absent when a == b).
template <int RM>
__device__ void slice_partials(const PcgArgs& A, const PcgShared& sh, const double* p) {
  const int last = sh.last, mid = sh.mid, dp = sh.dprime;
  const int nout = 2 * dp;
  for (int unit = sh.u_lo * sh.jc + blockIdx.x; unit < sh.u_hi * sh.jc; unit += gridDim.x) {
    const int u1 = unit / sh.jc, ch = unit - u1 * sh.jc;
    const int jm0 = (int)((long long)mid * ch / sh.jc), jm1 = (int)((long long)mid * (ch + 1) / sh.jc);
    int a, b;
    pair_of(u1, sh.R[0], a, b);
    const double* Bs = A.B + (size_t)(u1 - sh.u_lo) * sh.mmid * last * last;
    for (int o = threadIdx.x; o < nout; o += kThreads) {
      const int r = o % last;
      const int t = o / last;
      const int side = t & 1, im = t >> 1;
      if (side == 1 && a == b) continue;
      const double* pv = p + (size_t)(side == 0 ? b : a) * dp;
      // middle-mode digits (modes 1..N-2), kept in registers: every loop below
      // runs to the compile-time bound with a guard, so indices are static
      int idig[kMaxOrder], jdig[kMaxOrder];
      {
        int rem = im, remj = jm0;
#pragma unroll
        for (int n = kMaxOrder - 1; n >= 1; --n) {
          idig[n] = 0;
          jdig[n] = 0;
          if (n <= sh.order - 2) {
            idig[n] = rem % sh.R[n];
            rem /= sh.R[n];
            jdig[n] = remj % sh.R[n];
            remj /= sh.R[n];
          }
        }
      }
      double s0 = 0.0, s1 = 0.0;
      for (int jm = jm0; jm < jm1; ++jm) {
        int umid = 0;
#pragma unroll
        for (int n = 1; n < kMaxOrder; ++n)
          if (n <= sh.order - 2) {
            const int x = idig[n], y = jdig[n];
            umid = umid * sh.m[n] + upper_pair(min(x, y), max(x, y), sh.R[n]);
          }
        const double* row = Bs + ((size_t)umid * last + r) * last;
        const double* ps = pv + (size_t)jm * last;
        if ((last & 1) == 0) {
          double2 g[RM / 2];
#pragma unroll
          for (int c = 0; c < RM / 2; ++c)
            if (2 * c < last) g[c] = __ldg(reinterpret_cast<const double2*>(row) + c);
#pragma unroll
          for (int c = 0; c < RM / 2; ++c)
            if (2 * c < last) {
              const double2 pp = reinterpret_cast<const double2*>(ps)[c];
              s0 = fma(g[c].x, pp.x, s0);
              s1 = fma(g[c].y, pp.y, s1);
            }
        } else {
          double g[RM];
#pragma unroll
          for (int c = 0; c < RM; ++c)
            if (c < last) g[c] = __ldg(row + c);
#pragma unroll
          for (int c = 0; c < RM; ++c)
            if (c < last) s0 = fma(g[c], ps[c], s0);
        }
        bool carry = true;  // odometer over the middle modes
#pragma unroll
        for (int n = kMaxOrder - 1; n >= 1; --n)
          if (n <= sh.order - 2 && carry) {
            if (++jdig[n] < sh.R[n]) carry = false;
            else jdig[n] = 0;
          }
      }
      A.part[(((size_t)u1 * sh.jc + ch) * 2 + side) * dp + (size_t)im * last + r] = s0 + s1;
    }
  }
}

// (A) tiled path, order 3 with R_3 == 32 (C5: d = 32768, 2.3 GB of blocks streamed from HBM
// per matvec): every block B[u1][v(i2, j2)] (32 x 32, symmetric, 8 KB) is read ONCE and applied
// to the four targets q_a(i2) <- p_b(j2), q_b(i2) <- p_a(j2), q_a(j2) <- p_b(i2),
// q_b(j2) <- p_a(i2) (u1 = v(a, b)). Work unit = one warp on one tile of a slice: the blocks
// (i2, j2) with i2 in group I and j2 in group J (groups of 8, I <= J; off-diagonal tiles, 64
// blocks, are handed out first, then the 36-block diagonal ones) from an atomic ticket
// counter, so the 16 warps of every CTA stay busy to the end of the matvec. Lane (rq, c) =
// (l / 4, l % 4) holds rows rq + 8 rr (rr < 4), columns 8 h + 2 c + {0, 1} (h < 4) of a block:
// each load instruction covers 8 rows x 64 contiguous bytes. Row targets q(i2) accumulate
// in registers along a tile row, column targets q(j2) in the warp's shared accumulator; the
// tile's result (both sides, both roles: 1024 doubles) goes to part[u1][tile]. Which warp
// computes a tile does not change its value: the matvec is deterministic.
__device__ __forceinline__ int t32_tile_of(int I, int J, int ng) {
  return I == J ? ng * (ng - 1) / 2 + I : I * ng - I * (I + 1) / 2 + (J - I - 1);
}

__device__ void slice_partials_t32(const PcgArgs& A, const PcgShared& sh, const double* p,
                                   double* accw, unsigned ticket_base) {
  const int R2 = sh.R[1], dp = sh.dprime, ng = sh.ng;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rq = lane >> 2, c = lane & 3;
  const int nod = ng * (ng - 1) / 2;
  const int nsl = sh.u_hi - sh.u_lo;  // this rank's slices
  const unsigned nunits = (unsigned)nsl * sh.ntile;
  double* acc = accw + (size_t)w * 1024;
  unsigned* tickets = A.counter + 8;
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(tickets, 1u) - ticket_base;
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= nunits) break;
    int u1, tile, I, J;
    if (t < (unsigned)nsl * nod) {
      u1 = (int)(t / nod);
      tile = (int)(t % nod);
      I = 0;
      int rem = tile;
      while (rem >= ng - 1 - I) {
        rem -= ng - 1 - I;
        ++I;
      }
      J = I + 1 + rem;
    } else {
      const unsigned v = t - (unsigned)nsl * nod;
      u1 = (int)(v / ng);
      I = J = (int)(v % ng);
      tile = nod + I;
    }
    const int ul = u1;  // slice within this rank's blocks
    u1 += sh.u_lo;
    int a, b;
    pair_of(u1, sh.R[0], a, b);
    const bool two_sides = a != b;
    const double* Bs = A.B + (size_t)ul * sh.mmid * 1024;
    const double* pa = p + (size_t)a * dp;
    const double* pb = p + (size_t)b * dp;
    for (int e = lane; e < 1024; e += 32) acc[e] = 0.0;
    __syncwarp();
    for (int kk = 0; kk < 8; ++kk) {
      const int i2 = 8 * I + kk;
      double xbi[8], xai[8];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 vb = *reinterpret_cast<const double2*>(pb + i2 * 32 + 8 * h + 2 * c);
        xbi[2 * h] = vb.x;
        xbi[2 * h + 1] = vb.y;
        const double2 va = two_sides ? *reinterpret_cast<const double2*>(pa + i2 * 32 + 8 * h + 2 * c)
                                     : make_double2(0.0, 0.0);
        xai[2 * h] = va.x;
        xai[2 * h + 1] = va.y;
      }
      double y0[4] = {0.0, 0.0, 0.0, 0.0}, y2[4] = {0.0, 0.0, 0.0, 0.0};
      for (int jj = (I == J ? kk : 0); jj < 8; ++jj) {
        const int j2 = 8 * J + jj;
        const double* blk = Bs + (size_t)upper_pair(i2, j2, R2) * 1024;
        double2 g[4][4];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
          for (int h = 0; h < 4; ++h)
            g[rr][h] = __ldcs(reinterpret_cast<const double2*>(blk + (rq + 8 * rr) * 32 + 8 * h + 2 * c));
        double xbj[8], xaj[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const double2 vb = *reinterpret_cast<const double2*>(pb + j2 * 32 + 8 * h + 2 * c);
          xbj[2 * h] = vb.x;
          xbj[2 * h + 1] = vb.y;
          const double2 va = *reinterpret_cast<const double2*>(pa + j2 * 32 + 8 * h + 2 * c);
          xaj[2 * h] = va.x;
          xaj[2 * h + 1] = va.y;
        }
        const bool off = j2 != i2;
        double t1[4], t3[4];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          double s0 = 0.0, s2 = 0.0, s1 = 0.0, s3 = 0.0;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const double2 gg = g[rr][h];
            s0 = fma(gg.x, xbj[2 * h], s0);
            s0 = fma(gg.y, xbj[2 * h + 1], s0);
            s2 = fma(gg.x, xaj[2 * h], s2);
            s2 = fma(gg.y, xaj[2 * h + 1], s2);
            s1 = fma(gg.x, xbi[2 * h], s1);
            s1 = fma(gg.y, xbi[2 * h + 1], s1);
            s3 = fma(gg.x, xai[2 * h], s3);
            s3 = fma(gg.y, xai[2 * h + 1], s3);
          }
          y0[rr] += s0;
          y2[rr] += s2;
          t1[rr] = s1;
          t3[rr] = s3;
        }
        if (off) {  // column targets q_a(j2), q_b(j2): sum over the 4 column lanes
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            t1[rr] += __shfl_xor_sync(0xffffffffu, t1[rr], 1);
            t1[rr] += __shfl_xor_sync(0xffffffffu, t1[rr], 2);
            t3[rr] += __shfl_xor_sync(0xffffffffu, t3[rr], 1);
            t3[rr] += __shfl_xor_sync(0xffffffffu, t3[rr], 2);
          }
          if (c == 0) {
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
              acc[(1 * 8 + jj) * 32 + rq + 8 * rr] += t1[rr];        // side 0, role 1
              acc[(3 * 8 + jj) * 32 + rq + 8 * rr] += t3[rr];        // side 1, role 1
            }
          }
          __syncwarp();
        }
      }
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        y0[rr] += __shfl_xor_sync(0xffffffffu, y0[rr], 1);
        y0[rr] += __shfl_xor_sync(0xffffffffu, y0[rr], 2);
        y2[rr] += __shfl_xor_sync(0xffffffffu, y2[rr], 1);
        y2[rr] += __shfl_xor_sync(0xffffffffu, y2[rr], 2);
      }
      if (c == 0) {
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          acc[(0 * 8 + kk) * 32 + rq + 8 * rr] += y0[rr];             // side 0, role 0
          acc[(2 * 8 + kk) * 32 + rq + 8 * rr] += y2[rr];             // side 1, role 0
        }
      }
      __syncwarp();
    }
    double* out = A.part + ((size_t)u1 * sh.ntile + tile) * 1024;
    const int ne = two_sides ? 1024 : 512;
    for (int e = lane; e < ne; e += 32) out[e] = acc[e];
    __syncwarp();
  }
}

// (B) own rows for the tiled path: q[i1, i2, r] = sum over j1 (slice v(i1, j1), side i1 > j1)
// of the tiles holding i2 as a row (role 0) or column (role 1) target, in a fixed order.
__device__ void reduce_rows_t32(const PcgArgs& A, const PcgShared& sh, const double* p, int row0,
                                int nrows, double* qout) {
  const int dp = sh.dprime, R1 = sh.R[0], ng = sh.ng;
  for (int e = row0 + threadIdx.x; e < row0 + nrows; e += kThreads) {
    const int i1 = e / dp, rest = e - i1 * dp;
    const int i2 = rest >> 5, r = rest & 31;
    const int G = i2 >> 3, k = i2 & 7;
    double s = 0.0;
#pragma unroll 4
    for (int j1 = 0; j1 < R1; ++j1) {
      const int u1 = upper_pair(min(i1, j1), max(i1, j1), R1);
      if (u1 < sh.u_lo || u1 >= sh.u_hi) continue;  // another rank's slice
      const int side = i1 <= j1 ? 0 : 1;
      const double* base = A.part + (size_t)u1 * sh.ntile * 1024 + (size_t)(side * 2) * 256 + k * 32 + r;
      double v[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // role 0: tiles (G, J), J >= G; role 1: tiles (I, G), I <= G
        v[q] = (G + q < ng) ? __ldcg(base + (size_t)t32_tile_of(G, G + q, ng) * 1024) : 0.0;
        v[4 + q] = (q <= G) ? __ldcg(base + 256 + (size_t)t32_tile_of(q, G, ng) * 1024) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) s += v[q];
    }
    const int cnt = __ldg(A.aug_count + e);
    if (cnt > 0 && sh.aug_on) s = fma((double)cnt * A.aug_term, p[e], s);
    qout[e] = s;
  }
}

// (A) tiled path, order 4 (C3: R = 10, d = 10^4, 133 MB of blocks per matvec): every block
// B[u1][u2][u3] (L x L, L = R_4, symmetric) is read ONCE and applied to all of its targets:
// sides (q_a <- p_b, q_b <- p_a) x orientations of u2 = v(i2, j2) x orientations of
// u3 = v(i3, j3) (up to 8). Work unit = one warp on (u1, u2) and all m3 blocks of u3, from a
// ticket counter; the sources p_{a,b}[{i2, j2}][:][:] and the targets q_{a,b}[{i2, j2}][:][:]
// (4 R3 L values each) live in the warp's shared memory. Lanes form G = 32 / L groups, group g
// takes block u3 = u3_0 + g, lane r of a group row r of it; the groups add their
// contributions to the shared targets one after another (fixed order: deterministic). The
// unit's targets go to part[u1 m2 + u2][side][role][x3][r] (role 0: i2's row, 1: j2's).
constexpr int kT4H = 1;  // u3 ranges per t4 work unit (3 at C3 balanced the tail but tripled the per-unit
                         // source loads and partials: slower)
template <int LM>  // L <= LM <= 16
__device__ void slice_partials_t4(const PcgArgs& A, const PcgShared& sh, const double* p,
                                  double* accw, unsigned ticket_base) {
  // per block one m16n8k16 DMMA: C (16 x 8) = B_blk (L x L, zero-padded to 16 x 16) x S, the
  // 8 columns of S the sources of the block's 8 (side, u2 orientation, u3 orientation)
  // combinations; C[r][n] is combination n's contribution to its target row r. The 8 targets
  // of one block are distinct addresses, so the warp adds them to its shared targets at once.
  const int R1 = sh.R[0], R2 = sh.R[1], R3 = sh.R[2], L = sh.R[3];
  const int m2 = sh.m[1], m3 = sh.m[2];
  const int dp = sh.dprime, RL = R3 * L;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double* src = accw + (size_t)w * 8 * RL;  // [side source: 0 = p_b, 1 = p_a][role][x3][c]
  double* acc = src + 4 * RL;               // [side][role][x3][r]
  constexpr int H = kT4H;
  const unsigned nunits = (unsigned)(sh.u_hi - sh.u_lo) * m2 * H;
  unsigned* tickets = A.counter + 8;
  // B-fragment column g = combination n = g: side sd = g >> 2, o2 = (g >> 1) & 1, o3 = g & 1
  const int n_sd = g >> 2, n_o2 = (g >> 1) & 1, n_o3 = g & 1;
  // C columns of this lane: 2t, 2t + 1
  for (;;) {
    unsigned tk = 0;
    if (lane == 0) tk = atomicAdd(tickets, 1u) - ticket_base;
    tk = __shfl_sync(0xffffffffu, tk, 0);
    if (tk >= nunits) break;
    const int hh = (int)(tk % (unsigned)H);
    const unsigned tu = tk / (unsigned)H;
    const int ul = (int)(tu / m2), u2 = (int)(tu - (unsigned)ul * m2);
    const int u1 = ul + sh.u_lo;
    const int u3lo = (int)((long long)m3 * hh / H), u3hi = (int)((long long)m3 * (hh + 1) / H);
    int a, b, i2, j2;
    pair_of(u1, R1, a, b);
    pair_of(u2, R2, i2, j2);
    const bool two_sides = a != b, two2 = i2 != j2;
    {
      constexpr int kPer = 16;  // 4 R3 L <= 512
      double tv[kPer];
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int e = lane + 32 * k;
        tv[k] = 0.0;
        if (e < 4 * RL) {
          const int sd = e / (2 * RL), rem = e - sd * 2 * RL, role = rem / RL, xr = rem - role * RL;
          const int vec = sd == 0 ? b : a, row = role == 0 ? i2 : j2;
          if (sd == 0 || two_sides) tv[k] = __ldcg(p + (size_t)vec * dp + row * RL + xr);
        }
      }
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int e = lane + 32 * k;
        if (e < 4 * RL) {
          src[e] = tv[k];
          acc[e] = 0.0;
        }
      }
    }
    __syncwarp();
    const double* Bu = A.B + ((size_t)ul * sh.mmid + (size_t)u2 * m3) * L * L;
    const bool n_side_on = n_sd == 0 || two_sides;
    const bool n_o2_on = n_o2 == 0 || two2;
    const int n_yrole = n_o2 == 0 ? 1 : 0;  // x2 = i2 reads row j2 and vice versa
    constexpr int kAhead = 4;  // blocks in flight per warp (8: 2x slower, register spills)
    for (int u30 = u3lo; u30 < u3hi; u30 += kAhead) {
      double af[kAhead][8];
#pragma unroll
      for (int k = 0; k < kAhead; ++k) {
        const int u3 = u30 + k;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const int rr = g + 8 * (v & 1), cc = t + 4 * (v >> 1);
          af[k][v] = (u3 < u3hi && rr < L && cc < L) ? __ldcs(Bu + ((size_t)u3 * L + rr) * L + cc) : 0.0;
        }
      }
#pragma unroll
      for (int k = 0; k < kAhead; ++k) {
        const int u3 = u30 + k;
        if (u3 >= u3hi) break;
        int i3, j3;
        pair_of(u3, R3, i3, j3);
        const bool two3 = i3 != j3;
        // B fragment: column g's source at rows t + 4 v
        double bf[4];
        {
          const bool on = n_side_on && n_o2_on && (n_o3 == 0 || two3);
          const int y3 = n_o3 == 0 ? j3 : i3;
          const double* sv = src + (n_sd * 2 + n_yrole) * RL + y3 * L;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int kk = t + 4 * v;
            bf[v] = (on && kk < L) ? sv[kk] : 0.0;
          }
        }
        double c[4] = {0.0, 0.0, 0.0, 0.0};
        dmma_16x8x16(c, af[k], bf);
        // C[r][n]: rows g, g + 8; columns 2t, 2t + 1 -> targets
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int r = g + 8 * (v >> 1), n = 2 * t + (v & 1);
          const int sd = n >> 2, o2 = (n >> 1) & 1, o3 = n & 1;
          const bool on = r < L && (sd == 0 || two_sides) && (o2 == 0 || two2) && (o3 == 0 || two3);
          if (on) {
            const int x3 = o3 == 0 ? i3 : j3;
            acc[(sd * 2 + o2) * RL + x3 * L + r] += c[v];
          }
        }
        __syncwarp();
      }
    }
    double* out = A.part + (((size_t)u1 * m2 + u2) * H + hh) * 4 * RL;
    const int ne = two_sides ? 4 * RL : 2 * RL;
    for (int e = lane; e < ne; e += 32) out[e] = acc[e];
    __syncwarp();
  }
}

// (B) own rows for the order-4 tiled path: q[i1, x2, x3, r] = sum over j1 (slice v(i1, j1),
// side i1 > j1) and y (unit u2 = v(x2, y), role x2 > y) of part[u1 m2 + u2][side][role][x3 r].
// 16 lanes per row (lane k takes j1 = k, k + 16, ...), a fixed shuffle tree over them.
__device__ void reduce_rows_t4(const PcgArgs& A, const PcgShared& sh, const double* p, int row0,
                               int nrows, double* qout) {
  const int R1 = sh.R[0], R2 = sh.R[1], RL = sh.R[2] * sh.R[3], m2 = sh.m[1];
  const int dp = sh.dprime;
  const int k = threadIdx.x & 15;
  for (int base = row0; base < row0 + nrows; base += kThreads / 16) {
    const int e = base + (threadIdx.x >> 4);
    const bool ok = e < row0 + nrows;
    double s = 0.0;
    if (ok) {
      const int i1 = e / dp, rest = e - i1 * dp;
      const int x2 = rest / RL, xr = rest - x2 * RL;
      for (int j1 = k; j1 < R1; j1 += 16) {
        const int u1 = upper_pair(min(i1, j1), max(i1, j1), R1);
        if (u1 < sh.u_lo || u1 >= sh.u_hi) continue;  // another rank's slice
        const int side = i1 <= j1 ? 0 : 1;
        constexpr int H = kT4H;
        const double* pb = A.part + (size_t)u1 * m2 * H * 4 * RL + (size_t)(side * 2) * RL + xr;
        for (int y = 0; y < R2; ++y) {
          const int u2 = upper_pair(min(x2, y), max(x2, y), R2);
          const int role = x2 <= y ? 0 : 1;
          for (int h = 0; h < H; ++h)
            s += __ldcg(pb + ((size_t)u2 * H + h) * 4 * RL + (size_t)role * RL);
        }
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (ok && k == 0) {
      const int c = __ldg(A.aug_count + e);
      if (c > 0 && sh.aug_on) s = fma((double)c * A.aug_term, p[e], s);
      qout[e] = s;
    }
  }
}

// (A) fast path, order 3 with R_3 == 16: every unordered middle pair (i2 <= j2)
// of the slice is read ONCE (one 2 KB block) and applied to the four (side,
// orientation) targets -- q_a(i2) += B p_b(j2), q_a(j2) += B p_b(i2), q_b(i2) +=
// B p_a(j2), q_b(j2) += B p_a(i2) (B symmetric). Lane (r = l/4, c = l%4) reads
// columns {2c, 2c+1, 8+2c, 9+2c} of rows r and r+8 (8 lines per load), partial
// dots are reduced over the 4 column lanes by shuffles, and each warp adds its
// results to private accumulators acc[w][side][i2][r] (fixed order -> the final
// sum over warps is deterministic).
__device__ void slice_partials_n3(const PcgArgs& A, const PcgShared& sh, const double* p,
                                  double* accw) {
  const int R2 = sh.R[1], dp = sh.dprime;  // dp = R2 * 16
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, c = lane & 3;
  const int m2 = sh.m[1];
  for (int u1 = blockIdx.x; u1 < sh.m1; u1 += gridDim.x) {
    int a, b;
    pair_of(u1, sh.R[0], a, b);
    const bool two_sides = a != b;
    double* acc = accw + (size_t)w * 2 * dp;
    for (int e = lane; e < 2 * dp; e += 32) acc[e] = 0.0;
    __syncwarp();
    const double* Bs = A.B + (size_t)u1 * m2 * 256;
    const double* pa = p + (size_t)a * dp;
    const double* pb = p + (size_t)b * dp;
    // the L2 reads of a warp's blocks are issued kAhead at a time (latency, not
    // bandwidth, bounds this loop: ~9 blocks per warp)
#ifndef RTB_PCG_AHEAD
#define RTB_PCG_AHEAD 1
#endif
    constexpr int kAhead = RTB_PCG_AHEAD;
    for (int pbase = w; pbase < m2; pbase += kWarps * kAhead) {
      double2 gq[kAhead][2][2];
#pragma unroll
      for (int k = 0; k < kAhead; ++k) {
        const int pidx = pbase + k * kWarps;
        if (pidx < m2) {
          const double* blk = Bs + (size_t)pidx * 256;
#pragma unroll
          for (int rr = 0; rr < 2; ++rr)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              gq[k][rr][h] =
                  __ldg(reinterpret_cast<const double2*>(blk + (r + 8 * rr) * 16 + 8 * h + 2 * c));
        }
      }
#pragma unroll
      for (int k = 0; k < kAhead; ++k) {
      const int pidx = pbase + k * kWarps;
      if (pidx >= m2) break;
      int i2, j2;
      pair_of(pidx, R2, i2, j2);
      const bool two_orient = i2 != j2;
      const double2(&g)[2][2] = gq[k];
      // targets: 0 = q_a(i2) <- p_b(j2), 1 = q_a(j2) <- p_b(i2), 2 = q_b(i2) <- p_a(j2),
      // 3 = q_b(j2) <- p_a(i2)
      const double* src[4] = {pb + j2 * 16, pb + i2 * 16, pa + j2 * 16, pa + i2 * 16};
      double t[4][2];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const double2 p0 = *reinterpret_cast<const double2*>(src[v] + 2 * c);
        const double2 p1 = *reinterpret_cast<const double2*>(src[v] + 8 + 2 * c);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          double s = g[rr][0].x * p0.x;
          s = fma(g[rr][0].y, p0.y, s);
          s = fma(g[rr][1].x, p1.x, s);
          s = fma(g[rr][1].y, p1.y, s);
          t[v][rr] = s;
        }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          t[v][rr] += __shfl_xor_sync(0xffffffffu, t[v][rr], 1);
          t[v][rr] += __shfl_xor_sync(0xffffffffu, t[v][rr], 2);
        }
      if (c == 0) {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int row = r + 8 * rr;
          acc[i2 * 16 + row] += t[0][rr];
          if (two_orient) acc[j2 * 16 + row] += t[1][rr];
          if (two_sides) {
            acc[dp + i2 * 16 + row] += t[2][rr];
            if (two_orient) acc[dp + j2 * 16 + row] += t[3][rr];
          }
        }
      }
      __syncwarp();
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 2 * dp; e += kThreads) {
      const int side = e >= dp;
      if (side && !two_sides) continue;
      double s = 0.0;
      for (int ww = 0; ww < kWarps; ++ww) s += accw[(size_t)ww * 2 * dp + e];
      A.part[((size_t)u1 * 2 + side) * dp + (e - side * dp)] = s;
    }
    __syncthreads();
  }
}

// (B) own rows: q[e] = sum_{j1} partial + augmented diagonal * p[e].
template <bool JC1>  // JC1: one chunk per slice (the fast order-3 matvec)
__device__ void reduce_rows(const PcgArgs& A, const PcgShared& sh, const double* p, int row0,
                            int nrows, double* qout) {
  const int jc = JC1 ? 1 : sh.jc;
  const int dp = sh.dprime, R1 = sh.R[0];
  for (int e = row0 + threadIdx.x; e < row0 + nrows; e += kThreads) {
    const int i1 = e / dp, rest = e - i1 * dp;
    double s = 0.0;
    for (int j1 = 0; j1 < R1; ++j1) {
      const int u1 = upper_pair(min(i1, j1), max(i1, j1), R1);
      if (u1 < sh.u_lo || u1 >= sh.u_hi) continue;  // another rank's slice
      const int side = i1 <= j1 ? 0 : 1;
      for (int ch = 0; ch < jc; ++ch)
        s += __ldcg(A.part + (((size_t)u1 * jc + ch) * 2 + side) * dp + rest);
    }
    const int c = __ldg(A.aug_count + e);
    if (c > 0 && sh.aug_on) s = fma((double)c * A.aug_term, p[e], s);
    qout[e] = s;
  }
}

#ifndef RTB_EIG_ABOVE
#define RTB_EIG_ABOVE 4.0
#endif
constexpr double kEigenAbove = RTB_EIG_ABOVE;  // lambda / mu_min above which the eigen form is used
constexpr double kMaxLambdaOverMu = 1e12;     // beyond: not worth CG

// Warp n (one per mode, in parallel): mu_max(A_n^T A_n) and ||P_n||_2 = 1/mu_min by
// power iteration (lane = row). mu_max gives the ||G|| estimate of the stopping test
// (an underestimate only tightens it). The P form of the preconditioner drops lambda:
// every direction with lambda > mu(K^T K) becomes an outlier eigenvalue of M^-1 G that
// CG removes in about one iteration, so a moderate lambda / mu_min(K^T K) is cheap (C2:
// ~2.5, 15 iterations); above kEigenAbove the exact eigen form is used, and only then
// are the factor-Gram eigenpairs computed (skip flags for the eigensolver).
__global__ void k_pcg_prep(const double* __restrict__ grams, const double* __restrict__ pinv,
                           int stride, PcgShared sh, double lambda, double* prep, int* skip) {
  // warp w: mode w >> 1, matrix (w & 1) ? P_n : G_n; row i of M in lane i's registers,
  // the iterate v broadcast through shared memory (independent loads, short chains)
  __shared__ double est[2 * kMaxOrder];
  __shared__ double vs[2 * kMaxOrder][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2 * sh.order) {
    const int n = warp >> 1, which = warp & 1, R = sh.R[n];
    const double* M = (which ? pinv : grams) + (size_t)n * stride;
    double row[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) row[j] = (lane < R && j < R) ? M[lane * R + j] : 0.0;
    double v = lane < R ? 1.0 + 0.01 * lane : 0.0, mu = 0.0;
    for (int itp = 0; itp < 24; ++itp) {
      vs[warp][lane] = v;
      __syncwarp();
      double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        y0 = fma(row[j], vs[warp][j], y0);
        y1 = fma(row[j + 1], vs[warp][j + 1], y1);
        y2 = fma(row[j + 2], vs[warp][j + 2], y2);
        y3 = fma(row[j + 3], vs[warp][j + 3], y3);
      }
      const double y = (y0 + y1) + (y2 + y3);
      double yy = y * y, vy = v * y, vv = v * v;
      for (int o = 16; o > 0; o >>= 1) {
        yy += __shfl_xor_sync(0xffffffffu, yy, o);
        vy += __shfl_xor_sync(0xffffffffu, vy, o);
        vv += __shfl_xor_sync(0xffffffffu, vv, o);
      }
      mu = vv > 0.0 ? vy / vv : 0.0;
      v = yy > 0.0 ? y * rsqrt(yy) : 0.0;
      __syncwarp();
    }
    if (lane == 0) est[2 * n + which] = mu;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 1.0, pn = 1.0;
    for (int n = 0; n < sh.order; ++n) {
      g *= est[2 * n];
      pn *= est[2 * n + 1];
    }
    const bool eig = !(lambda * pn <= kEigenAbove);
    prep[0] = g + lambda;
    prep[1] = pn;
    prep[2] = eig ? 1.0 : 0.0;
    for (int n = 0; n < sh.order; ++n) skip[n] = eig ? 0 : 1;
  }
}

template <int RM, int RX, bool BIG>
__global__ void __launch_bounds__(kThreads, 1) k_pcg(const PcgArgs A, const PcgShared shc) {
  extern __shared__ __align__(16) double sm[];
  const PcgShared& sh = shc;
  const int d = sh.d;
  const int dv = (d + 1) & ~1;
  double* Ps = sm;                          // [order][RM][RM]: P_n (P form) or V_n (eigen form)
  double* VTs = Ps + sh.order * RM * RM;    // [order][RM][RM]: V_n^T (eigen form)
  // the d-vectors: shared memory, or (large d) this CTA's slice of A.vglobal
  // (BIG is a template parameter so that the shared-memory form keeps LDS/STS accesses)
  constexpr bool big = BIG;
  double* vb = big ? A.vglobal + (size_t)blockIdx.x * 6 * dv : VTs + sh.order * RM * RM;
  double* dinv = vb;                        // [d]: 1 / (lambda + prod mu) (eigen form)
  double* r = dinv + dv;
  double* p = r + dv;
  double* s0 = p + dv;
  double* s1 = s0 + dv;
  double* xs = s1 + dv;  // full x, kept redundantly like r and p
  double* red = big ? VTs + sh.order * RM * RM : xs + dv;
  // fast order-3 matvec: per-warp accumulators, in s0/s1 when they are large enough
  const bool fast3 = sh.order == 3 && sh.last == 16 && !big;
  const int row0 = min(d, (int)blockIdx.x * sh.rows_per_cta);
  const int nrows = min(d, row0 + sh.rows_per_cta) - row0;
  const size_t acc_need = (size_t)kWarps * 2 * sh.dprime;
  double* accw = acc_need <= (size_t)2 * dv ? s0 : red + 32;
  // tiled rank-32 matvec (large d): per-warp tile accumulators after red
  const bool t32 = big && sh.t32;
  double* acc32 = red + 32;
  unsigned mv = 0;  // matvecs so far: ticket base of the next one
  const unsigned tick_per = (unsigned)(sh.u_hi - sh.u_lo) * sh.ntile + gridDim.x * kWarps;
  auto mv_partials = [&]() {
    if (t32) slice_partials_t32(A, sh, p, acc32, (mv++) * tick_per);
    else if (fast3) slice_partials_n3(A, sh, p, accw);
    else slice_partials<RM>(A, sh, p);
  };
  auto mv_reduce = [&]() {
    if (t32) reduce_rows_t32(A, sh, p, row0, nrows, A.q);
    else if (fast3) reduce_rows<true>(A, sh, p, row0, nrows, A.q);
    else reduce_rows<false>(A, sh, p, row0, nrows, A.q);
  };

  // applicability: every augmented column drawn (then G >= lambda * min c_j > 0)
  // and every factor Gram Cholesky-factorable (the preconditioner)
  int missing = 0;
  for (int e = threadIdx.x; e < d; e += kThreads) missing |= __ldg(A.aug_count + e) == 0;
  if (threadIdx.x < sh.order) missing |= __ldg(A.linv_ok + threadIdx.x) == 0;
  if (__syncthreads_or(missing) || !(A.lambda > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.status[0] = 3;
      A.status[1] = 0;
    }
    return;
  }

  for (int n = 0; n < sh.order; ++n) {
    const int R = sh.R[n];
    const double* Pg = A.pinv + (size_t)n * A.linv_stride;
    for (int e = threadIdx.x; e < RM * RM; e += kThreads) {
      const int i = e / RM, j = e - i * RM;
      Ps[n * RM * RM + e] = (i < R && j < R) ? Pg[i * R + j] : 0.0;
    }
  }
  __syncthreads();
  const double gnorm = A.prep[0], pnorm = A.prep[1];
  // lambda-free P form while lambda is small against mu_min(K^T K) (few outlier
  // eigenvalues), else the exact eigen form of (x) A_n^T A_n + lambda I
  const bool eig = A.prep[2] != 0.0;
  if (!(A.lambda * pnorm <= kMaxLambdaOverMu)) {  // hopeless for CG: Cholesky path
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.status[0] = 3;
      A.status[1] = 0;
    }
    return;
  }
  if (eig) {
    for (int n = 0; n < sh.order; ++n) {
      const int R = sh.R[n];
      const double* Vg = A.evecs + (size_t)n * A.linv_stride;
      for (int e = threadIdx.x; e < RM * RM; e += kThreads) {
        const int i = e / RM, j = e - i * RM;
        const bool in = i < R && j < R;
        Ps[n * RM * RM + e] = in ? Vg[i * R + j] : 0.0;   // W[i][j] = V[i][j]
        VTs[n * RM * RM + e] = in ? Vg[j * R + i] : 0.0;  // W[i][j] = V[j][i]
      }
    }
    for (int e = threadIdx.x; e < d; e += kThreads) {
      double m = 1.0;
      int rem = e;
      for (int n = sh.order - 1; n >= 0; --n) {
        const int j = rem % sh.R[n];
        rem /= sh.R[n];
        m *= fmax(A.evals[(size_t)n * A.linv_stride + j], 0.0);
      }
      dinv[e] = 1.0 / (m + A.lambda);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < d; e += kThreads) {
    r[e] = A.b[e];
    xs[e] = 0.0;
  }
  __syncthreads();

  unsigned sync_target = 0;

  double bb = 0.0;
  for (int e = threadIdx.x; e < d; e += kThreads) bb = fma(r[e], r[e], bb);
  bb = block_sum_det(bb, red);
  if (bb == 0.0) {
    for (int e = row0 + threadIdx.x; e < row0 + nrows; e += kThreads) A.x[e] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.status[0] = 0;
      A.status[1] = 0;
    }
    return;
  }
  // warm start from x0 = A.x (the previous sweep's core: the system changes little
  // between sweeps): r = b - G x0, kept only if it beats the cold residual ||b||
  if (A.warm_dev ? *A.warm_dev : A.warm) {
    for (int e = threadIdx.x; e < d; e += kThreads) {
      const double x0 = A.x[e];
      xs[e] = x0;
      p[e] = x0;
    }
    __syncthreads();
    mv_partials();
    __syncthreads();
    sync_target += gridDim.x;
    grid_barrier(A.counter, sync_target);
    mv_reduce();
    __syncthreads();
    sync_target += gridDim.x;
    grid_barrier(A.counter, sync_target);
    double r0 = 0.0;
    for (int e = threadIdx.x; e < d; e += kThreads) {
      const double re = A.b[e] - __ldcg(A.q + e);
      s0[e] = re;
      r0 = fma(re, re, r0);
    }
    r0 = block_sum_det(r0, red);
    if (r0 < bb && isfinite(r0)) {
      for (int e = threadIdx.x; e < d; e += kThreads) r[e] = s0[e];
    } else {
      for (int e = threadIdx.x; e < d; e += kThreads) xs[e] = 0.0;
    }
    __syncthreads();
  }
  double* z = precondition<RM, RX>(sh, r, s0, s1, Ps, VTs, dinv, eig);
  double rho = 0.0;
  for (int e = threadIdx.x; e < d; e += kThreads) {
    p[e] = z[e];
    rho = fma(r[e], z[e], rho);
  }
  rho = block_sum_det(rho, red);

  const double tol2 = A.tol * A.tol;
  int it = 0;
  int fail = 0;
  const bool prof = A.prof && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long t0 = prof ? gtimer() : 0, t1;
#define RTB_PCG_MARK(k)                 \
  if (prof) {                           \
    t1 = gtimer();                      \
    A.prof[k] += t1 - t0;               \
    t0 = t1;                            \
  }
  for (; it < A.max_iter; ++it) {
    mv_partials();
    __syncthreads();
    RTB_PCG_MARK(0)
    sync_target += gridDim.x;
    grid_barrier(A.counter, sync_target);
    RTB_PCG_MARK(1)
    mv_reduce();
    __syncthreads();
    RTB_PCG_MARK(2)
    sync_target += gridDim.x;
    grid_barrier(A.counter, sync_target);
    RTB_PCG_MARK(3)
    // every CTA: alpha from the full p.q, full r and x updates
    double pq = 0.0;
    for (int e = threadIdx.x; e < d; e += kThreads) {
      const double qe = __ldcg(A.q + e);
      s0[e] = qe;
      pq = fma(p[e], qe, pq);
    }
    pq = block_sum_det(pq, red);
    if (!(pq > 0.0) || !isfinite(pq)) {
      fail = 2;
      break;
    }
    const double alpha = rho / pq;
    double rr = 0.0, xx = 0.0;
    for (int e = threadIdx.x; e < d; e += kThreads) {
      const double re = fma(-alpha, s0[e], r[e]);
      r[e] = re;
      rr = fma(re, re, rr);
      const double xe = fma(alpha, p[e], xs[e]);
      xs[e] = xe;
      xx = fma(xe, xe, xx);
    }
    block_sum2_det(rr, xx, red);
    RTB_PCG_MARK(4)
    if (rr <= tol2 * fmax(bb, gnorm * gnorm * xx)) {
      ++it;
      break;
    }
    z = precondition<RM, RX>(sh, r, s0, s1, Ps, VTs, dinv, eig, prof ? A.prof : nullptr);
    RTB_PCG_MARK(5)
    double rho2 = 0.0;
    for (int e = threadIdx.x; e < d; e += kThreads) rho2 = fma(r[e], z[e], rho2);
    rho2 = block_sum_det(rho2, red);
    const double beta = rho2 / rho;
    rho = rho2;
    for (int e = threadIdx.x; e < d; e += kThreads) p[e] = fma(beta, p[e], z[e]);
    __syncthreads();
    RTB_PCG_MARK(6)
  }
#undef RTB_PCG_MARK
  // x out (own rows); true residual ||b - G x|| with one more matvec
  double xx = 0.0;
  for (int e = threadIdx.x; e < d; e += kThreads) {
    p[e] = xs[e];
    xx = fma(xs[e], xs[e], xx);
  }
  xx = block_sum_det(xx, red);
  for (int e = row0 + threadIdx.x; e < row0 + nrows; e += kThreads) A.x[e] = xs[e];
  mv_partials();
  sync_target += gridDim.x;
  grid_barrier(A.counter, sync_target);
  mv_reduce();
  __syncthreads();
  double res = 0.0;
  for (int e = row0 + threadIdx.x; e < row0 + nrows; e += kThreads) {
    const double t = A.b[e] - A.q[e];
    res = fma(t, t, res);
  }
  res = block_sum_det(res, red);
  if (threadIdx.x == 0) A.rpart[blockIdx.x] = res;
  sync_target += gridDim.x;
  grid_barrier(A.counter, sync_target);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double tot = 0.0;
    for (int c = 0; c < (int)gridDim.x; ++c) tot += __ldcg(A.rpart + c);
    int st = fail;
    const double scale = gnorm * sqrt(xx) + sqrt(bb);
    if (!st && !(tot <= A.check_tol * A.check_tol * scale * scale)) st = 1;
    A.status[0] = st;
    A.status[1] = it;
  }
}

// ---------------------------------------------------------------------------
// Large-d PCG with DISTRIBUTED vectors (k_pcg_dv). k_pcg's large-d form keeps six d-vectors per
// CTA in global memory and updates / preconditions all of them redundantly in every CTA: at
// C5 (d = 32768) that is 148 x 1.5 MB of vector traffic per iteration (3.7 ms of
// preconditioning per solve), at C3 (d = 10^4) 0.6 ms. Here every d-vector exists once (x, r,
// p, z, scratch, in the workspace); each CTA updates its own rows, dot products are per-CTA
// partials summed by every CTA in a fixed order after a grid barrier (deterministic), and
// M^-1 r = (x)_n P_n r is N grid-strided mode products with a grid barrier between modes.
// Per iteration: matvec (slice partials, own-row sums), alpha, the r / x update, N mode
// products, rho, the p update: 5 + N grid barriers and no redundant vector work.
__device__ __forceinline__ void mode_product_dv(const double* __restrict__ in, double* __restrict__ out,
                                                const double* P, int RM, int R, int J, int d) {
  const int RJ = R * J;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d; e += gridDim.x * blockDim.x) {
    const int o = e / RJ, rem = e - o * RJ;
    const int j = rem / J, k = rem - j * J;
    const double* x = in + o * RJ + k;
    double acc = 0.0;
    for (int i = 0; i < R; ++i) acc = fma(P[i * RM + j], __ldcg(x + i * J), acc);
    out[e] = acc;
  }
}

template <int RM>
__global__ void __launch_bounds__(kThreads, 1) k_pcg_dv(const PcgArgs A, const PcgShared shc) {
  extern __shared__ __align__(16) double sm[];
  const PcgShared& sh = shc;
  const int d = sh.d;
  const int dv = (d + 1) & ~1;
  double* Ps = sm;                          // [order][RM][RM]: P_n (P form) or V_n (eigen form)
  double* VTs = Ps + sh.order * RM * RM;    // [order][RM][RM]: V_n^T (eigen form)
  double* red = VTs + sh.order * RM * RM;   // [32] block reductions
  double* acc32 = red + 32;                 // tiled rank-32 matvec accumulators
  double* gx = A.vglobal;                   // the d-vectors, one copy each
  double* gr = gx + dv;
  double* gp = gr + dv;
  double* ga = gp + dv;
  double* gb = ga + dv;
  double* gdinv = gb + dv;
  __shared__ double bcast[2];
  double* gpart0 = gdinv + dv;              // [2][gridDim.x][2] per-CTA partial sums,
  int nsum = 0;                             // double-buffered by sum parity
  const bool t32 = sh.t32 != 0;
  const int row0 = min(d, (int)blockIdx.x * sh.rows_per_cta);
  const int row1 = min(d, row0 + sh.rows_per_cta);
  unsigned sync_target = 0;
  auto gsync = [&]() {
    sync_target += gridDim.x;
    grid_barrier(A.counter, sync_target);
  };
  // sums of up to 2 per-CTA partials over the grid, identical in every CTA
  // (a CTA writes sum k + 2's partial only after sum k + 1's barrier, which every CTA reaches
  // only after reading sum k's partials: two buffers suffice)
  auto gsum2 = [&](double& v0, double& v1) {
    block_sum2_det(v0, v1, red);
    double* gpart = gpart0 + (size_t)(nsum & 1) * gridDim.x * 2;
    ++nsum;
    if (threadIdx.x == 0) {
      gpart[blockIdx.x * 2] = v0;
      gpart[blockIdx.x * 2 + 1] = v1;
    }
    gsync();
    // warp 0 sums the partials (lane-strided, then a fixed shuffle tree: the same order in
    // every CTA) and broadcasts
    if (threadIdx.x < 32) {
      double t0 = 0.0, t1 = 0.0;
      for (int c = threadIdx.x; c < (int)gridDim.x; c += 32) {
        t0 += __ldcg(gpart + c * 2);
        t1 += __ldcg(gpart + c * 2 + 1);
      }
      for (int o = 16; o > 0; o >>= 1) {
        t0 += __shfl_xor_sync(0xffffffffu, t0, o);
        t1 += __shfl_xor_sync(0xffffffffu, t1, o);
      }
      if (threadIdx.x == 0) {
        bcast[0] = t0;
        bcast[1] = t1;
      }
    }
    __syncthreads();
    v0 = bcast[0];
    v1 = bcast[1];
    __syncthreads();
  };
  auto gsum = [&](double v) {
    double z = 0.0;
    gsum2(v, z);
    return v;
  };
  unsigned mv = 0;
  const unsigned tick_per = (unsigned)(sh.u_hi - sh.u_lo) * sh.ntile + gridDim.x * kWarps;
  // q (own rows, A.q) = G src, src published in global memory
  const bool t4 = sh.t4 != 0;
  const unsigned tick4 = (unsigned)(sh.u_hi - sh.u_lo) * sh.m[1] * sh.t4h + gridDim.x * kWarps;
  const bool mprof = A.prof && blockIdx.x == 0 && threadIdx.x == 0;
  auto matvec = [&](const double* src) {
    const unsigned long long m0 = mprof ? gtimer() : 0;
    if (t32) slice_partials_t32(A, sh, src, acc32, (mv++) * tick_per);
    else if (t4) slice_partials_t4<RM>(A, sh, src, acc32, (mv++) * tick4);
    else slice_partials<RM>(A, sh, src);
    __syncthreads();
    const unsigned long long m1 = mprof ? gtimer() : 0;
    gsync();
    const unsigned long long m2 = mprof ? gtimer() : 0;
    if (t32) reduce_rows_t32(A, sh, src, row0, row1 - row0, A.q);
    else if (t4) reduce_rows_t4(A, sh, src, row0, row1 - row0, A.q);
    else reduce_rows<false>(A, sh, src, row0, row1 - row0, A.q);
    __syncthreads();
    if (mprof) {  // CTA 0: its own partials, the wait for the slowest CTA, its row sums
      A.prof[1] += m1 - m0;
      A.prof[2] += m2 - m1;
      A.prof[3] += gtimer() - m2;
    }
  };

  int missing = 0;
  for (int e = threadIdx.x; e < d; e += kThreads) missing |= __ldg(A.aug_count + e) == 0;
  if (threadIdx.x < sh.order) missing |= __ldg(A.linv_ok + threadIdx.x) == 0;
  const double pnorm = A.prep[1];
  if (__syncthreads_or(missing) || !(A.lambda > 0.0) || !(A.lambda * pnorm <= kMaxLambdaOverMu)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.status[0] = 3;
      A.status[1] = 0;
    }
    return;
  }
  for (int n = 0; n < sh.order; ++n) {
    const int R = sh.R[n];
    const double* Pg = A.pinv + (size_t)n * A.linv_stride;
    for (int e = threadIdx.x; e < RM * RM; e += kThreads) {
      const int i = e / RM, j = e - i * RM;
      Ps[n * RM * RM + e] = (i < R && j < R) ? Pg[i * R + j] : 0.0;
    }
  }
  const double gnorm = A.prep[0];
  const bool eig = A.prep[2] != 0.0;
  if (eig) {
    for (int n = 0; n < sh.order; ++n) {
      const int R = sh.R[n];
      const double* Vg = A.evecs + (size_t)n * A.linv_stride;
      for (int e = threadIdx.x; e < RM * RM; e += kThreads) {
        const int i = e / RM, j = e - i * RM;
        const bool in = i < R && j < R;
        Ps[n * RM * RM + e] = in ? Vg[i * R + j] : 0.0;
        VTs[n * RM * RM + e] = in ? Vg[j * R + i] : 0.0;
      }
    }
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
      double m = 1.0;
      int rem = e;
      for (int n = sh.order - 1; n >= 0; --n) {
        const int j = rem % sh.R[n];
        rem /= sh.R[n];
        m *= fmax(A.evals[(size_t)n * A.linv_stride + j], 0.0);
      }
      gdinv[e] = 1.0 / (m + A.lambda);
    }
  }
  __syncthreads();
  // z = M^-1 src (src complete in global memory): N (or 2N + 1) grid-strided passes
  auto precond = [&](const double* src) -> double* {
    const double* cur = src;
    double* dst = ga;
    for (int n = 0; n < sh.order; ++n) {
      mode_product_dv(cur, dst, Ps + n * RM * RM, RM, sh.R[n], sh.J[n], d);
      gsync();
      cur = dst;
      dst = (dst == ga) ? gb : ga;
    }
    if (eig) {
      double* t = const_cast<double*>(cur);
      for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d; e += gridDim.x * blockDim.x)
        t[e] *= gdinv[e];
      gsync();
      for (int n = 0; n < sh.order; ++n) {
        mode_product_dv(cur, dst, VTs + n * RM * RM, RM, sh.R[n], sh.J[n], d);
        gsync();
        cur = dst;
        dst = (dst == ga) ? gb : ga;
      }
    }
    return const_cast<double*>(cur);
  };

  double bb = 0.0;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
    const double be = A.b[e];
    gr[e] = be;
    gx[e] = 0.0;
    bb = fma(be, be, bb);
  }
  bb = gsum(bb);
  if (bb == 0.0) {
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) A.x[e] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.status[0] = 0;
      A.status[1] = 0;
    }
    return;
  }
  if (A.warm_dev ? *A.warm_dev : A.warm) {
    // r0 = b - G x0, kept only if it beats the cold residual ||b||
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) gx[e] = A.x[e];
    __syncthreads();
    gsync();
    matvec(gx);
    double r0 = 0.0;
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
      const double re = A.b[e] - A.q[e];
      r0 = fma(re, re, r0);
    }
    r0 = gsum(r0);
    const bool keep = r0 < bb && isfinite(r0);
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
      if (keep) gr[e] = A.b[e] - A.q[e];
      else gx[e] = 0.0;
    }
    __syncthreads();
    gsync();
  } else {
    gsync();  // r complete before the first preconditioning
  }
  double* z = precond(gr);
  double rho = 0.0;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
    gp[e] = z[e];
    rho = fma(gr[e], z[e], rho);
  }
  rho = gsum(rho);  // its barrier also publishes p
  const double tol2 = A.tol * A.tol;
  int it = 0, fail = 0;
  const bool prof = A.prof && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long t0 = prof ? gtimer() : 0, t1;
#define RTB_DV_MARK(k)                  \
  if (prof) {                           \
    t1 = gtimer();                      \
    A.prof[k] += t1 - t0;               \
    t0 = t1;                            \
  }
  for (; it < A.max_iter; ++it) {
    matvec(gp);
    RTB_DV_MARK(0)
    double pq = 0.0;
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) pq = fma(gp[e], A.q[e], pq);
    pq = gsum(pq);
    if (!(pq > 0.0) || !isfinite(pq)) {
      fail = 2;
      break;
    }
    const double alpha = rho / pq;
    double rr = 0.0, xx = 0.0;
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
      const double re = fma(-alpha, A.q[e], gr[e]);
      gr[e] = re;
      rr = fma(re, re, rr);
      const double xe = fma(alpha, gp[e], gx[e]);
      gx[e] = xe;
      xx = fma(xe, xe, xx);
    }
    gsum2(rr, xx);  // its barrier also completes r for the preconditioner
    RTB_DV_MARK(4)
    if (rr <= tol2 * fmax(bb, gnorm * gnorm * xx)) {
      ++it;
      break;
    }
    z = precond(gr);
    RTB_DV_MARK(5)
    double rho2 = 0.0;
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) rho2 = fma(gr[e], z[e], rho2);
    rho2 = gsum(rho2);
    const double beta = rho2 / rho;
    rho = rho2;
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) gp[e] = fma(beta, gp[e], z[e]);
    __syncthreads();
    gsync();  // p published
    RTB_DV_MARK(6)
  }
#undef RTB_DV_MARK
  // x out; true residual ||b - G x|| with one more matvec
  double xx = 0.0;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
    A.x[e] = gx[e];
    xx = fma(gx[e], gx[e], xx);
  }
  xx = gsum(xx);  // also publishes x for the matvec
  matvec(gx);
  double res = 0.0;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
    const double t = A.b[e] - A.q[e];
    res = fma(t, t, res);
  }
  res = gsum(res);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int st = fail;
    const double scale = gnorm * sqrt(xx) + sqrt(bb);
    if (!st && !(res <= A.check_tol * A.check_tol * scale * scale)) st = 1;
    A.status[0] = st;
    A.status[1] = it;
  }
}

// ---------------------------------------------------------------------------
// Distributed solve across GPUs (k_pcg_dist_*): the large-d PCG of k_pcg_dv with the matvec
// split over ranks by mode-1 slices. Rank r holds the blocks of slices u1 in [u_lo, u_hi) only
// and computes q_r = sum over its slices (+ the augmented diagonal on one rank); the caller's
// all-reduce sums q over ranks between launches; every rank then runs the identical CG vector
// step on its own GPU (distributed over its CTAs as in k_pcg_dv), so x, r and p stay identical
// everywhere without exchanging them. Three cooperative launches per iteration
// (matvec | all-reduce | step), the CG state in device memory; the host checks the done flag
// every few iterations. The single-GPU case is k_pcg_dv (one launch).
struct DistState {
  double rho, bb, xx, gn;
  int mode, it, fail, pad;  // mode: 0 warm-start matvec, 1 CG, 2 final check, 3 done
};
enum { kDWarm = 0, kDCg = 1, kDCheck = 2, kDDone = 3 };

struct DvCtx {  // the k_pcg_dv helpers for the split kernels
  double *gx, *gr, *gp, *ga, *gb, *gdinv, *gpart0;
};

template <int RM>
__device__ void dist_setup(const PcgArgs& A, const PcgShared& sh, double* Ps, double* VTs,
                           bool eig) {
  for (int n = 0; n < sh.order; ++n) {
    const int R = sh.R[n];
    const double* Pg = eig ? A.evecs + (size_t)n * A.linv_stride : A.pinv + (size_t)n * A.linv_stride;
    for (int e = threadIdx.x; e < RM * RM; e += kThreads) {
      const int i = e / RM, j = e - i * RM;
      const bool in = i < R && j < R;
      Ps[n * RM * RM + e] = in ? Pg[i * R + j] : 0.0;
      if (eig) VTs[n * RM * RM + e] = in ? Pg[j * R + i] : 0.0;
    }
  }
  __syncthreads();
}

// block sums of per-CTA partials across the grid (the k_pcg_dv scheme; parity per launch)
struct GridSum {
  double* gpart0;
  double* red;
  double* bcast;
  unsigned* counter;
  unsigned target = 0;
  int nsum = 0;
  __device__ void sync() {
    target += gridDim.x;
    grid_barrier(counter, target);
  }
  __device__ void sum2(double& v0, double& v1) {
    block_sum2_det(v0, v1, red);
    double* gpart = gpart0 + (size_t)(nsum & 1) * gridDim.x * 2;
    ++nsum;
    if (threadIdx.x == 0) {
      gpart[blockIdx.x * 2] = v0;
      gpart[blockIdx.x * 2 + 1] = v1;
    }
    sync();
    if (threadIdx.x < 32) {
      double t0 = 0.0, t1 = 0.0;
      for (int c = threadIdx.x; c < (int)gridDim.x; c += 32) {
        t0 += __ldcg(gpart + c * 2);
        t1 += __ldcg(gpart + c * 2 + 1);
      }
      for (int o = 16; o > 0; o >>= 1) {
        t0 += __shfl_xor_sync(0xffffffffu, t0, o);
        t1 += __shfl_xor_sync(0xffffffffu, t1, o);
      }
      if (threadIdx.x == 0) {
        bcast[0] = t0;
        bcast[1] = t1;
      }
    }
    __syncthreads();
    v0 = bcast[0];
    v1 = bcast[1];
    __syncthreads();
  }
  __device__ double sum(double v) {
    double z = 0.0;
    sum2(v, z);
    return v;
  }
};

template <int RM>
__device__ double* dist_precond(const PcgShared& sh, GridSum& gs, const double* src, const DvCtx& c,
                                const double* Ps, const double* VTs, bool eig) {
  const double* cur = src;
  double* dst = c.ga;
  for (int n = 0; n < sh.order; ++n) {
    mode_product_dv(cur, dst, Ps + n * RM * RM, RM, sh.R[n], sh.J[n], sh.d);
    gs.sync();
    cur = dst;
    dst = (dst == c.ga) ? c.gb : c.ga;
  }
  if (eig) {
    double* t = const_cast<double*>(cur);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < sh.d; e += gridDim.x * blockDim.x)
      t[e] *= c.gdinv[e];
    gs.sync();
    for (int n = 0; n < sh.order; ++n) {
      mode_product_dv(cur, dst, VTs + n * RM * RM, RM, sh.R[n], sh.J[n], sh.d);
      gs.sync();
      cur = dst;
      dst = (dst == c.ga) ? c.gb : c.ga;
    }
  }
  return const_cast<double*>(cur);
}

__device__ DvCtx dv_ctx(const PcgArgs& A, int d) {
  const int dv = (d + 1) & ~1;
  DvCtx c;
  c.gx = A.vglobal;
  c.gr = c.gx + dv;
  c.gp = c.gr + dv;
  c.ga = c.gp + dv;
  c.gb = c.ga + dv;
  c.gdinv = c.gb + dv;
  c.gpart0 = c.gdinv + dv;
  return c;
}

// z = M^-1 r, rho = r.z, p = z; the caller's barrier after the sum publishes p
template <int RM>
__device__ void dist_start_cg(const PcgArgs& A, const PcgShared& sh, GridSum& gs, const DvCtx& c,
                              const double* Ps, const double* VTs, bool eig, int row0, int row1,
                              DistState* S) {
  double* z = dist_precond<RM>(sh, gs, c.gr, c, Ps, VTs, eig);
  double rho = 0.0;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
    c.gp[e] = z[e];
    rho = fma(c.gr[e], z[e], rho);
  }
  rho = gs.sum(rho);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    S->rho = rho;
    S->mode = kDCg;
  }
}

template <int RM>
__global__ void __launch_bounds__(kThreads, 1) k_pcg_dist_init(const PcgArgs A, const PcgShared shc) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double bcast[2];
  const PcgShared& sh = shc;
  const int d = sh.d;
  double* Ps = sm;
  double* VTs = Ps + sh.order * RM * RM;
  double* red = VTs + sh.order * RM * RM;
  const DvCtx c = dv_ctx(A, d);
  GridSum gs{c.gpart0, red, bcast, A.counter};
  DistState* S = reinterpret_cast<DistState*>(A.rpart);
  const int row0 = min(d, (int)blockIdx.x * sh.rows_per_cta), row1 = min(d, row0 + sh.rows_per_cta);
  int missing = 0;
  for (int e = threadIdx.x; e < d; e += kThreads) missing |= __ldg(A.aug_count + e) == 0;
  if (threadIdx.x < sh.order) missing |= __ldg(A.linv_ok + threadIdx.x) == 0;
  if (__syncthreads_or(missing) || !(A.lambda > 0.0) || !(A.lambda * A.prep[1] <= kMaxLambdaOverMu)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.status[0] = 3;
      A.status[1] = 0;
      S->mode = kDDone;
    }
    return;
  }
  const bool eig = A.prep[2] != 0.0;
  dist_setup<RM>(A, sh, Ps, VTs, eig);
  if (eig) {
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
      double m = 1.0;
      int rem = e;
      for (int n = sh.order - 1; n >= 0; --n) {
        const int j = rem % sh.R[n];
        rem /= sh.R[n];
        m *= fmax(A.evals[(size_t)n * A.linv_stride + j], 0.0);
      }
      c.gdinv[e] = 1.0 / (m + A.lambda);
    }
  }
  double bb = 0.0;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
    const double be = A.b[e];
    c.gr[e] = be;
    c.gx[e] = 0.0;
    bb = fma(be, be, bb);
  }
  bb = gs.sum(bb);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    S->bb = bb;
    S->gn = A.prep[0];
    S->it = 0;
    S->fail = 0;
  }
  if (bb == 0.0) {
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) A.x[e] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.status[0] = 0;
      A.status[1] = 0;
      S->mode = kDDone;
    }
    return;
  }
  if (A.warm_dev ? *A.warm_dev : A.warm) {
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) c.gx[e] = A.x[e];
    if (blockIdx.x == 0 && threadIdx.x == 0) S->mode = kDWarm;
    return;
  }
  dist_start_cg<RM>(A, sh, gs, c, Ps, VTs, eig, row0, row1, S);
}

// this rank's share of q = G src (src: x for the warm start and the final check, else p)
template <int RM>
__global__ void __launch_bounds__(kThreads, 1) k_pcg_dist_mv(const PcgArgs A, const PcgShared shc) {
  extern __shared__ __align__(16) double sm[];
  const PcgShared& sh = shc;
  const DistState* S = reinterpret_cast<const DistState*>(A.rpart);
  const int mode = S->mode;
  if (mode == kDDone) return;
  const int d = sh.d;
  double* red = sm + 2 * sh.order * RM * RM;
  double* acc32 = red + 32;
  const DvCtx c = dv_ctx(A, d);
  const double* src = mode == kDCg ? c.gp : c.gx;
  const int row0 = min(d, (int)blockIdx.x * sh.rows_per_cta), row1 = min(d, row0 + sh.rows_per_cta);
  const unsigned nsl = (unsigned)(sh.u_hi - sh.u_lo);
  if (sh.t32) slice_partials_t32(A, sh, src, acc32, 0u);
  else if (sh.t4) slice_partials_t4<RM>(A, sh, src, acc32, 0u);
  else slice_partials<RM>(A, sh, src);
  (void)nsl;
  __syncthreads();
  grid_barrier(A.counter, gridDim.x);
  if (sh.t32) reduce_rows_t32(A, sh, src, row0, row1 - row0, A.q);
  else if (sh.t4) reduce_rows_t4(A, sh, src, row0, row1 - row0, A.q);
  else reduce_rows<false>(A, sh, src, row0, row1 - row0, A.q);
}

// one CG state transition on the summed q (identical on every rank)
template <int RM>
__global__ void __launch_bounds__(kThreads, 1) k_pcg_dist_step(const PcgArgs A, const PcgShared shc) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double bcast[2];
  const PcgShared& sh = shc;
  DistState* S = reinterpret_cast<DistState*>(A.rpart);
  const int mode = S->mode;
  if (mode == kDDone) return;
  const int d = sh.d;
  double* Ps = sm;
  double* VTs = Ps + sh.order * RM * RM;
  double* red = VTs + sh.order * RM * RM;
  const DvCtx c = dv_ctx(A, d);
  GridSum gs{c.gpart0, red, bcast, A.counter};
  const int row0 = min(d, (int)blockIdx.x * sh.rows_per_cta), row1 = min(d, row0 + sh.rows_per_cta);
  const bool eig = A.prep[2] != 0.0;
  const double bb = S->bb, gnorm = S->gn;
  __syncthreads();  // every thread has read the state before CTA 0 may rewrite it
  gs.sync();
  if (mode == kDWarm) {
    double r0 = 0.0;
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
      const double re = A.b[e] - A.q[e];
      r0 = fma(re, re, r0);
    }
    r0 = gs.sum(r0);
    const bool keep = r0 < bb && isfinite(r0);
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
      if (keep) c.gr[e] = A.b[e] - A.q[e];
      else c.gx[e] = 0.0;
    }
    __syncthreads();
    gs.sync();
    dist_setup<RM>(A, sh, Ps, VTs, eig);
    dist_start_cg<RM>(A, sh, gs, c, Ps, VTs, eig, row0, row1, S);
    return;
  }
  if (mode == kDCheck) {
    double res = 0.0;
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
      const double t = A.b[e] - A.q[e];
      res = fma(t, t, res);
      A.x[e] = c.gx[e];
    }
    res = gs.sum(res);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      int st = S->fail;
      const double scale = gnorm * sqrt(S->xx) + sqrt(bb);
      if (!st && !(res <= A.check_tol * A.check_tol * scale * scale)) st = 1;
      A.status[0] = st;
      A.status[1] = S->it;
      S->mode = kDDone;
    }
    return;
  }
  // kDCg
  const double rho = S->rho;
  int it = S->it;
  double pq = 0.0;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) pq = fma(c.gp[e], A.q[e], pq);
  pq = gs.sum(pq);
  auto to_check = [&](int fail) {
    double xx = 0.0;
    for (int e = row0 + threadIdx.x; e < row1; e += kThreads) xx = fma(c.gx[e], c.gx[e], xx);
    xx = gs.sum(xx);  // its barrier also completes x as the next matvec source
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      S->xx = xx;
      S->fail = fail;
      S->it = it;
      S->mode = kDCheck;
    }
  };
  if (!(pq > 0.0) || !isfinite(pq)) {
    to_check(2);
    return;
  }
  const double alpha = rho / pq;
  double rr = 0.0, xq = 0.0;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) {
    const double re = fma(-alpha, A.q[e], c.gr[e]);
    c.gr[e] = re;
    rr = fma(re, re, rr);
    const double xe = fma(alpha, c.gp[e], c.gx[e]);
    c.gx[e] = xe;
    xq = fma(xe, xe, xq);
  }
  gs.sum2(rr, xq);
  ++it;
  if (rr <= A.tol * A.tol * fmax(bb, gnorm * gnorm * xq) || it >= A.max_iter) {
    to_check(0);
    return;
  }
  dist_setup<RM>(A, sh, Ps, VTs, eig);
  double* z = dist_precond<RM>(sh, gs, c.gr, c, Ps, VTs, eig);
  double rho2 = 0.0;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) rho2 = fma(c.gr[e], z[e], rho2);
  rho2 = gs.sum(rho2);
  const double beta = rho2 / rho;
  for (int e = row0 + threadIdx.x; e < row1; e += kThreads) c.gp[e] = fma(beta, c.gp[e], z[e]);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    S->rho = rho2;
    S->it = it;
  }
}

// ---------------------------------------------------------------------------
// Split-role PCG (order 3, R_3 = 16, m_1 slices < #SMs): the Gram stays in SHARED MEMORY for
// the whole solve. CTA u < m_1 holds slice u_1 = u of the compact (vech) Gram S -- row u_1
// of S, m_2 x 136 values, 148 KB at C2 -- and computes that slice's matvec partials; the
// remaining CTAs ("vector CTAs", 12 at C2) hold r, p, x and the scratch vectors and run the
// CG recurrences, redundantly and bit-identically, each publishing its share of the next
// matvec source (p, or x0 / x) to global memory. Per matvec, three grid barriers: source
// published -> slice partials -> own-row sums (all CTAs) -> q read by the vector CTAs.
// The slices are read from shared memory instead of streaming 38 MB of blocks from L2 per
// iteration (k_pcg's slice phase). Matvec source selector `ctl` (first vector CTA):
// 1 = CG step / warm start, 2 = final residual check, 0 = done.
struct PcgSplitArgs {
  const double* S;   // compact Gram [m1][m2 * 136]
  double* pg;        // [d] published matvec source
  int* ctl;
};

// slice partials from the shared-memory slice Bp (m2 x 136): warp w takes a contiguous range
// of the slice's row-major (i2 <= j2) blocks; along a row i2 the sources p_b(i2), p_a(i2)
// stay in registers and the targets q_a(i2), q_b(i2) accumulate in registers; the
// transposed targets q_a(j2), q_b(j2) go to the warp's shared accumulators.
// lane l: block row r = l & 15, columns c = 8 (l >> 4) + k, k < 8.
__device__ void split_slice(const PcgShared& sh, const double* Bp, const double* pa,
                            const double* pb, bool two_sides, double* accw, int m2,
                            const int (&off)[8]) {
  const int R2 = sh.R[1], dp = sh.dprime;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane & 15, h = lane >> 4;
  double* acc = accw + (size_t)w * 2 * dp;
  const int blo = (m2 * w) / kWarps, bhi = (m2 * (w + 1)) / kWarps;
  if (blo >= bhi) return;
  int i2, j2;
  pair_of(blo, R2, i2, j2);
  double xb_i[8], xa_i[8];  // p_b(i2), p_a(i2) at this lane's columns
  double y0 = 0.0, y2 = 0.0;  // q_a(i2)[r], q_b(i2)[r] (this lane's column half)
  auto load_row = [&]() {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      xb_i[k] = pb[i2 * 16 + 8 * h + k];
      xa_i[k] = two_sides ? pa[i2 * 16 + 8 * h + k] : 0.0;
    }
  };
  auto flush_row = [&]() {
    y0 += __shfl_xor_sync(0xffffffffu, y0, 16);
    y2 += __shfl_xor_sync(0xffffffffu, y2, 16);
    if (h == 0) {
      acc[i2 * 16 + r] += y0;
      if (two_sides) acc[dp + i2 * 16 + r] += y2;
    }
    __syncwarp();
    y0 = y2 = 0.0;
  };
  load_row();
  for (int u = blo; u < bhi; ++u) {
    const double* Bu = Bp + (size_t)u * 136;
    double m[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = Bu[off[k]];
    const double* xbj = pb + j2 * 16 + 8 * h;
    const double* xaj = pa + j2 * 16 + 8 * h;
    double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      const double2 vb = *reinterpret_cast<const double2*>(xbj + k);
      t0 = fma(m[k], vb.x, t0);
      t0 = fma(m[k + 1], vb.y, t0);
      t1 = fma(m[k], xb_i[k], t1);
      t1 = fma(m[k + 1], xb_i[k + 1], t1);
      if (two_sides) {
        const double2 va = *reinterpret_cast<const double2*>(xaj + k);
        t2 = fma(m[k], va.x, t2);
        t2 = fma(m[k + 1], va.y, t2);
        t3 = fma(m[k], xa_i[k], t3);
        t3 = fma(m[k + 1], xa_i[k + 1], t3);
      }
    }
    y0 += t0;  // q_a(i2) += M p_b(j2)
    y2 += t2;  // q_b(i2) += M p_a(j2)
    if (j2 != i2) {  // q_a(j2) += M p_b(i2), q_b(j2) += M p_a(i2)
      t1 += __shfl_xor_sync(0xffffffffu, t1, 16);
      t3 += __shfl_xor_sync(0xffffffffu, t3, 16);
      if (h == 0) {
        acc[j2 * 16 + r] += t1;
        if (two_sides) acc[dp + j2 * 16 + r] += t3;
      }
      __syncwarp();
    }
    // next block (row-major upper triangle)
    if (u + 1 < bhi) {
      if (++j2 == R2) {
        flush_row();
        ++i2;
        j2 = i2;
        load_row();
      }
    }
  }
  flush_row();
}

// The same slice matvec on the FP64 tensor cores: per block, C (16 x 8) += M (16 x 16) B with
// B's columns the four sources p_b(j2), p_b(i2), p_a(j2), p_a(i2) (columns 4-7 zero), one
// m16n8k16 DMMA. Columns 0 / 2 (targets q_a(i2), q_b(i2)) accumulate in the C registers
// along a row of blocks; columns 1 / 3 (q_a(j2), q_b(j2)) are added to the warp's shared
// accumulators after each off-diagonal block and reset. offA: this lane's packed offsets of
// its A-fragment entries M[g + 8 (v & 1)][t + 4 (v >> 1)].
__device__ void split_slice_dmma(const PcgShared& sh, const double* __restrict__ Bp,
                                 const double* __restrict__ pa, const double* __restrict__ pb,
                                 bool two_sides, double* __restrict__ accw, int m2,
                                 const int (&offA)[8]) {
  const int R2 = sh.R[1], dp = sh.dprime;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double* acc = accw + (size_t)w * 2 * dp;
  const int blo = (m2 * w) / kWarps, bhi = (m2 * (w + 1)) / kWarps;
  if (blo >= bhi) return;
  int i2, j2;
  pair_of(blo, R2, i2, j2);
  // B column g (< 4) of this lane: which source, and whether it is the row's (i2) block
  const bool srcb = g < 2, src_i = (g & 1) != 0;
  const bool bcol = g < 4 && (srcb || two_sides);
  const double* sbase = srcb ? pb : pa;
  const bool tgt = t < 2 && (t == 0 || two_sides);  // lanes t = 0 / 1: side-0 / side-1 targets
  double c[4] = {0.0, 0.0, 0.0, 0.0};
  double a[8], b[4];
  auto load = [&](int u, int ii, int jj) {  // operands of block u = (ii, jj)
    const double* Bu = Bp + (size_t)u * 136;
#pragma unroll
    for (int v = 0; v < 8; ++v) a[v] = Bu[offA[v]];
    const double* src = sbase + (src_i ? ii : jj) * 16;
#pragma unroll
    for (int v = 0; v < 4; ++v) b[v] = bcol ? src[t + 4 * v] : 0.0;
  };
  load(blo, i2, j2);
  for (int u = blo; u < bhi; ++u) {
    dmma_16x8x16(c, a, b);
    // next block's operands while this one's DMMAs run (the shared loads do not alias acc)
    int ni = i2, nj = j2 + 1;
    if (nj == R2) {
      ++ni;
      nj = ni;
    }
    if (u + 1 < bhi) load(u + 1, ni, nj);
    const double t1 = c[1], t3 = c[3];
    c[1] = c[3] = 0.0;
    if (j2 != i2 && tgt) {  // columns 1 / 3: q_side(j2)
      double* q = acc + t * dp + j2 * 16;
      q[g] += t1;
      q[g + 8] += t3;
    }
    if (ni != i2 || u + 1 == bhi) {  // row done: columns 0 / 2: q_side(i2)
      if (tgt) {
        double* q = acc + t * dp + i2 * 16;
        q[g] += c[0];
        q[g + 8] += c[2];
      }
      c[0] = c[2] = 0.0;
    }
    i2 = ni;
    j2 = nj;
  }
}

template <int RX>
__global__ void __launch_bounds__(kThreads, 1) k_pcg_split(const PcgArgs A, const PcgShared shc,
                                                          const PcgSplitArgs X) {
  extern __shared__ __align__(16) double sm[];
  const PcgShared& sh = shc;
  const int d = sh.d, dp = sh.dprime;
  const int dv = (d + 1) & ~1;
  const int m1 = sh.m1, m2 = sh.m[1];
  const bool slice_cta = (int)blockIdx.x < m1;
  const int nvec = (int)gridDim.x - m1, vid = (int)blockIdx.x - m1;
  const int tid = threadIdx.x;
  constexpr int RM = 16;

  // applicability (every CTA decides the same)
  int missing = 0;
  for (int e = tid; e < d; e += kThreads) missing |= __ldg(A.aug_count + e) == 0;
  if (tid < sh.order) missing |= __ldg(A.linv_ok + tid) == 0;
  const double pnorm = A.prep[1];
  if (__syncthreads_or(missing) || !(A.lambda > 0.0) || !(A.lambda * pnorm <= kMaxLambdaOverMu)) {
    if (blockIdx.x == 0 && tid == 0) {
      A.status[0] = 3;
      A.status[1] = 0;
    }
    return;
  }
  const int row0 = min(d, (int)blockIdx.x * sh.rows_per_cta);
  const int nrows = min(d, row0 + sh.rows_per_cta) - row0;
  unsigned sync_target = 0;
  auto gsync = [&]() {
    sync_target += gridDim.x;
    grid_barrier(A.counter, sync_target);
  };
  // own rows: q[e] = sum over the slices' partials + augmented diagonal * source[e]
  // 16 lanes per row, one slice partial each (R_1 <= 16), summed by a fixed shuffle tree
  auto reduce_own = [&]() {
    const int R1 = sh.R[0];
    const int j1 = tid & 15;
    for (int base = row0; base < row0 + nrows; base += kThreads / 16) {
      const int e = base + (tid >> 4);
      const bool ok = e < row0 + nrows;
      double s = 0.0;
      if (ok && j1 < R1) {
        const int i1 = e / dp, rest = e - i1 * dp;
        const int u1 = upper_pair(min(i1, j1), max(i1, j1), R1);
        const int side = i1 <= j1 ? 0 : 1;
        s = __ldcg(A.part + ((size_t)u1 * 2 + side) * dp + rest);
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (ok && j1 == 0) {
        const int c = __ldg(A.aug_count + e);
        if (c > 0) s = fma((double)c * A.aug_term, __ldcg(X.pg + e), s);
        A.q[e] = s;
      }
    }
  };

  if (slice_cta) {
    // ---------------- slice CTA ----------------
    double* Bp = sm;                                   // [m2][136]
    double* pa = Bp + (size_t)m2 * 136;                // [dp]
    double* pb = pa + dp;                              // [dp]
    double* accw = pb + dp;                            // [kWarps][2][dp]
    const int u1 = blockIdx.x;
    int a, b;
    pair_of(u1, sh.R[0], a, b);
    const bool two = a != b;
    {
      const double2* src = reinterpret_cast<const double2*>(X.S + (size_t)u1 * m2 * 136);
      double2* dst = reinterpret_cast<double2*>(Bp);
      for (int e = tid; e < m2 * 68; e += kThreads) dst[e] = __ldg(src + e);
    }
    const int lane = tid & 31;
    int off[8];
    static constexpr bool kDmmaSlice = true;
    if (kDmmaSlice) {
      const int g = lane >> 2, t = lane & 3;
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int rr = g + 8 * (v & 1), cc = t + 4 * (v >> 1);
        off[v] = upper_pair(min(rr, cc), max(rr, cc), 16);
      }
    } else {
      const int r = lane & 15, h = lane >> 4;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = 8 * h + k;
        off[k] = upper_pair(min(r, c), max(r, c), 16);
      }
    }
    for (;;) {
      gsync();  // source published
      if (__ldcg(X.ctl) == 0) break;
      for (int e = tid; e < dp; e += kThreads) {
        pa[e] = __ldcg(X.pg + (size_t)a * dp + e);
        pb[e] = __ldcg(X.pg + (size_t)b * dp + e);
      }
      for (int e = tid; e < kWarps * 2 * dp; e += kThreads) accw[e] = 0.0;
      __syncthreads();
      const bool pf = A.prof && blockIdx.x == 0 && tid == 0;
      const unsigned long long ts0 = pf ? gtimer() : 0;
      if (kDmmaSlice) split_slice_dmma(sh, Bp, pa, pb, two, accw, m2, off);
      else split_slice(sh, Bp, pa, pb, two, accw, m2, off);
      __syncthreads();
      if (pf) A.prof[4] += gtimer() - ts0;
      for (int e = tid; e < 2 * dp; e += kThreads) {
        const int side = e >= dp;
        if (side && !two) continue;
        double s = 0.0;
        for (int w = 0; w < kWarps; ++w) s += accw[(size_t)w * 2 * dp + e];
        A.part[((size_t)u1 * 2 + side) * dp + (e - side * dp)] = s;
      }
      gsync();  // partials
      reduce_own();
      gsync();  // q
    }
    return;
  }

  // ---------------- vector CTA ----------------
  double* Ps = sm;                          // [order][RM][RM]
  double* VTs = Ps + sh.order * RM * RM;
  double* dinv = VTs + sh.order * RM * RM;
  double* r = dinv + dv;
  double* p = r + dv;
  double* s0 = p + dv;
  double* s1 = s0 + dv;
  double* xs = s1 + dv;
  double* red = xs + dv;
  double* Wf = red + 64;                    // [kWfDoubles] (precondition16's fragment tables)
  const int sh0 = (int)((long long)d * vid / nvec), sh1 = (int)((long long)d * (vid + 1) / nvec);
  auto publish = [&](const double* v, int c) {  // my share of the next matvec source
    for (int e = sh0 + tid; e < sh1; e += kThreads) X.pg[e] = v[e];
    if (vid == 0 && tid == 0) *X.ctl = c;
  };
  for (int n = 0; n < sh.order; ++n) {
    const int R = sh.R[n];
    const double* Pg = A.pinv + (size_t)n * A.linv_stride;
    for (int e = tid; e < RM * RM; e += kThreads) {
      const int i = e / RM, j = e - i * RM;
      Ps[n * RM * RM + e] = (i < R && j < R) ? Pg[i * R + j] : 0.0;
    }
  }
  __syncthreads();
  const double gnorm = A.prep[0];
  const bool eig = A.prep[2] != 0.0;
  if (eig) {
    for (int n = 0; n < sh.order; ++n) {
      const int R = sh.R[n];
      const double* Vg = A.evecs + (size_t)n * A.linv_stride;
      for (int e = tid; e < RM * RM; e += kThreads) {
        const int i = e / RM, j = e - i * RM;
        const bool in = i < R && j < R;
        Ps[n * RM * RM + e] = in ? Vg[i * R + j] : 0.0;
        VTs[n * RM * RM + e] = in ? Vg[j * R + i] : 0.0;
      }
    }
    for (int e = tid; e < d; e += kThreads) {
      double m = 1.0;
      int rem = e;
      for (int n = sh.order - 1; n >= 0; --n) {
        const int j = rem % sh.R[n];
        rem /= sh.R[n];
        m *= fmax(A.evals[(size_t)n * A.linv_stride + j], 0.0);
      }
      dinv[e] = 1.0 / (m + A.lambda);
    }
    __syncthreads();
  }
  bool pre16 = false;
  if constexpr (RX == 16) pre16 = sh.order == 3 && sh.R[0] == 16;
  if (pre16) build_frags16(Ps, VTs, Wf);
  for (int e = tid; e < d; e += kThreads) {
    r[e] = A.b[e];
    xs[e] = 0.0;
  }
  __syncthreads();
  double bb = 0.0;
  for (int e = tid; e < d; e += kThreads) bb = fma(r[e], r[e], bb);
  bb = block_sum_det(bb, red);
  const double tol2 = A.tol * A.tol;
  // z from precond() is canonical, or in the pre16_swz layout on the 16 x 16 x 16 path
  auto zi = [&](int e) { return pre16 ? pre16_swz(e) : e; };
  enum { kWarm, kCg, kCheck };
  int mode = kCg, it = 0, fail = 0;
  double rho = 0.0, xx = 0.0;
  auto precond = [&]() -> double* {
    if (pre16)
      return precondition16(r, s0, s1, Wf, dinv, eig,
                            (A.prof && vid == 0 && tid == 0) ? A.prof : nullptr);
    return precondition<RM, RX>(sh, r, s0, s1, Ps, VTs, dinv, eig);
  };
  auto start_cg = [&]() {  // z = M^-1 r, p = z, rho; publish p
    double* z = precond();
    double rh = 0.0;
    for (int e = tid; e < d; e += kThreads) {
      const double ze = z[zi(e)];
      p[e] = ze;
      rh = fma(r[e], ze, rh);
    }
    rho = block_sum_det(rh, red);
    publish(p, 1);
    mode = kCg;
  };
  auto start_check = [&]() {  // final residual check: matvec with x
    double t = 0.0;
    for (int e = tid; e < d; e += kThreads) t = fma(xs[e], xs[e], t);
    xx = block_sum_det(t, red);
    publish(xs, 2);
    mode = kCheck;
  };
  if (bb == 0.0) {
    for (int e = sh0 + tid; e < sh1; e += kThreads) A.x[e] = 0.0;
    if (vid == 0 && tid == 0) {
      A.status[0] = 0;
      A.status[1] = 0;
    }
    publish(xs, 0);
  } else if (A.warm_dev ? *A.warm_dev : A.warm) {
    for (int e = tid; e < d; e += kThreads) xs[e] = A.x[e];
    __syncthreads();
    publish(xs, 1);
    mode = kWarm;
  } else {
    start_cg();
  }
  const bool pf = A.prof && vid == 0 && tid == 0;
  unsigned long long tv = pf ? gtimer() : 0;
  auto mark = [&](int k) {
    if (pf) {
      const unsigned long long t1 = gtimer();
      A.prof[k] += t1 - tv;
      tv = t1;
    }
  };
  for (;;) {
    mark(3);
    gsync();  // source published
    mark(0);
    if (__ldcg(X.ctl) == 0) break;
    gsync();  // partials
    mark(1);
    reduce_own();
    gsync();  // q
    mark(2);
    if (mode == kWarm) {
      double r0 = 0.0;
      for (int e = tid; e < d; e += kThreads) {
        const double re = A.b[e] - __ldcg(A.q + e);
        s0[e] = re;
        r0 = fma(re, re, r0);
      }
      r0 = block_sum_det(r0, red);
      if (r0 < bb && isfinite(r0)) {
        for (int e = tid; e < d; e += kThreads) r[e] = s0[e];
      } else {
        for (int e = tid; e < d; e += kThreads) xs[e] = 0.0;
      }
      __syncthreads();
      start_cg();
    } else if (mode == kCg) {
      double pq = 0.0;
      for (int e = tid; e < d; e += kThreads) {
        const double qe = __ldcg(A.q + e);
        s0[e] = qe;
        pq = fma(p[e], qe, pq);
      }
      pq = block_sum_det(pq, red);
      mark(8);
      if (!(pq > 0.0) || !isfinite(pq)) {
        fail = 2;
        start_check();
        continue;
      }
      const double alpha = rho / pq;
      double rr = 0.0, xq = 0.0;
      for (int e = tid; e < d; e += kThreads) {
        const double re = fma(-alpha, s0[e], r[e]);
        r[e] = re;
        rr = fma(re, re, rr);
        const double xe = fma(alpha, p[e], xs[e]);
        xs[e] = xe;
        xq = fma(xe, xe, xq);
      }
      block_sum2_det(rr, xq, red);
      mark(9);
      ++it;
      if (rr <= tol2 * fmax(bb, gnorm * gnorm * xq) || it >= A.max_iter) {
        start_check();
        continue;
      }
      double* z = precond();
      mark(10);
      double rho2 = 0.0;
      for (int e = tid; e < d; e += kThreads) rho2 = fma(r[e], z[zi(e)], rho2);
      rho2 = block_sum_det(rho2, red);
      mark(11);
      const double beta = rho2 / rho;
      rho = rho2;
      for (int e = tid; e < d; e += kThreads) p[e] = fma(beta, p[e], z[zi(e)]);
      __syncthreads();
      publish(p, 1);
      mark(5);
    } else {  // kCheck: q = G x
      for (int e = sh0 + tid; e < sh1; e += kThreads) A.x[e] = xs[e];
      if (vid == 0) {
        double res = 0.0;
        for (int e = tid; e < d; e += kThreads) {
          const double t = A.b[e] - __ldcg(A.q + e);
          res = fma(t, t, res);
        }
        res = block_sum_det(res, red);
        if (tid == 0) {
          int st = fail;
          const double scale = gnorm * sqrt(xx) + sqrt(bb);
          if (!st && !(res <= A.check_tol * A.check_tol * scale * scale)) st = 1;
          A.status[0] = st;
          A.status[1] = it;
        }
      }
      publish(xs, 0);
    }
  }
}

int num_sms() {
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : kNumSMs;
  }();
  return sms;
}

int rank_bucket(int order, const int* ranks) {
  int rmax = 0;
  for (int n = 0; n < order; ++n) rmax = ranks[n] > rmax ? ranks[n] : rmax;
  return rmax <= 8 ? 8 : rmax <= 16 ? 16 : rmax <= 32 ? 32 : 0;
}

size_t pcg_smem(int d, int order, const int* ranks, int rm) {
  const size_t dv = (size_t)((d + 1) & ~1);
  size_t extra = 0;  // (P_n blocks: order * rm^2)
  if (order == 3 && ranks[2] == 16) {
    const size_t need = (size_t)kWarps * 2 * (d / ranks[0]);
    if (need > 2 * dv) extra = need;
  }
  return 8 * (2 * (size_t)order * rm * rm + 6 * dv + 32 + extra);
}

PcgShared pcg_shape(const PcgSpec& spec) {
  PcgShared sh{};
  sh.d = spec.d;
  sh.order = spec.order;
  for (int n = spec.order - 1; n >= 0; --n) {
    sh.R[n] = spec.ranks[n];
    sh.m[n] = spec.ranks[n] * (spec.ranks[n] + 1) / 2;
  }
  return sh;
}

}  // namespace

void pcg_prepare(const PcgSpec& spec, double* prep_dev, int* skip_dev, cudaStream_t st) {
  k_pcg_prep<<<1, 64 * spec.order, 0, st>>>(spec.grams, spec.pinv, spec.linv_stride,
                                            pcg_shape(spec), spec.lambda, prep_dev, skip_dev);
  RTB_LAUNCH_CHECK();
}

size_t pcg_work_bytes(int d, int r1) {
  const size_t m1 = (size_t)r1 * (r1 + 1) / 2;
  const size_t dp = (size_t)d / r1;
  return ((size_t)d + m1 * 2 * dp + 1024) * 8 + 256;
}

// large d: the six d-vectors leave shared memory for per-CTA global slices
static bool pcg_big(int d, int order, const int* ranks) {
  const int rm = rank_bucket(order, ranks);
  return rm > 0 && pcg_smem(d, order, ranks, rm) > 220 * 1024;
}
static size_t pcg_smem_big(int order, int rm) { return 8 * (2 * (size_t)order * rm * rm + 32); }

// tiled order-4 matvec (slice_partials_t4, k_pcg_dv only): the warp's sources and targets
// (8 R3 R4 doubles) in shared memory, R4 <= 32
static bool pcg_t4(int d, int order, const int* ranks) {
  static const bool off = std::getenv("RTB_NO_PCG_T4") != nullptr;  // experiments
  return !off && order == 4 && ranks[3] <= 16 && ranks[2] * ranks[3] <= 128 &&
         (size_t)kWarps * 8 * ranks[2] * ranks[3] * 8 <= 160 * 1024 && pcg_big(d, order, ranks);
}

// tiled rank-32 matvec (slice_partials_t32): large d, order 3, R_3 = 32, R_2 a multiple of 8
static bool pcg_t32(int d, int order, const int* ranks) {
  static const bool off = std::getenv("RTB_NO_PCG_T32") != nullptr;  // experiments
  return !off && order == 3 && ranks[2] == 32 && ranks[1] % 8 == 0 && pcg_big(d, order, ranks);
}
static int t32_ntile(const int* ranks) {
  const int ng = ranks[1] / 8;
  return ng * (ng + 1) / 2;
}

// chunks per slice of the generic matvec: about three work units per SM (fast3: 1)
static int pcg_jc(int d, int order, const int* ranks) {
  const bool fast3 = order == 3 && ranks[2] == 16 && !pcg_big(d, order, ranks);
  if (fast3) return 1;
  const int m1 = ranks[0] * (ranks[0] + 1) / 2;
  int mid = 1;
  for (int n = 1; n < order - 1; ++n) mid *= ranks[n];
  const int jc = (3 * num_sms() + m1 - 1) / m1;
  return std::max(1, std::min(jc, mid));
}

// q, partials [m1][jc][2][d'], residual partials, counter
static size_t pcg_base_bytes(int d, int order, const int* ranks) {
  const size_t m1 = (size_t)ranks[0] * (ranks[0] + 1) / 2;
  const size_t dp = (size_t)d / ranks[0];
  const size_t part = pcg_t32(d, order, ranks) ? m1 * t32_ntile(ranks) * 1024
                    : pcg_t4(d, order, ranks)
                        ? m1 * ((size_t)ranks[1] * (ranks[1] + 1) / 2) * kT4H * 4 * ranks[2] * ranks[3]
                        : m1 * pcg_jc(d, order, ranks) * 2 * dp;
  return ((size_t)d + part + 1024) * 8 + 256 +
         ((size_t)d + 32) * 8;  // + the split form's published source and selector
}

size_t pcg_work_bytes(int d, int order, const int* ranks) {
  size_t b = pcg_base_bytes(d, order, ranks);
  if (pcg_big(d, order, ranks)) b = ((b + 255) & ~size_t(255)) + (size_t)num_sms() * 6 * ((d + 1) & ~1) * 8 + 256;
  return b;
}

bool pcg_supported(int d, int order, const int* ranks) {
  const int rm = rank_bucket(order, ranks);
  return d >= 1 && d <= (1 << 20) && order >= 2 && order <= kMaxOrder && rm > 0;
}

// shape, workspace carving and launch arguments shared by pcg_solve and pcg_solve_dist
static void pcg_setup(const PcgSpec& spec, const double* blocks, const double* b, double* x,
                      void* work, int* status_dev, PcgShared& sh, PcgArgs& a, size_t& smem,
                      bool& big, int& rm) {
  const int d = spec.d;
  const int grid = num_sms();
  if (!pcg_supported(d, spec.order, spec.ranks)) throw Error(4, "pcg_solve: unsupported shape");
  sh = PcgShared{};
  sh.d = d;
  sh.order = spec.order;
  sh.rows_per_cta = (d + grid - 1) / grid;
  int inner = 1;
  for (int n = spec.order - 1; n >= 0; --n) {
    sh.R[n] = spec.ranks[n];
    sh.m[n] = spec.ranks[n] * (spec.ranks[n] + 1) / 2;
    sh.J[n] = inner;
    inner *= spec.ranks[n];
  }
  if (inner != d) throw Error(1, "pcg_solve: prod(ranks) != d");
  sh.dprime = d / sh.R[0];
  sh.last = sh.R[spec.order - 1];
  sh.mid = sh.dprime / sh.last;
  sh.mmid = 1;
  for (int n = 1; n < spec.order - 1; ++n) sh.mmid *= sh.m[n];
  sh.m1 = sh.m[0];
  sh.u_lo = 0;
  sh.u_hi = sh.m1;
  sh.aug_on = 1;
  sh.jc = pcg_jc(d, spec.order, spec.ranks);
  rm = rank_bucket(spec.order, spec.ranks);
  big = pcg_big(d, spec.order, spec.ranks);
  sh.t32 = pcg_t32(d, spec.order, spec.ranks) ? 1 : 0;
  static const bool no_dv_t4 = std::getenv("RTB_NO_PCG_DV") != nullptr;
  sh.t4 = (!no_dv_t4 && pcg_t4(d, spec.order, spec.ranks)) ? 1 : 0;
  sh.t4h = kT4H;
  sh.ng = spec.ranks[1] / 8;
  sh.ntile = t32_ntile(spec.ranks);
  smem = big ? pcg_smem_big(spec.order, rm) + (sh.t32 ? (size_t)kWarps * 1024 * 8 : 0) +
                                (sh.t4 ? (size_t)kWarps * 8 * spec.ranks[2] * spec.ranks[3] * 8 : 0)
                          : pcg_smem(d, spec.order, spec.ranks, rm);

  char* w = static_cast<char*>(work);
  a = PcgArgs{};
  a.B = blocks;
  a.b = b;
  a.x = x;
  a.q = reinterpret_cast<double*>(w);
  a.part = a.q + d;
  a.rpart = a.part + (sh.t32 ? (size_t)sh.m1 * sh.ntile * 1024
                      : sh.t4 ? (size_t)sh.m1 * sh.m[1] * kT4H * 4 * spec.ranks[2] * spec.ranks[3]
                              : (size_t)sh.m1 * sh.jc * 2 * sh.dprime);
  a.counter = reinterpret_cast<unsigned*>(a.rpart + 1024);
  a.vglobal = nullptr;
  if (big) {  // after the counter block (pcg_work_bytes(d, order, ranks))
    const size_t off = ((pcg_base_bytes(d, spec.order, spec.ranks) + 255) & ~size_t(255));
    a.vglobal = reinterpret_cast<double*>(w + off);
  }
  a.status = status_dev;
  a.pinv = spec.pinv;
  a.linv_stride = spec.linv_stride;
  a.linv_ok = spec.linv_ok;
  a.grams = spec.grams;
  a.evals = spec.evals;
  a.evecs = spec.evecs;
  a.prep = spec.prep;
  a.aug_count = spec.aug_count;
  a.aug_term = spec.aug_term;
  a.lambda = spec.lambda;
  a.max_iter = spec.max_iter;
  a.tol = spec.tol;
  a.check_tol = spec.check_tol;
  a.warm = spec.warm;
  a.warm_dev = spec.warm_dev;
}

void pcg_solve(const PcgSpec& spec, const double* blocks, const double* b, double* x, void* work,
               int* status_dev, cudaStream_t st) {
  const int d = spec.d;
  const int grid = num_sms();
  PcgShared sh;
  PcgArgs a;
  size_t smem = 0;
  bool big = false;
  int rm = 0;
  pcg_setup(spec, blocks, b, x, work, status_dev, sh, a, smem, big, rm);
  static unsigned long long* prof_buf = nullptr;
  static const bool prof_on = std::getenv("RTB_PCG_PROF") != nullptr;
  if (prof_on) {
    if (!prof_buf) RTB_CUDA(cudaMalloc(&prof_buf, 16 * 8));
    RTB_CUDA(cudaMemsetAsync(prof_buf, 0, 16 * 8, st));
    a.prof = prof_buf;
  }
  RTB_CUDA(cudaMemsetAsync(a.counter, 0, 64, st));
  bool all16 = true;
  for (int n = 0; n < spec.order; ++n) all16 &= spec.ranks[n] == 16;
  static const bool no_dv = std::getenv("RTB_NO_PCG_DV") != nullptr;  // experiments
  void* fn = big ? (no_dv ? (rm == 8 ? (void*)k_pcg<8, 0, true>
                                     : rm == 16 ? (void*)k_pcg<16, 0, true> : (void*)k_pcg<32, 0, true>)
                          : (rm == 8 ? (void*)k_pcg_dv<8>
                                     : rm == 16 ? (void*)k_pcg_dv<16> : (void*)k_pcg_dv<32>))
           : all16 ? (void*)k_pcg<16, 16, false>
           : rm == 8 ? (void*)k_pcg<8, 0, false>
           : rm == 16 ? (void*)k_pcg<16, 0, false> : (void*)k_pcg<32, 0, false>;
  set_max_smem_impl(fn, 220 * 1024);
  void* args[] = {(void*)&a, (void*)&sh};
  RTB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, smem, st));
  RTB_LAUNCH_CHECK();
  if (!big && all16) count_variant("k_pcg<16,16>");
  if (sh.t32) count_variant("k_pcg_t32");
  if (big && !no_dv) count_variant("k_pcg_dv");
  if (sh.t4) count_variant("k_pcg_t4");
  if (prof_on) {
    unsigned long long h[16];
    int stat[2];
    RTB_CUDA(cudaMemcpyAsync(h, prof_buf, 128, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaMemcpyAsync(stat, status_dev, 8, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr,
                 "[pcg] d=%d iters=%d status=%d ns: slice %llu bar1 %llu reduce %llu bar2 %llu "
                 "vec %llu precond %llu tail %llu | stages %llu %llu %llu | gnorm %.3e pnorm %.3e\n",
                 d, stat[1], stat[0], h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[8], h[9], h[10],
                 __builtin_bit_cast(double, h[14]), __builtin_bit_cast(double, h[15]));
  }
}


bool pcg_dist_ok(int d, int order, const int* ranks) {
  static const bool off = std::getenv("RTB_NO_PCG_DIST") != nullptr;  // experiments
  return !off && pcg_supported(d, order, ranks) && pcg_big(d, order, ranks);
}

void pcg_dist_slices(int m1, int rank, int count, int* u_lo, int* u_hi) {
  *u_lo = (int)((long long)m1 * rank / count);
  *u_hi = (int)((long long)m1 * (rank + 1) / count);
}

void pcg_solve_dist(const PcgSpec& spec, const double* blocks_local, int rank, int count,
                    const double* b, double* x, void* work, int* status_dev, cudaStream_t st,
                    const std::function<void(double*, size_t)>& allreduce) {
  if (!pcg_dist_ok(spec.d, spec.order, spec.ranks)) throw Error(4, "pcg_solve_dist: unsupported shape");
  const int d = spec.d;
  const int grid = num_sms();
  PcgShared sh;
  PcgArgs a;
  size_t smem = 0;
  bool big = false;
  int rm = 0;
  pcg_setup(spec, blocks_local, b, x, work, status_dev, sh, a, smem, big, rm);
  pcg_dist_slices(sh.m1, rank, count, &sh.u_lo, &sh.u_hi);
  sh.aug_on = rank == 0 ? 1 : 0;
  void *fi, *fm, *fs;
  if (rm == 8) {
    fi = (void*)k_pcg_dist_init<8>; fm = (void*)k_pcg_dist_mv<8>; fs = (void*)k_pcg_dist_step<8>;
  } else if (rm == 16) {
    fi = (void*)k_pcg_dist_init<16>; fm = (void*)k_pcg_dist_mv<16>; fs = (void*)k_pcg_dist_step<16>;
  } else {
    fi = (void*)k_pcg_dist_init<32>; fm = (void*)k_pcg_dist_mv<32>; fs = (void*)k_pcg_dist_step<32>;
  }
  for (void* f : {fi, fm, fs}) set_max_smem_impl(f, 220 * 1024);
  void* args[] = {(void*)&a, (void*)&sh};
  auto launch = [&](void* f) {
    RTB_CUDA(cudaMemsetAsync(a.counter, 0, 64, st));  // barrier counter and matvec tickets
    RTB_CUDA(cudaLaunchCooperativeKernel(f, dim3(grid), dim3(kThreads), args, smem, st));
    RTB_LAUNCH_CHECK();
  };
  launch(fi);
  // the CG state is on the device: the host polls its mode every few iterations (a pinned
  // slot of this call's own: shards may run in threads of one process)
  struct Slot {
    int* p = pinned_slot();
    ~Slot() { pinned_slot_free(p); }
  } slot;
  int* done_host = slot.p;
  const int* mode_dev = &reinterpret_cast<const DistState*>(a.rpart)->mode;
  const int max_steps = spec.max_iter + 3;  // warm start + iterations + final check
  for (int k = 0; k < max_steps; ++k) {
    launch(fm);
    allreduce(a.q, (size_t)d);
    launch(fs);
    if (k >= 6 && (k % 3 == 0 || k == max_steps - 1)) {
      RTB_CUDA(cudaMemcpyAsync(done_host, mode_dev, 4, cudaMemcpyDeviceToHost, st));
      RTB_CUDA(cudaStreamSynchronize(st));
      if (*done_host == kDDone) break;
    }
  }
  count_variant("k_pcg_dist");
  static const bool prof_on = std::getenv("RTB_PCG_PROF") != nullptr;
  if (prof_on) {
    int stat[2];
    DistState S;
    RTB_CUDA(cudaMemcpyAsync(stat, status_dev, 8, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaMemcpyAsync(&S, a.rpart, sizeof(S), cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr, "[pcg_dist] rank %d/%d slices [%d,%d) d=%d status=%d iters=%d mode=%d "
                 "bb=%.3e xx=%.3e rho=%.3e\n", rank, count, sh.u_lo, sh.u_hi, d, stat[0], stat[1],
                 S.mode, S.bb, S.xx, S.rho);
  }
}

static size_t split_slice_smem(int d, const int* ranks) {
  const size_t m2 = (size_t)ranks[1] * (ranks[1] + 1) / 2, dp = (size_t)d / ranks[0];
  return (m2 * 136 + 2 * dp + (size_t)kWarps * 2 * dp) * 8;
}
static size_t split_vector_smem(int d, int order) {
  return ((size_t)2 * order * 16 * 16 + 6 * (size_t)((d + 1) & ~1) + 64 + kWfDoubles) * 8;
}

bool pcg_split_ok(int d, int order, const int* ranks) {
  static const bool off = std::getenv("RTB_NO_PCG_SPLIT") != nullptr;
  if (off || order != 3 || ranks[2] != 16 || ranks[0] > 16 || ranks[1] > 16) return false;
  if (!pcg_supported(d, order, ranks) || pcg_big(d, order, ranks)) return false;
  const int m1 = ranks[0] * (ranks[0] + 1) / 2;
  if (m1 + 4 > num_sms()) return false;
  return std::max(split_slice_smem(d, ranks), split_vector_smem(d, order)) <= 227 * 1024 - 1024;
}

void pcg_solve_compact(const PcgSpec& spec, const double* S, const double* b, double* x,
                       void* work, int* status_dev, cudaStream_t st) {
  const int d = spec.d;
  const int grid = num_sms();
  if (!pcg_split_ok(d, spec.order, spec.ranks)) throw Error(4, "pcg_solve_compact: unsupported shape");
  PcgShared sh{};
  sh.d = d;
  sh.order = spec.order;
  sh.rows_per_cta = (d + grid - 1) / grid;
  int inner = 1;
  for (int n = spec.order - 1; n >= 0; --n) {
    sh.R[n] = spec.ranks[n];
    sh.m[n] = spec.ranks[n] * (spec.ranks[n] + 1) / 2;
    sh.J[n] = inner;
    inner *= spec.ranks[n];
  }
  if (inner != d) throw Error(1, "pcg_solve_compact: prod(ranks) != d");
  sh.dprime = d / sh.R[0];
  sh.last = sh.R[spec.order - 1];
  sh.mid = sh.dprime / sh.last;
  sh.mmid = sh.m[1];
  sh.m1 = sh.m[0];
  sh.u_lo = 0;
  sh.u_hi = sh.m1;
  sh.aug_on = 1;
  sh.jc = 1;
  const size_t smem = std::max(split_slice_smem(d, spec.ranks), split_vector_smem(d, spec.order));
  char* w = static_cast<char*>(work);
  PcgArgs a{};
  a.b = b;
  a.x = x;
  a.q = reinterpret_cast<double*>(w);
  a.part = a.q + d;
  a.rpart = a.part + (size_t)sh.m1 * 2 * sh.dprime;
  a.counter = reinterpret_cast<unsigned*>(a.rpart + 1024);
  a.status = status_dev;
  a.pinv = spec.pinv;
  a.linv_stride = spec.linv_stride;
  a.linv_ok = spec.linv_ok;
  a.grams = spec.grams;
  a.evals = spec.evals;
  a.evecs = spec.evecs;
  a.prep = spec.prep;
  a.aug_count = spec.aug_count;
  a.aug_term = spec.aug_term;
  a.lambda = spec.lambda;
  a.max_iter = spec.max_iter;
  a.tol = spec.tol;
  a.check_tol = spec.check_tol;
  a.warm = spec.warm;
  a.warm_dev = spec.warm_dev;
  PcgSplitArgs xa{};
  xa.S = S;
  xa.pg = reinterpret_cast<double*>(reinterpret_cast<char*>(a.counter) + 256);
  xa.ctl = reinterpret_cast<int*>(xa.pg + d);
  RTB_CUDA(cudaMemsetAsync(a.counter, 0, 64, st));
  bool all16 = true;
  for (int n = 0; n < spec.order; ++n) all16 &= spec.ranks[n] == 16;
  void* fn = all16 ? (void*)k_pcg_split<16> : (void*)k_pcg_split<0>;
  set_max_smem_impl(fn, (int)smem);
  static unsigned long long* prof_buf = nullptr;
  static const bool prof_on = std::getenv("RTB_PCG_PROF") != nullptr;
  if (prof_on) {
    if (!prof_buf) RTB_CUDA(cudaMalloc(&prof_buf, 16 * 8));
    RTB_CUDA(cudaMemsetAsync(prof_buf, 0, 16 * 8, st));
    a.prof = prof_buf;
  }
  void* args[] = {(void*)&a, (void*)&sh, (void*)&xa};
  RTB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, smem, st));
  RTB_LAUNCH_CHECK();
  count_variant("k_pcg_split");
  if (prof_on) {
    unsigned long long h[16];
    int stat[2];
    RTB_CUDA(cudaMemcpyAsync(h, prof_buf, 128, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaMemcpyAsync(stat, status_dev, 8, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr,
                 "[pcg_split] d=%d iters=%d status=%d ns (vector CTA 0): publish-barrier %llu "
                 "slice+barrier %llu reduce+barrier %llu cg-vector %llu other-vector %llu | "
                 "slice CTA 0 compute %llu | cg: q+pq %llu update+rr %llu precond %llu rho %llu | "
                 "precond: pass %llu (unused %llu) eig-pass %llu (unused %llu)\n",
                 d, stat[1], stat[0], h[0], h[1], h[2], h[5], h[3], h[4], h[8], h[9], h[10], h[11],
                 h[12], h[13], h[6], h[7]);
  }
}

}  // namespace rtb
