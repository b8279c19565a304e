// k_c4.cu -- BASELINE config 4: Kronecker-product sampling + fused fiber gather / SYRK.
//
// Pinned interpretation (BASELINE.md "C4 interpretation"): per sample
//   1. draw (j2, j3) from the augmented product leverage distribution of A2 (x) A3
//      (ProductLeverageSampler with d = R2 R3 augmented rows, ref kronecker.cpp:159-181;
//      our k_draw.cu decode, bit-identical to the reference stream);
//   2. z = a2(j2) (x) a3(j3) (width W = R2 R3 = 1024);
//   3. gather the mode-1 fiber X[:, j2, j3] (I1 FP32 values, upcast to FP64);
//   4. accumulate the W x W Gram and the W x I1 RHS:  G = sum w^2 z z^T + lambda sum_aug,
//      RHS = sum w^2 z x^T.
//
// The reference streams every draw into the triangle (sketch_ridge.cpp:105-128). Here:
//   (A) one radix sort of the draws by flat data index j2 I3 + j3 (augmented draws carry a
//       sentinel and sort last); equal indices are merged into one record with weight
//       c = sum of their w^2 in sorted (= draw) order, so every distinct sampled row is
//       touched once (at s = 1e7 over the 4.2M rows of A2 (x) A3: ~2.9M distinct of 5M
//       data draws). The merge is the exact identity sum_t w_t^2 z z^T = (sum_t w_t^2) z z^T.
//   (B) Gram through a dense record-weight matrix C (I3 x I2, C[j3][j2] = c):
//         G[(p,q),(p',q')] = sum_{j2} A2[j2,p] A2[j2,p'] T[j2,(q,q')],
//         T[j2,(q,q')]     = sum_{j3} C[j2,j3] A3[j3,q] A3[j3,q'],
//       two FP64 DMMA GEMMs (k_gemm_tn) over vech Khatri-Rao row products (unordered
//       pairs only: 528 of 1024 columns at R = 32), then the expansion into (p,q) order
//       plus the augmented diagonal.
//   (C) RHS factored by j2 bucket: D_b = sum_{t in b} c_t a3(j3_t) x_t^T (R3 x I1), 2 R3 I1
//       flops per record (k_c4_dfib), then RHS = sum_b a2(b) (x) D_b = A2^T D (k_gemm_tn).
//       The rows c_t a3(j3_t) are pre-scaled into a record-ordered array.
// Fixed summation orders throughout: deterministic.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace rtb {

namespace {

constexpr int kRowW = 32;      // padded width of the pre-scaled a3 rows

__global__ void k_c4_iota(unsigned long long s, unsigned* vals) {
  const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < s) vals[t] = (unsigned)t;
}

// over the sorted draw indices (data rows < total, augmented rows total + j after them):
// head[t] = 1 where a run of equal data indices starts; astart[j] (W + 1) = first sorted
// position of augmented index j (runs are contiguous, so counts are differences -- no
// atomics); *ndata = number of data draws
__global__ void k_c4_heads(const unsigned long long* __restrict__ keys_s, unsigned long long s,
                           unsigned long long total, int W, unsigned* __restrict__ head,
                           int* __restrict__ astart, unsigned long long* __restrict__ ndata) {
  const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  const unsigned long long k = keys_s[t];
  const bool has_prev = t > 0;
  const unsigned long long pk = has_prev ? keys_s[t - 1] : 0ULL;
  head[t] = (k < total && (!has_prev || pk != k)) ? 1u : 0u;
  if (k >= total && (!has_prev || pk != k)) {
    const long long j = (long long)(k - total);
    const long long jp = (has_prev && pk >= total) ? (long long)(pk - total) : -1;
    for (long long jj = jp + 1; jj <= j; ++jj) astart[jj] = (int)t;
    if (!has_prev || pk < total) *ndata = t;
  }
  if (t == s - 1) {
    const long long jl = k >= total ? (long long)(k - total) : -1;
    for (long long jj = jl + 1; jj <= W; ++jj) astart[jj] = (int)s;
    if (k < total) *ndata = s;
  }
}

// one thread per run head: record u = (key, c = sum of w^2 over the run in draw order)
__global__ void k_c4_unique(const unsigned long long* __restrict__ keys_s,
                            const unsigned* __restrict__ vals_s, const unsigned* __restrict__ head,
                            const unsigned* __restrict__ uid, const double* __restrict__ w,
                            unsigned long long s, unsigned long long* __restrict__ ukey,
                            double* __restrict__ uc, unsigned long long* __restrict__ nuniq) {
  const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  if (t == s - 1) *nuniq = (unsigned long long)uid[t] + head[t];
  if (!head[t]) return;
  const unsigned long long k = keys_s[t];
  double c = 0.0;
  for (unsigned long long r = t; r < s && keys_s[r] == k; ++r) {
    const double wt = w[vals_s[r]];
    c += wt * wt;
  }
  const unsigned u = uid[t];
  ukey[u] = k;
  uc[u] = c;
}

// bstart[b] (I2 + 1) = first record of bucket j2 = b (records are sorted by key)
__global__ void k_c4_bounds(const unsigned long long* __restrict__ ukey,
                            const unsigned long long* __restrict__ nuniq, unsigned long long s,
                            int I2, int I3, int* __restrict__ bstart) {
  const unsigned long long u = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long U = *nuniq;
  if (U == 0) {
    if (u == 0)
      for (int b = 0; b <= I2; ++b) bstart[b] = 0;
    return;
  }
  if (u >= U || u >= s) return;
  const long long j2 = (long long)(ukey[u] / (unsigned long long)I3);
  const long long jp = u > 0 ? (long long)(ukey[u - 1] / (unsigned long long)I3) : -1;
  for (long long b = jp + 1; b <= j2; ++b) bstart[b] = (int)u;
  if (u == U - 1)
    for (long long b = j2 + 1; b <= I2; ++b) bstart[b] = (int)U;
}

// pre-scaled record rows c_u a3(j3_u), zero-padded to 32 columns (grid-stride, 16 B stores)
__global__ void k_c4_rows(const unsigned long long* __restrict__ ukey, const double* __restrict__ uc,
                          const unsigned long long* __restrict__ nuniq, int I3,
                          const double* __restrict__ A3, int R3, double* __restrict__ rows) {
  const unsigned long long n = *nuniq * (kRowW / 2);
  for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long u = e / (kRowW / 2);
    const int q = 2 * (int)(e % (kRowW / 2));
    const double cu = uc[u];
    const double* a = A3 + (size_t)(ukey[u] % (unsigned long long)I3) * R3;
    reinterpret_cast<double2*>(rows)[e] =
        make_double2(q < R3 ? cu * a[q] : 0.0, q + 1 < R3 ? cu * a[q + 1] : 0.0);
  }
}

// ---- Gram (B) ----
// C^T[j3][j2] = c of record (j2, j3); the matrix is zeroed first, records are distinct
__global__ void k_c4_scatter(const unsigned long long* __restrict__ ukey, const double* __restrict__ uc,
                             const unsigned long long* __restrict__ nuniq, int I2, int I3,
                             double* __restrict__ ct) {
  const unsigned long long u = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= *nuniq) return;
  const unsigned long long k = ukey[u];
  const unsigned long long j2 = k / (unsigned long long)I3, j3 = k % (unsigned long long)I3;
  ct[j3 * (unsigned long long)I2 + j2] = uc[u];
}

// vech Khatri-Rao row products: kr[i][u] = A[i,a] A[i,b], u = vech pair (a <= b)
__global__ void k_c4_kr(const double* __restrict__ A, int I, int R, double* __restrict__ kr) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int m = R * (R + 1) / 2;
  if (e >= (long long)I * m) return;
  const long long i = e / m;
  int a, b;
  pair_of((int)(e % m), R, a, b);
  kr[e] = A[i * R + a] * A[i * R + b];
}

// out[m][n] = sum_k A[k][m] B[k][n]  (A: K x M, B: K x N, row-major, leading dims lda/ldb).
// (32 WM) x (16 (8 / WM)) output tile per CTA (WM = 2: 64 x 64; WM = 1: 32 x 128 for M <= 32),
// 8 warps of 32 x 16 (4 x 2 DMMA.8x8x4 tiles), K chunks of 16 through a two-buffer cp.async
// ring; rows padded to 4 mod 16 doubles make the fragment loads conflict-free.
constexpr int kGK = 16;
// blockIdx.z = batch entry (A, B, out advanced by sA, sB, sO).
template <int WM>
__global__ void __launch_bounds__(256) k_gemm_tn(const double* __restrict__ A, long long lda,
                                                 const double* __restrict__ B, long long ldb,
                                                 int M, int N, int K, double* __restrict__ out,
                                                 long long ldo, long long sA, long long sB,
                                                 long long sO) {
  constexpr int TM = 32 * WM, TN = 16 * (8 / WM), LDA = TM + 4, LDB = TN + 4;
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  out += blockIdx.z * sO;
  __shared__ __align__(16) double As[2][kGK][LDA];
  __shared__ __align__(16) double Bs[2][kGK][LDB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const long long m0 = (long long)blockIdx.y * TM, n0 = (long long)blockIdx.x * TN;
  const int wm = warp / (8 / WM), wn = warp % (8 / WM);
  double c[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  const int nk = (K + kGK - 1) / kGK;
  auto load = [&](int kc, int buf) {
    const int k0 = kc * kGK;
    for (int e = tid; e < kGK * TM; e += 256) {
      const int k = e / TM, j = e % TM;
      const bool v = k0 + k < K && m0 + j < M;
      cp_async8(&As[buf][k][j], A + (v ? (long long)(k0 + k) * lda + m0 + j : 0), v);
    }
    for (int e = tid; e < kGK * TN; e += 256) {
      const int k = e / TN, j = e % TN;
      const bool v = k0 + k < K && n0 + j < N;
      cp_async8(&Bs[buf][k][j], B + (v ? (long long)(k0 + k) * ldb + n0 + j : 0), v);
    }
  };
  load(0, 0);
  cp_async_commit();
  for (int kc = 0; kc < nk; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nk) load(kc + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kGK; ks += 4) {
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][ks + t][wm * 32 + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Bs[buf][ks + t][wn * 16 + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(c[i][j][0], c[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long m = m0 + wm * 32 + i * 8 + g, n = n0 + wn * 16 + j * 8 + 2 * t + h;
        if (m < M && n < N) out[m * ldo + n] = c[i][j][h];
      }
}

// G[(p,q),(p',q')] = G'[v(p,p')][v(q,q')] + [p = p', q = q'] (augmented draws of (p,q)) aug_term
// (G' over vech pairs: the Gram of Kronecker rows depends on the unordered index pairs)
__global__ void k_c4_gram_out(const double* __restrict__ gp, int R2, int R3,
                              const int* __restrict__ astart, double aug_term,
                              double* __restrict__ gram) {
  const long long W = (long long)R2 * R3;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= W * W) return;
  const long long r = e / W, col = e % W;
  const int p = (int)(r / R3), q = (int)(r % R3), pp = (int)(col / R3), qq = (int)(col % R3);
  const int m3 = R3 * (R3 + 1) / 2;
  const int u2 = p <= pp ? upper_pair(p, pp, R2) : upper_pair(pp, p, R2);
  const int u3 = q <= qq ? upper_pair(q, qq, R3) : upper_pair(qq, q, R3);
  double v = gp[(long long)u2 * m3 + u3];
  if (r == col) v += (double)(astart[r + 1] - astart[r]) * aug_term;
  gram[e] = v;
}

// ---- RHS (C) ----
// Two steps. k_c4_dfib: D[b][q][i] = sum over the records t of bucket b of
// rows[t][q] x_t[i] (rows = c_t a3(j3_t), x_t = the sampled mode-1 fiber), a GEMM per bucket
// with M = R3 (<= 32), N = I1, K = the bucket's records. Then RHS (R2 x R3 I1) = A2^T D by
// k_gemm_tn (the fold RHS[(p,q), i] = sum_b a2(b)[p] D_b[q][i]).
//
// k_c4_dfib: persistent, two CTAs per SM; work item = (bucket b, 256-column tile of i),
// bucket-major, static round robin. Per item the bucket's record keys are staged in shared
// memory (segments of kSeg records), then chunks of 16 records flow through a kSt-stage
// cp.async ring: the pre-scaled rows (16 x 16 B per chunk) and the tile's 256 fiber values
// per record (MODE 1: fiber-major X with I1 % 4 == 0, one 1 KB run per record = 64 x 16 B
// copies; MODE 2: fiber-major, 4 B copies; MODE 0: canonical row-major X, 256 strided 4 B
// copies), FP32 kept in shared memory and upcast at the fragment load. 8 warps, warp w owns
// the 32 x 32 tile D[:, 32 w .. 32 w + 31] as 4 x 4 DMMA.8x8x4 tiles (16 independent
// accumulator chains; per k-step 4 A + 4 B fragment loads feed 16 DMMAs). Each (b, i) is
// produced by one CTA in record order: deterministic, and fibers are read from HBM once.
constexpr int kQLDT = 36;         // rows [k][q]: conflict-free A fragments
constexpr int kDT = 256;          // fiber columns per work item
constexpr int kQLDB = kDT + 8;    // fiber values (floats) [k][i]: conflict-free B fragments
constexpr int kSt = 4;            // ring stages
constexpr int kRC = 16;           // records per chunk
constexpr int kSeg = 2048;        // records per key segment
template <int MODE>
__global__ void __launch_bounds__(256, 2) k_c4_dfib(
    const float* __restrict__ X, int I1, int I2, int I3, int R3,
    const unsigned long long* __restrict__ ukey, const double* __restrict__ rows,
    const int* __restrict__ bstart, int blo, int bhi, double* __restrict__ D) {
  extern __shared__ __align__(16) double c4s[];
  unsigned long long* Ks = reinterpret_cast<unsigned long long*>(c4s);     // [kSeg]
  double* At = c4s + kSeg;                                                 // [kSt][kRC][kQLDT]
  float* Bf = reinterpret_cast<float*>(At + kSt * kRC * kQLDT);            // [kSt][kRC][kQLDB]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long slab = (long long)I2 * I3;
  const int NT = (I1 + kDT - 1) / kDT;
  const long long nitems = (long long)(bhi - blo) * NT;
  for (long long item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int b = blo + (int)(item / NT), n0 = (int)(item % NT) * kDT;
    const int r0 = bstart[b], cnt = bstart[b + 1] - r0;
    double c[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) c[i][j][0] = c[i][j][1] = 0.0;
    for (int seg = 0; seg < cnt; seg += kSeg) {
      const int len = min(kSeg, cnt - seg);
      __syncthreads();  // Ks / ring free (previous segment or item done)
      for (int k = tid; k < len; k += 256) cp_async8(Ks + k, ukey + r0 + seg + k, true);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      const int nchk = (len + kRC - 1) / kRC;
      auto load = [&](int ch) {
        if (ch >= nchk) return;
        const int sb = ch % kSt, kb = ch * kRC, n = min(kRC, len - kb);
        double* at = At + (size_t)sb * kRC * kQLDT;
        float* bf = Bf + (size_t)sb * kRC * kQLDB;
        {
          const int k = tid >> 4, pc = tid & 15;
          const bool v = k < n;
          cp_async16(at + k * kQLDT + 2 * pc,
                     rows + (v ? ((size_t)(r0 + seg + kb + k) * kRowW + 2 * pc) : 0), v);
        }
        if (MODE == 1) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int e = tid + 256 * j, k = e >> 6, pc = e & 63;
            const bool v = k < n && n0 + 4 * pc < I1;
            const unsigned long long key = Ks[kb + (k < n ? k : 0)];
            cp_async16(bf + k * kQLDB + 4 * pc, X + (v ? key * (unsigned long long)I1 + n0 + 4 * pc : 0), v);
          }
        } else {
          const int col = n0 + tid;
#pragma unroll 4
          for (int k = 0; k < kRC; ++k) {
            const bool v = k < n && col < I1;
            const unsigned long long key = Ks[kb + (k < n ? k : 0)];
            const long long off = !v ? 0
                                  : MODE == 2 ? (long long)(key * (unsigned long long)I1) + col
                                              : (long long)col * slab + (long long)key;
            cp_async4(bf + k * kQLDB + tid, X + off, v);
          }
        }
      };
#pragma unroll
      for (int ch = 0; ch < kSt - 1; ++ch) {
        load(ch);
        cp_async_commit();
      }
      for (int ch = 0; ch < nchk; ++ch) {
        load(ch + kSt - 1);
        cp_async_commit();
        cp_async_wait<kSt - 1>();
        __syncthreads();  // chunk ch landed
        const int sb = ch % kSt;
        const double* at = At + (size_t)sb * kRC * kQLDT;
        const float* bf = Bf + (size_t)sb * kRC * kQLDB + warp * 32 + g;
        const int kpad = (min(kRC, len - ch * kRC) + 3) & ~3;
        for (int ks = 0; ks < kpad; ks += 4) {
          const int k = ks + t;
          double a[4], bv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = at[k * kQLDT + i * 8 + g];
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = (double)bf[k * kQLDB + j * 8];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_8x8x4(c[i][j][0], c[i][j][1], a[i], bv[j]);
        }
        __syncthreads();  // stage sb free
      }
      cp_async_wait<0>();
    }
    // D tile out (empty buckets write zeros)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = i * 8 + g;
      if (q >= R3) continue;
      double* drow = D + ((size_t)(b - blo) * R3 + q) * I1;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = n0 + warp * 32 + j * 8 + 2 * t;
        if (col + 1 < I1 && (I1 % 2 == 0)) {
          *reinterpret_cast<double2*>(drow + col) = make_double2(c[i][j][0], c[i][j][1]);
        } else {
          if (col < I1) drow[col] = c[i][j][0];
          if (col + 1 < I1) drow[col + 1] = c[i][j][1];
        }
      }
    }
  }
}

constexpr size_t kDfibSmem = (size_t)kSeg * 8 + (size_t)kSt * kRC * kQLDT * 8 +
                             (size_t)kSt * kRC * kQLDB * 4;
static_assert(kDfibSmem * 2 <= 227 * 1024, "two k_c4_dfib CTAs per SM");

// Canonical (row-major) X, I3 % 4 == 0: the sampled values X[i, b, j3] of bucket b lie in the
// rows X[i, b, :] (contiguous over j3), so instead of gathering strided fibers the kernel
// reads 16-wide j3 windows of those rows -- only the windows that hold a sampled j3 -- and
// runs D_b[:, tile] += W_b(window)^T X_b(window) with W_b[j3][q] = c a3(j3)[q] for the
// sampled j3 (zero rows elsewhere; X values there are masked, so non-finite unsampled
// entries cannot leak in). Same work items, ring, warp tiling and determinism as k_c4_dfib;
// the B tile is [i][j3] (64 B row segments, padded to 20 floats: conflict-free fragments).
constexpr int kSW = 16;            // j3 window per chunk
constexpr int kSLB = kSW + 4;      // B tile row stride (floats)
constexpr int kSSt = 3;            // ring stages
__global__ void __launch_bounds__(256, 2) k_c4_dslab(
    const float* __restrict__ X, int I1, int I2, int I3, int R3,
    const unsigned long long* __restrict__ ukey, const double* __restrict__ rows,
    const int* __restrict__ bstart, int blo, int bhi, double* __restrict__ D) {
  extern __shared__ __align__(16) double c4s[];
  unsigned long long* Ks = reinterpret_cast<unsigned long long*>(c4s);     // [kSeg]
  int* cst = reinterpret_cast<int*>(Ks + kSeg);                            // [kSeg + 1] window starts
  double* At = reinterpret_cast<double*>(cst + kSeg + 4);                  // [kSSt][kSW][kQLDT] (16 B aligned)
  float* Bf = reinterpret_cast<float*>(At + kSSt * kSW * kQLDT);           // [kSSt][kDT][kSLB]
  unsigned* msk = reinterpret_cast<unsigned*>(Bf + kSSt * kDT * kSLB);     // [kSSt] sampled-row masks
  __shared__ int wsum[8], nwin_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long slab = (long long)I2 * I3;
  const int NT = (I1 + kDT - 1) / kDT;
  const long long nitems = (long long)(bhi - blo) * NT;
  for (long long item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int b = blo + (int)(item / NT), n0 = (int)(item % NT) * kDT;
    const int r0 = bstart[b], cnt = bstart[b + 1] - r0;
    const unsigned long long kb = (unsigned long long)b * I3;
    double c[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) c[i][j][0] = c[i][j][1] = 0.0;
    for (int seg = 0; seg < cnt; seg += kSeg) {
      const int len = min(kSeg, cnt - seg);
      __syncthreads();  // Ks / cst / ring free
      for (int k = tid; k < len; k += 256) cp_async8(Ks + k, ukey + r0 + seg + k, true);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      // window list: records k whose window (j3 / kSW) differs from record k-1's start a window
      {
        const int per = (len + 255) / 256, k0 = tid * per, k1 = min(len, k0 + per);
        int n = 0;
        for (int k = k0; k < k1; ++k)
          n += (k == 0 || (int)((Ks[k] - kb) / kSW) != (int)((Ks[k - 1] - kb) / kSW));
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int off = incl - n;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        for (int k = k0; k < k1; ++k)
          if (k == 0 || (int)((Ks[k] - kb) / kSW) != (int)((Ks[k - 1] - kb) / kSW)) cst[off++] = k;
        if (tid == 255) {
          int tot = 0;
          for (int w = 0; w < 8; ++w) tot += wsum[w];
          nwin_s = tot;
          cst[tot] = len;
        }
        __syncthreads();
      }
      const int nwin = nwin_s;
      auto load = [&](int ch) {
        if (ch >= nwin) return;
        const int sb = ch % kSSt;
        const int ka = cst[ch], kz = cst[ch + 1];
        const int j0 = (int)((Ks[ka] - kb) / kSW) * kSW;
        double* at = At + (size_t)sb * kSW * kQLDT;
        float* bf = Bf + (size_t)sb * kDT * kSLB;
        {  // A rows: the window's sampled j3 take their pre-scaled record row, others zero
          const int r = tid >> 4, pc = tid & 15;
          int u = -1;
          for (int k = ka; k < kz; ++k)
            if ((int)(Ks[k] - kb) - j0 == r) u = k;
          cp_async16(at + r * kQLDT + 2 * pc,
                     rows + (u >= 0 ? ((size_t)(r0 + seg + u) * kRowW + 2 * pc) : 0), u >= 0);
          if (tid < 32) {
            unsigned m = 0;
            for (int k = ka; k < kz; ++k) m |= 1u << ((int)(Ks[k] - kb) - j0);
            if (tid == 0) msk[sb] = m;
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // B: the tile's 256 rows X[i, b, j0 .. j0 + 15]
          const int e = tid + 256 * j, i = e >> 2, pc = e & 3;
          const bool v = n0 + i < I1 && j0 + 4 * pc < I3;
          cp_async16(bf + i * kSLB + 4 * pc,
                     X + (v ? (long long)(n0 + i) * slab + (long long)kb + j0 + 4 * pc : 0), v);
        }
      };
#pragma unroll
      for (int ch = 0; ch < kSSt - 1; ++ch) {
        load(ch);
        cp_async_commit();
      }
      for (int ch = 0; ch < nwin; ++ch) {
        load(ch + kSSt - 1);
        cp_async_commit();
        cp_async_wait<kSSt - 1>();
        __syncthreads();  // window ch landed (and its mask)
        const int sb = ch % kSSt;
        const double* at = At + (size_t)sb * kSW * kQLDT;
        const float* bf = Bf + (size_t)sb * kDT * kSLB + (warp * 32 + g) * kSLB;
        const unsigned m = msk[sb];
#pragma unroll
        for (int ks = 0; ks < kSW; ks += 4) {
          const int k = ks + t;
          const bool on = (m >> k) & 1u;
          double a[4], bv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = at[k * kQLDT + i * 8 + g];
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = on ? (double)bf[j * 8 * kSLB + k] : 0.0;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_8x8x4(c[i][j][0], c[i][j][1], a[i], bv[j]);
        }
        __syncthreads();  // stage sb free
      }
      cp_async_wait<0>();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = i * 8 + g;
      if (q >= R3) continue;
      double* drow = D + ((size_t)(b - blo) * R3 + q) * I1;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = n0 + warp * 32 + j * 8 + 2 * t;
        if (col + 1 < I1 && (I1 % 2 == 0)) {
          *reinterpret_cast<double2*>(drow + col) = make_double2(c[i][j][0], c[i][j][1]);
        } else {
          if (col < I1) drow[col] = c[i][j][0];
          if (col + 1 < I1) drow[col + 1] = c[i][j][1];
        }
      }
    }
  }
}

constexpr size_t kDslabSmem = (size_t)kSeg * 8 + (size_t)(kSeg + 4) * 4 +
                              (size_t)kSSt * kSW * kQLDT * 8 + (size_t)kSSt * kDT * kSLB * 4 +
                              kSSt * 4 + 16;
static_assert(kDslabSmem * 2 <= 227 * 1024, "two k_c4_dslab CTAs per SM");

// ---- fiber-major conversion: out[(i2 I3 + i3) I1 + i1] = x[(i1 I2 + i2) I3 + i3] ----
// a transpose of the I1 x (I2 I3) matrix in 32 x 32 tiles
__global__ void k_c4_to_fm(const float* __restrict__ x, long long rows, long long cols,
                           float* __restrict__ out) {
  __shared__ float tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32, r0 = (long long)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const long long r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = x[r * cols + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const long long c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][k];
  }
}

struct C4Layout {
  unsigned long long *keys_s, *ukey, *ndata, *nuniq;
  unsigned *vals, *vals_s, *head, *uid;
  int *astart, *bstart;
  double *uc, *rows, *dfib;
  void* cub_sort;
  size_t cub_sort_bytes;
  void* cub_scan;
  size_t cub_scan_bytes;
  char* end;
};

template <typename F>
C4Layout c4_carve(unsigned long long s, int I1, int I2, int R3, int W, F&& take) {
  C4Layout l{};
  size_t sb = 0, cb = 0;
  cub::DeviceRadixSort::SortPairs<unsigned long long, unsigned>(
      nullptr, sb, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
      (const unsigned*)nullptr, (unsigned*)nullptr, (int)s);
  cub::DeviceScan::ExclusiveSum(nullptr, cb, (const unsigned*)nullptr, (unsigned*)nullptr, (int)s);
  l.keys_s = (unsigned long long*)take(s * 8);
  l.ukey = (unsigned long long*)take(s * 8);
  l.ndata = (unsigned long long*)take(8);
  l.nuniq = (unsigned long long*)take(8);
  l.vals = (unsigned*)take(s * 4);
  l.vals_s = (unsigned*)take(s * 4);
  l.head = (unsigned*)take(s * 4);
  l.uid = (unsigned*)take(s * 4);
  l.astart = (int*)take((size_t)(W + 1) * 4);
  l.bstart = (int*)take((size_t)(I2 + 1) * 4);
  l.uc = (double*)take(s * 8);
  l.rows = (double*)take(s * kRowW * 8);
  l.dfib = (double*)take((size_t)I2 * R3 * I1 * 8);
  l.cub_sort_bytes = sb;
  l.cub_sort = take(sb);
  l.cub_scan_bytes = cb;
  l.cub_scan = take(cb);
  l.end = (char*)take(0);
  return l;
}

size_t gram_part_bytes(int I2, int I3, int R2, int R3) {
  const size_t r2 = (size_t)R2 * (R2 + 1) / 2, r3 = (size_t)R3 * (R3 + 1) / 2;
  return ((size_t)I3 * I2 + (size_t)I3 * r3 + (size_t)I2 * r2 + (size_t)I2 * r3 + r2 * r3) * 8 +
         5 * 256;
}

}  // namespace

// out = A^T B (k_gemm_tn), tile shape by M; batch entries z = 0 .. batch-1 at strides
void gemm_tn(const double* A, long long lda, const double* B, long long ldb, int M, long long N,
             int K, double* out, long long ldo, cudaStream_t st, int batch, long long sA,
             long long sB, long long sO) {
  if (batch < 1 || batch > 65535) throw Error(1, "gemm_tn: batch out of range");
  if (M <= 32) {
    const long long gx = (N + 127) / 128;
    if (gx > 0x7fffffffLL) throw Error(1, "gemm_tn: N too large");
    k_gemm_tn<1><<<dim3((unsigned)gx, ceil_div(M, 32), batch), 256, 0, st>>>(
        A, lda, B, ldb, M, (int)N, K, out, ldo, sA, sB, sO);
  } else {
    const long long gx = (N + 63) / 64;
    if (gx > 0x7fffffffLL) throw Error(1, "gemm_tn: N too large");
    k_gemm_tn<2><<<dim3((unsigned)gx, ceil_div(M, 64), batch), 256, 0, st>>>(
        A, lda, B, ldb, M, (int)N, K, out, ldo, sA, sB, sO);
  }
  RTB_LAUNCH_CHECK();
}

size_t c4_work_bytes(unsigned long long s, int I1, int I2, int I3, int R2, int R3, bool gram) {
  size_t off = 0;
  auto take = [&](size_t b) {
    const size_t r = off;
    off += (b + 255) & ~size_t(255);
    return (void*)r;
  };
  c4_carve(s, I1, I2, R3, R2 * R3, take);
  return off + (gram ? gram_part_bytes(I2, I3, R2, R3) : 0) + 256;
}

void c4_to_fiber_major(const float* x, int I1, int I2, int I3, float* out, cudaStream_t st) {
  const long long cols = (long long)I2 * I3;
  const dim3 grid((unsigned)ceil_div<long long>(cols, 32LL), (unsigned)ceil_div(I1, 32));
  if (grid.y > 65535) throw Error(1, "c4_to_fiber_major: I1 too large");
  k_c4_to_fm<<<grid, dim3(32, 8), 0, st>>>(x, I1, cols, out);
  RTB_LAUNCH_CHECK();
}

void c4_sketch(const float* x, bool fiber_major, int I1, int I2, int I3, const double* A2, int R2,
               const double* A3, int R3, const unsigned long long* idx, const double* w,
               unsigned long long s, double lambda, void* work, size_t work_bytes, double* gram,
               double* rhs, unsigned long long* data_draws_dev, unsigned long long* unique_dev,
               cudaEvent_t ev_gram_done, cudaStream_t st, int shard_rank, int shard_count) {
  if (R3 > 32 || R2 > 32) throw Error(1, "c4_sketch: ranks must be <= 32");
  if (shard_count < 1 || shard_rank < 0 || shard_rank >= shard_count)
    throw Error(1, "c4_sketch: bad shard");
  // this shard's j2 buckets (its share of the Gram and RHS partial sums)
  const int blo = (int)((long long)I2 * shard_rank / shard_count);
  const int bhi = (int)((long long)I2 * (shard_rank + 1) / shard_count);
  const int nb = bhi - blo;
  if (s > 0xffffffffULL) throw Error(1, "c4_sketch: at most 2^32 - 1 draws");
  const int W = R2 * R3;
  if (work_bytes < c4_work_bytes(s, I1, I2, I3, R2, R3, gram != nullptr))
    throw Error(4, "c4_sketch: workspace");
  char* p = static_cast<char*>(work);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return (void*)r;
  };
  C4Layout l = c4_carve(s, I1, I2, R3, W, take);
  const unsigned long long total = (unsigned long long)I2 * I3;
  int bits = 1;
  while ((1ULL << bits) <= total + (unsigned long long)W) ++bits;
  const unsigned sb = (unsigned)ceil_div<unsigned long long>(s, 256ULL);
  // sort the raw draw indices (augmented ones, total + j, sort after the data rows)
  k_c4_iota<<<sb, 256, 0, st>>>(s, l.vals);
  RTB_LAUNCH_CHECK();
  size_t cb = l.cub_sort_bytes;
  RTB_CUDA(cub::DeviceRadixSort::SortPairs(l.cub_sort, cb, idx, l.keys_s, l.vals, l.vals_s,
                                           (int)s, 0, bits, st));
  k_c4_heads<<<sb, 256, 0, st>>>(l.keys_s, s, total, W, l.head, l.astart, l.ndata);
  RTB_LAUNCH_CHECK();
  cb = l.cub_scan_bytes;
  RTB_CUDA(cub::DeviceScan::ExclusiveSum(l.cub_scan, cb, l.head, l.uid, (int)s, st));
  k_c4_unique<<<sb, 256, 0, st>>>(l.keys_s, l.vals_s, l.head, l.uid, w, s, l.ukey, l.uc, l.nuniq);
  RTB_LAUNCH_CHECK();
  k_c4_bounds<<<sb, 256, 0, st>>>(l.ukey, l.nuniq, s, I2, I3, l.bstart);
  RTB_LAUNCH_CHECK();
  if (data_draws_dev)
    RTB_CUDA(cudaMemcpyAsync(data_draws_dev, l.ndata, 8, cudaMemcpyDeviceToDevice, st));
  if (unique_dev) RTB_CUDA(cudaMemcpyAsync(unique_dev, l.nuniq, 8, cudaMemcpyDeviceToDevice, st));
  if (gram) {
    double* ct = (double*)take((size_t)I3 * I2 * 8);
    const int m2 = R2 * (R2 + 1) / 2, m3 = R3 * (R3 + 1) / 2;
    double* ka3 = (double*)take((size_t)I3 * m3 * 8);
    double* ka2 = (double*)take((size_t)I2 * m2 * 8);
    double* tm = (double*)take((size_t)I2 * m3 * 8);
    double* gp = (double*)take((size_t)m2 * m3 * 8);
    RTB_CUDA(cudaMemsetAsync(ct, 0, (size_t)I3 * I2 * 8, st));
    k_c4_scatter<<<sb, 256, 0, st>>>(l.ukey, l.uc, l.nuniq, I2, I3, ct);
    RTB_LAUNCH_CHECK();
    k_c4_kr<<<(unsigned)ceil_div<long long>((long long)I3 * m3, 256LL), 256, 0, st>>>(A3, I3, R3, ka3);
    RTB_LAUNCH_CHECK();
    k_c4_kr<<<(unsigned)ceil_div<long long>((long long)I2 * m2, 256LL), 256, 0, st>>>(A2, I2, R2, ka2);
    RTB_LAUNCH_CHECK();
    // T (this shard's j2 rows x m3) = C KA3: out[j2][v(q,q')] = sum_j3 CT[j3][j2] KA3[j3][v(q,q')]
    if (nb > 0) {
      gemm_tn(ct + blo, I2, ka3, m3, nb, m3, I3, tm, m3, st);
      // G' (m2 x m3) = KA2^T T over the shard's j2
      gemm_tn(ka2 + (size_t)blo * m2, m2, tm, m3, m2, m3, nb, gp, m3, st);
    } else {
      RTB_CUDA(cudaMemsetAsync(gp, 0, (size_t)m2 * m3 * 8, st));
    }
    GramSpec gs{};
    gs.s = s;
    gs.d = W;
    gs.lambda = lambda;
    k_c4_gram_out<<<(unsigned)ceil_div<long long>((long long)W * W, 256LL), 256, 0, st>>>(
        gp, R2, R3, l.astart, shard_rank == 0 ? gram_aug_term(gs) : 0.0, gram);
    RTB_LAUNCH_CHECK();
  }
  if (ev_gram_done) RTB_CUDA(cudaEventRecord(ev_gram_done, st));
  if (!(x && rhs)) return;
  k_c4_rows<<<kNumSMs * 8, 256, 0, st>>>(l.ukey, l.uc, l.nuniq, I3, A3, R3, l.rows);
  RTB_LAUNCH_CHECK();
  set_max_smem(k_c4_dfib<0>, (int)kDfibSmem);
  set_max_smem(k_c4_dfib<1>, (int)kDfibSmem);
  set_max_smem(k_c4_dfib<2>, (int)kDfibSmem);
  const long long nitems = (long long)nb * ceil_div(I1, kDT);
  const int grid = (int)std::max<long long>(1, std::min<long long>(nitems, 2LL * kNumSMs));
  // canonical X: windows of the rows X[i, b, :] once the sampled rows are dense enough that a
  // 16-wide window holds more than ~one of them (below, the strided gathers move less)
  const bool slab_windows = !fiber_major && I3 % 4 == 0 &&
                            0.5 * (double)s >= 0.03 * (double)I2 * (double)I3;
  if (slab_windows) {
    set_max_smem(k_c4_dslab, (int)kDslabSmem);
    k_c4_dslab<<<grid, 256, kDslabSmem, st>>>(x, I1, I2, I3, R3, l.ukey, l.rows, l.bstart, blo,
                                               bhi, l.dfib);
  } else {
    auto kern = !fiber_major ? k_c4_dfib<0> : (I1 % 4 == 0 ? k_c4_dfib<1> : k_c4_dfib<2>);
    kern<<<grid, 256, kDfibSmem, st>>>(x, I1, I2, I3, R3, l.ukey, l.rows, l.bstart, blo, bhi,
                                       l.dfib);
  }
  RTB_LAUNCH_CHECK();
  // RHS (R2 x R3 I1) = A2^T D
  const long long n = (long long)R3 * I1;
  if (nb > 0) gemm_tn(A2 + (size_t)blo * R2, R2, l.dfib, n, R2, n, nb, rhs, n, st);
  else RTB_CUDA(cudaMemsetAsync(rhs, 0, (size_t)R2 * n * 8, st));
}

}  // namespace rtb
