// k_ttm.cu -- tensor-times-matrix passes over the resident tensor X.
//
// The exact factor update (ref tucker.cpp:70-89) needs
//   M_n = X_(n) (kron_{m != n} A_m) G_(n)^T = (X x_{m!=n} A_m^T)_(n) G_(n)^T
// and the loss (ref tucker.cpp:216-229) needs sum (X - Xhat)^2. Both are
// HBM-streaming passes over X with a skinny FP64 contraction, run on the FP64
// tensor cores (mma.sync m8n8k4 -> SASS DMMA.8x8x4):
//
//  * k_ttm_last<RP,VEC,FUSED>: T[o,:] = X[o,:] A_N (contracts the contiguous
//    last mode). FUSED also rebuilds Xhat[o,:] = P[o,:] A_N^T in registers
//    from P = G x_1 A_1 ... x_{N-1} A_{N-1} and accumulates (X - Xhat)^2, so one
//    read of X serves both the loss and the next sweep's factor updates.
//  * k_ttm_mid<RP,VEC>: out[o,r,j] = sum_i A[i,r] X[o,i,j] for an inner
//    (strided) mode, tiled over the contiguous j range.
//  * k_ttm_generic: scalar fallback for small tensors / odd ranks.
//  * k_contract_except: M[i,r] = sum_{o,j} Y[o,i,j] G[o,r,j].
#include "common.cuh"

#include <algorithm>
#include <cstdlib>
#include "kernels.h"

#include <cuda.h>
#include <cudaTypedefs.h>

namespace rtb {

namespace {
// Optional device flag: while set (set_ttm_guard), the launched kernels return at
// once unless *need != 0. Lets the direct loss pass be enqueued behind the fast
// loss formula and run only when that formula is numerically unsafe.
thread_local const int* g_need = nullptr;
#define RTB_GUARD() \
  if (need && *need == 0) return;
constexpr int kBK = 32;     // reduction chunk
constexpr int kPadX = 4;    // smem row padding (doubles) -> conflict-free frags
constexpr int kStages = 3;  // cp.async pipeline depth
}  // namespace

// ---------------------------------------------------------------------------
// Last-mode contraction. X is O x I row-major, A is I x R, T is O x R.
// Block = 128 threads (4 warps x 16 rows), 64 rows of X per CTA.
template <int RP, int VEC, bool FUSED>
__global__ void __launch_bounds__(128) k_ttm_last(const double* __restrict__ X, long long O, int I,
                                                  const double* __restrict__ A, int R,
                                                  double* __restrict__ T,
                                                  const double* __restrict__ P,
                                                  double* __restrict__ partial,
                                                  const int* __restrict__ need) {
  RTB_GUARD()
  constexpr int BM = 64;
  constexpr int LD = kBK + kPadX;
  extern __shared__ __align__(16) double xs[];  // [kStages][BM][LD]
  __shared__ double red[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long o0 = (long long)blockIdx.x * BM;
  const int nchunks = ceil_div(I, kBK);

  auto load_chunk = [&](int c, int stage) {
    double* dst = xs + stage * BM * LD;
    const int i0 = c * kBK;
    constexpr int PER_ROW = kBK / VEC;
    for (int e = tid; e < BM * PER_ROW; e += 128) {
      const int r = e / PER_ROW, col = (e % PER_ROW) * VEC;
      const long long o = o0 + r;
      const bool ok = (o < O) && (i0 + col < I);
      const double* src = ok ? X + o * I + i0 + col : X;
      if (VEC == 2)
        cp_async16(dst + r * LD + col, src, ok);
      else
        cp_async8(dst + r * LD + col, src, ok);
    }
  };

  // P fragments (A operand of the Xhat GEMM): rows m-tile, k = rank index.
  double pf[2][RP / 4];
  if (FUSED) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int ks = 0; ks < RP / 4; ++ks) {
        const long long o = o0 + warp * 16 + mt * 8 + g;
        const int k = ks * 4 + t;
        pf[mt][ks] = (o < O && k < R) ? P[o * R + k] : 0.0;
      }
  }
  double acc[2][RP / 8][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < RP / 8; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  double resid = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nchunks) load_chunk(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (c + kStages - 1 < nchunks) load_chunk(c + kStages - 1, (c + kStages - 1) % kStages);
    cp_async_commit();
    const double* xt = xs + (c % kStages) * BM * LD + warp * 16 * LD;
    const int i0 = c * kBK;
    // T += X_tile (16 x 32 per warp) * A_chunk (32 x RP)
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const int i = i0 + ks * 4 + t;
      double bf[RP / 8];
#pragma unroll
      for (int nt = 0; nt < RP / 8; ++nt) {
        const int r = nt * 8 + g;
        bf[nt] = (i < I && r < R) ? __ldg(A + (size_t)i * R + r) : 0.0;
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const double af = xt[(mt * 8 + g) * LD + ks * 4 + t];
#pragma unroll
        for (int nt = 0; nt < RP / 8; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af, bf[nt]);
      }
    }
    if (FUSED) {
      // Xhat_tile (16 x 32) = P_rows (16 x RP) * A_chunk^T (RP x 32); residual.
#pragma unroll
      for (int nt = 0; nt < kBK / 8; ++nt) {
        const int i = i0 + nt * 8 + g;
        double bf[RP / 4];
#pragma unroll
        for (int ks = 0; ks < RP / 4; ++ks) {
          const int k = ks * 4 + t;
          bf[ks] = (i < I && k < R) ? __ldg(A + (size_t)i * R + k) : 0.0;
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < RP / 4; ++ks) dmma_8x8x4(c0, c1, pf[mt][ks], bf[ks]);
          const double2 xv =
              *reinterpret_cast<const double2*>(xt + (mt * 8 + g) * LD + nt * 8 + 2 * t);
          const double d0 = xv.x - c0, d1 = xv.y - c1;
          resid += d0 * d0 + d1 * d1;  // zero-filled tails contribute exactly 0
        }
      }
    }
  }
  cp_async_wait<0>();
  // store T
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const long long o = o0 + warp * 16 + mt * 8 + g;
    if (o >= O) continue;
#pragma unroll
    for (int nt = 0; nt < RP / 8; ++nt) {
      const int r = nt * 8 + 2 * t;
      if (r < R) T[o * R + r] = acc[mt][nt][0];
      if (r + 1 < R) T[o * R + r + 1] = acc[mt][nt][1];
    }
  }
  if (FUSED) {
    const double s = block_sum<128>(resid, red);
    if (tid == 0) partial[blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// Persistent last-mode contraction (one CTA per SM, 8 warps x 16 rows = 128-row
// blocks): A_N (I x R, padded rows) stays resident in shared memory for the whole
// pass, X streams through a kStages2-deep cp.async pipeline that runs across row
// blocks, so every DMMA operand comes from shared memory. FUSED also rebuilds
// Xhat = P A^T tile by tile and accumulates (X - Xhat)^2 (one partial per CTA).
constexpr int kStages2 = 3;
#ifndef RTB_L3BK
#define RTB_L3BK 64
#define RTB_L3ST 2
#endif
constexpr int kL3BK = RTB_L3BK;     // k_ttm_last3 chunk width (columns per barrier)
constexpr int kL3Stages = RTB_L3ST; // k_ttm_last3 ring depth
#ifndef RTB_L4BK
#define RTB_L4BK 32
#define RTB_L4ST 4
#endif
constexpr int kL4BK = RTB_L4BK;     // k_ttm_last4 chunk width
constexpr int kL4Stages = RTB_L4ST; // k_ttm_last4 ring depth
constexpr int BM2 = 128;
template <int RP>
constexpr int lda2() { return RP + 4; }

// PGEN (3-way): the P rows are not read from a materialised P = G x_1 A_1 x_2 A_2 but
// formed per row block from W = G x_1 A_1 (I_1 x R_2 x R_3, L2-resident) and A_2:
// P[(i1, i2), r3] = sum_r2 A_2[i2, r2] W[i1, r2, r3].
struct PGen {
  const double* W;
  const double* A2;
  int I2, R2;
};

template <int RP, bool FUSED>
__global__ void __launch_bounds__(512, 1) k_ttm_last2(const double* __restrict__ X, long long O,
                                                      int I, const double* __restrict__ A, int R,
                                                      double* __restrict__ T,
                                                      const double* __restrict__ P,
                                                      double* __restrict__ partial,
                                                      const int* __restrict__ need, PGen pg) {
  RTB_GUARD()
  constexpr int LD = kBK + kPadX;
  constexpr int LDA = lda2<RP>();
  // 16 warps. FUSED: warps 0-7 accumulate T for 16 rows each, warps 8-15 rebuild
  // Xhat for the same rows and accumulate the residual (warp specialisation keeps
  // both register sets small and doubles the DMMA chains in flight). Not fused:
  // 16 warps x 8 rows of T.
  constexpr int ROWS = FUSED ? 16 : 8;
  constexpr int MT = ROWS / 8;
  extern __shared__ __align__(16) double sm2[];
  const int Ip = ceil_div(I, kBK) * kBK;  // A rows zero-padded to whole chunks
  double* as = sm2;                        // [Ip][LDA]
  double* xs = as + (size_t)Ip * LDA;      // [kStages2][BM2][LD]
  __shared__ double red[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const bool rwarp = FUSED && warp >= 8;
  const int wrow = FUSED ? (warp & 7) : warp;
  const long long nrb = ceil_div<long long>(O, BM2);
  const int nchunks = ceil_div(I, kBK);
  for (int e = tid; e < Ip * LDA; e += 512) {
    const int i = e / LDA, r = e - i * LDA;
    as[e] = (i < I && r < R) ? A[(size_t)i * R + r] : 0.0;
  }
  const long long my_blocks = blockIdx.x < nrb ? (nrb - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nitems = my_blocks * nchunks;
  auto load_item = [&](long long q, int stage) {
    const long long rb = blockIdx.x + (q / nchunks) * gridDim.x;
    const int c = (int)(q % nchunks);
    const long long o0 = rb * BM2;
    const int i0 = c * kBK;
    double* dst = xs + (size_t)stage * BM2 * LD;
    for (int e = tid; e < BM2 * (kBK / 2); e += 512) {
      const int r = e / (kBK / 2), col = (e % (kBK / 2)) * 2;
      const long long o = o0 + r;
      const bool ok = (o < O) && (i0 + col < I);
      cp_async16(dst + r * LD + col, ok ? X + o * I + i0 + col : X, ok);
    }
  };
#pragma unroll
  for (int sidx = 0; sidx < kStages2 - 1; ++sidx) {
    if (sidx < nitems) load_item(sidx, sidx);
    cp_async_commit();
  }
  double acc[2][MT][RP / 8][2];  // even / odd k steps: twice the DMMA chains
  double pf[MT][RP / 4];
  double resid0 = 0.0, resid1 = 0.0;
  for (long long q = 0; q < nitems; ++q) {
    const int c = (int)(q % nchunks);
    const long long rb = blockIdx.x + (q / nchunks) * gridDim.x;
    const long long o0 = rb * BM2 + wrow * ROWS;
    if (c == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < RP / 8; ++nt) acc[h][mt][nt][0] = acc[h][mt][nt][1] = 0.0;
      if (rwarp) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int ks = 0; ks < RP / 4; ++ks) {
            const long long o = o0 + mt * 8 + g;
            const int k = ks * 4 + t;
            pf[mt][ks] = (o < O && k < R) ? P[o * R + k] : 0.0;
          }
      }
    }
    cp_async_wait<kStages2 - 2>();
    __syncthreads();
    if (q + kStages2 - 1 < nitems) load_item(q + kStages2 - 1, (int)((q + kStages2 - 1) % kStages2));
    cp_async_commit();
    const double* xt = xs + (size_t)(q % kStages2) * BM2 * LD + wrow * ROWS * LD;
    const int i0 = c * kBK;
    if (!rwarp) {
      // T += X_tile (ROWS x 32) A_chunk (32 x RP)
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        const double* ar = as + (size_t)(i0 + ks * 4 + t) * LDA;
        double bf[RP / 8];
#pragma unroll
        for (int nt = 0; nt < RP / 8; ++nt) bf[nt] = ar[nt * 8 + g];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double af = xt[(mt * 8 + g) * LD + ks * 4 + t];
#pragma unroll
          for (int nt = 0; nt < RP / 8; ++nt)
            dmma_8x8x4(acc[ks & 1][mt][nt][0], acc[ks & 1][mt][nt][1], af, bf[nt]);
        }
      }
      if (c == nchunks - 1) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const long long o = o0 + mt * 8 + g;
          if (o >= O) continue;
#pragma unroll
          for (int nt = 0; nt < RP / 8; ++nt) {
            const int r = nt * 8 + 2 * t;
            if (r < R) T[o * R + r] = acc[0][mt][nt][0] + acc[1][mt][nt][0];
            if (r + 1 < R) T[o * R + r + 1] = acc[0][mt][nt][1] + acc[1][mt][nt][1];
          }
        }
      }
    } else {
      // Xhat_tile (16 x 32) = P_rows (16 x RP) A_chunk^T (RP x 32); residual
#pragma unroll
      for (int nt = 0; nt < kBK / 8; ++nt) {
        const double* ar = as + (size_t)(i0 + nt * 8 + g) * LDA;
        double bf[RP / 4];
#pragma unroll
        for (int ks = 0; ks < RP / 4; ++ks) bf[ks] = ar[ks * 4 + t];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < RP / 4; ks += 2) {
            dmma_8x8x4(c0, c1, pf[mt][ks], bf[ks]);
            if (ks + 1 < RP / 4) dmma_8x8x4(e0, e1, pf[mt][ks + 1], bf[ks + 1]);
          }
          c0 += e0;
          c1 += e1;
          const double2 xv =
              *reinterpret_cast<const double2*>(xt + (mt * 8 + g) * LD + nt * 8 + 2 * t);
          const double d0 = xv.x - c0, d1 = xv.y - c1;
          resid0 = fma(d0, d0, resid0);  // zero-filled tails contribute exactly 0
          resid1 = fma(d1, d1, resid1);
        }
      }
    }
  }
  cp_async_wait<0>();
  if (FUSED) {
    const double s = block_sum<512>(resid0 + resid1, red);
    if (tid == 0) partial[blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// Strided-mode contraction: X viewed as (O, I, J), out (O, R, J). Columns are
// the flattened (o, j) pairs (so small J packs several o into one 64-column
// tile); blockIdx.y splits the I reduction (ksplit > 1 writes partial sums to
// out + split * O*R*J, summed in fixed order by k_sum_splits).
// block 128 (4 warps x 16 columns).
template <int RP, int VEC>
__global__ void __launch_bounds__(128) k_ttm_mid(const double* __restrict__ X, long long O, int I,
                                                 long long J, const double* __restrict__ A, int R,
                                                 double* __restrict__ out, int ich) {
  constexpr int BJ = 64;
  constexpr int LD = BJ + kPadX;
  extern __shared__ __align__(16) double xs[];  // [kStages][kBK][LD]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long ncol = O * J;
  const long long c0 = (long long)blockIdx.x * BJ;
  const int ibeg = blockIdx.y * ich, iend = min(I, ibeg + ich);
  const int nchunks = ceil_div(iend - ibeg, kBK);
  double* dst_out = out + (long long)blockIdx.y * O * R * J;

  // whole tile inside one o (J % 64 == 0): no per-element index division
  const bool one_o = (J % BJ) == 0;
  const long long o_t = one_o ? c0 / J : 0, j_t = one_o ? c0 - o_t * J : 0;
  auto load_chunk = [&](int c, int stage) {
    double* dst = xs + stage * kBK * LD;
    const int i0 = ibeg + c * kBK;
    constexpr int PER_ROW = BJ / VEC;
    for (int e = tid; e < kBK * PER_ROW; e += 128) {
      const int r = e / PER_ROW, col = (e % PER_ROW) * VEC;
      const long long cc = c0 + col;
      const bool ok = (i0 + r < iend) && (cc < ncol);
      long long o, j;
      if (one_o) {
        o = o_t;
        j = j_t + col;
      } else {
        o = ok ? cc / J : 0;
        j = ok ? cc - o * J : 0;
      }
      const double* src = ok ? X + (o * I + i0 + r) * J + j : X;
      if (VEC == 2)
        cp_async16(dst + r * LD + col, src, ok);
      else
        cp_async8(dst + r * LD + col, src, ok);
    }
  };

  double acc[RP / 8][2][2];
#pragma unroll
  for (int mt = 0; mt < RP / 8; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nchunks) load_chunk(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (c + kStages - 1 < nchunks) load_chunk(c + kStages - 1, (c + kStages - 1) % kStages);
    cp_async_commit();
    const double* xt = xs + (c % kStages) * kBK * LD;
    const int i0 = ibeg + c * kBK;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const int i = i0 + ks * 4 + t;
      double af[RP / 8];
#pragma unroll
      for (int mt = 0; mt < RP / 8; ++mt) {
        const int r = mt * 8 + g;
        af[mt] = (i < iend && r < R) ? __ldg(A + (size_t)i * R + r) : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const double bf = xt[(ks * 4 + t) * LD + warp * 16 + nt * 8 + g];
#pragma unroll
        for (int mt = 0; mt < RP / 8; ++mt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf);
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int mt = 0; mt < RP / 8; ++mt) {
    const int r = mt * 8 + g;
    if (r >= R) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long cc = c0 + warp * 16 + nt * 8 + 2 * t + h;
        if (cc < ncol) {
          const long long o = one_o ? o_t : cc / J;
          const long long j = one_o ? j_t + (cc - c0) : cc - o * J;
          dst_out[(o * R + r) * J + j] = acc[mt][nt][h];
        }
      }
    }
  }
}

// Persistent strided-mode contraction for large column counts (the F_N projection
// X x_1 A_1^T): A^T (R x I, padded) resident in shared memory, 128-column tiles (8
// warps x 16 columns) of X streamed through a KS-deep cp.async pipeline that runs
// across tiles; every DMMA operand from shared memory. Requires J % 128 == 0 (a
// tile never straddles two o).
constexpr int BJ2 = 128;
constexpr int kStagesMid = 4;
#ifndef RTB_MIDKB
#define RTB_MIDKB 64
#define RTB_MIDST 2
#endif
constexpr int kMidKB = RTB_MIDKB;      // k_ttm_mid3: rows of X (reduction index) per chunk
constexpr int kMidStages = RTB_MIDST;  // k_ttm_mid3: ring depth
template <int RP, bool COMPUTE = true>
__global__ void __launch_bounds__(256, 1) k_ttm_mid2(const double* __restrict__ X, long long O,
                                                     int I, long long J,
                                                     const double* __restrict__ A, int R,
                                                     double* __restrict__ out) {
  constexpr int LDX = BJ2 + 8;     // (8t + g) mod 16 -> 2-way at most
  extern __shared__ __align__(16) double sm3[];
  const int Ip = ceil_div(I, kBK) * kBK;
  const int LDT = Ip + 4;                 // A^T rows: (4g + t) mod 16 -> 2-way at most
  double* at = sm3;                       // [RP][LDT]
  double* xs = at + (size_t)RP * LDT;     // [kStagesMid][kBK][LDX]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long ntiles = O * J / BJ2;
  const int nchunks = ceil_div(I, kBK);
  for (int e = tid; e < RP * LDT; e += 256) {
    const int r = e / LDT, i = e - r * LDT;
    at[e] = (i < I && r < R) ? A[(size_t)i * R + r] : 0.0;
  }
  const long long my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nitems = my_tiles * nchunks;
  auto load_item = [&](long long q, int stage) {
    const long long tile = blockIdx.x + (q / nchunks) * gridDim.x;
    const int c = (int)(q % nchunks);
    const long long c0 = tile * BJ2;
    const long long o = c0 / J, j0 = c0 - o * J;
    const int i0 = c * kBK;
    double* dst = xs + (size_t)stage * kBK * LDX;
    for (int e = tid; e < kBK * (BJ2 / 2); e += 256) {
      const int r = e / (BJ2 / 2), col = (e % (BJ2 / 2)) * 2;
      const bool ok = i0 + r < I;
      cp_async16(dst + r * LDX + col, ok ? X + (o * I + i0 + r) * J + j0 + col : X, ok);
    }
  };
#pragma unroll
  for (int sidx = 0; sidx < kStagesMid - 1; ++sidx) {
    if (sidx < nitems) load_item(sidx, sidx);
    cp_async_commit();
  }
  // two accumulator sets (even / odd k steps): twice the independent DMMA chains
  double acc[2][RP / 8][2][2];
  for (long long q = 0; q < nitems; ++q) {
    const int c = (int)(q % nchunks);
    if (c == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int mt = 0; mt < RP / 8; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) acc[h][mt][nt][0] = acc[h][mt][nt][1] = 0.0;
    }
    cp_async_wait<kStagesMid - 2>();
    __syncthreads();
    if (q + kStagesMid - 1 < nitems)
      load_item(q + kStagesMid - 1, (int)((q + kStagesMid - 1) % kStagesMid));
    cp_async_commit();
    const double* xt = xs + (size_t)(q % kStagesMid) * kBK * LDX + warp * 16;
    const int i0 = c * kBK;
    if (!COMPUTE) {
      acc[0][0][0][0] += xt[lane];  // touch the stage, no contraction (bandwidth probe)
      continue;
    }
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      double af[RP / 8];
#pragma unroll
      for (int mt = 0; mt < RP / 8; ++mt) af[mt] = at[(size_t)(mt * 8 + g) * LDT + i0 + ks * 4 + t];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const double bf = xt[(ks * 4 + t) * LDX + nt * 8 + g];
#pragma unroll
        for (int mt = 0; mt < RP / 8; ++mt)
          dmma_8x8x4(acc[ks & 1][mt][nt][0], acc[ks & 1][mt][nt][1], af[mt], bf);
      }
    }
    if (c == nchunks - 1) {
      const long long tile = blockIdx.x + (q / nchunks) * gridDim.x;
      const long long c0 = tile * BJ2;
      const long long o = c0 / J, j0 = c0 - o * J + warp * 16;
#pragma unroll
      for (int mt = 0; mt < RP / 8; ++mt) {
        const int r = mt * 8 + g;
        if (r >= R) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          double2 v2;
          v2.x = acc[0][mt][nt][0] + acc[1][mt][nt][0];
          v2.y = acc[0][mt][nt][1] + acc[1][mt][nt][1];
          *reinterpret_cast<double2*>(out + (o * R + r) * J + j0 + nt * 8 + 2 * t) = v2;
        }
      }
    }
  }
  cp_async_wait<0>();
}

// Producer / consumer version of the same pass: warp 8 only issues the cp.async
// copies of the ring (and arrives on full[s] when they land), warps 0-7 only compute
// and release a stage with one arrive on empty[s]. No block-wide barrier per chunk,
// so the consumer warps drift and the DMMA pipe does not drain between chunks.
template <int RP, bool COMPUTE = true>
__global__ void __launch_bounds__(288, 1) k_ttm_mid3(const double* __restrict__ X, long long O,
                                                     int I, long long J,
                                                     const double* __restrict__ A, int R,
                                                     double* __restrict__ out) {
  constexpr int LDX = BJ2 + 8;
  constexpr int S = kMidStages;
  extern __shared__ __align__(16) double sm3[];
  __shared__ __align__(8) unsigned long long full[S], empty[S];
  const int Ip = ceil_div(I, kMidKB) * kMidKB;
  const int LDT = Ip + 4;
  double* at = sm3;                       // [RP][LDT]
  double* xs = at + (size_t)RP * LDT;     // [S][kMidKB][LDX]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long ntiles = O * J / BJ2;
  const int nchunks = ceil_div(I, kMidKB);
  for (int e = tid; e < RP * LDT; e += blockDim.x) {
    const int r = e / LDT, i = e - r * LDT;
    at[e] = (i < I && r < R) ? A[(size_t)i * R + r] : 0.0;
  }
  // stages zeroed once: rows of a short last chunk are never copied
  for (int e = tid; e < S * kMidKB * LDX; e += blockDim.x) xs[e] = 0.0;
  if (tid == 0) {
    for (int s2 = 0; s2 < S; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], 8);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const long long my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nitems = my_tiles * nchunks;
  if (warp == 8) {
    // producer: one 1 KB bulk copy (TMA, cp.async.bulk) per row of the chunk, all
    // completing on full[s] with the expected byte count
    for (long long q = 0; q < nitems; ++q) {
      const int st = (int)(q % S);
      if (q >= S) mbar_wait(&empty[st], (unsigned)(((q / S) - 1) & 1));
      const long long tile = blockIdx.x + (q / nchunks) * gridDim.x;
      const int c = (int)(q % nchunks);
      const long long c0 = tile * BJ2;
      const long long o = c0 / J, j0 = c0 - o * J;
      const int i0 = c * kMidKB;
      const int rows = min(kMidKB, I - i0);
      double* dst = xs + (size_t)st * kMidKB * LDX;
      if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&full[st], (unsigned)(rows * BJ2 * 8));
      }
      __syncwarp();
      for (int rr = lane; rr < rows; rr += 32)
        bulk_g2s(dst + rr * LDX, X + (o * I + i0 + rr) * J + j0, BJ2 * 8, &full[st]);
    }
    return;
  }
  double acc[RP / 8][2][2];
  for (long long q = 0; q < nitems; ++q) {
    const int st = (int)(q % S);
    const int c = (int)(q % nchunks);
    if (c == 0) {
#pragma unroll
      for (int mt = 0; mt < RP / 8; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    }
    mbar_wait(&full[st], (unsigned)((q / S) & 1));
    const double* xt = xs + (size_t)st * kMidKB * LDX + warp * 16;
    const int i0 = c * kMidKB;
    if (!COMPUTE) {
      acc[0][0][0] += xt[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      continue;
    }
#pragma unroll
    for (int ks = 0; ks < kMidKB / 4; ++ks) {
      double af[RP / 8];
#pragma unroll
      for (int mt = 0; mt < RP / 8; ++mt) af[mt] = at[(size_t)(mt * 8 + g) * LDT + i0 + ks * 4 + t];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const double bf = xt[(ks * 4 + t) * LDX + nt * 8 + g];
#pragma unroll
        for (int mt = 0; mt < RP / 8; ++mt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (c == nchunks - 1) {
      const long long tile = blockIdx.x + (q / nchunks) * gridDim.x;
      const long long c0 = tile * BJ2;
      const long long o = c0 / J, j0 = c0 - o * J + warp * 16;
#pragma unroll
      for (int mt = 0; mt < RP / 8; ++mt) {
        const int r = mt * 8 + g;
        if (r >= R) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          double2 v2;
          v2.x = acc[mt][nt][0];
          v2.y = acc[mt][nt][1];
          *reinterpret_cast<double2*>(out + (o * R + r) * J + j0 + nt * 8 + 2 * t) = v2;
        }
      }
    }
  }
}

constexpr int kMid5KB = 32, kMid5St = 4;  // k_ttm_mid5: rows per box, ring depth
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// row-major O x I FP64 matrix as 128-row x 16-column boxes, SWIZZLE_128B, zero OOB fill
static bool x_tensor_map(CUtensorMap* m, const double* X, long long O, int I) {
  auto enc = tmap_encode();
  if (!enc || (I % 2) || (reinterpret_cast<uintptr_t>(X) & 15) || O >= (1LL << 31)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)I, (cuuint64_t)O};
  cuuint64_t strides[1] = {(cuuint64_t)I * 8};
  cuuint32_t box[2] = {16, (cuuint32_t)BM2};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// X (O, I, J) row-major FP64 as 16 (j) x kMid5KB (i) x 1 (o) boxes, SWIZZLE_128B, zero OOB fill
static bool mid_tensor_map(CUtensorMap* m, const double* X, long long O, int I, long long J,
                           int kb = kMid5KB) {
  auto enc = tmap_encode();
  if (!enc || (J % 2) || (reinterpret_cast<uintptr_t>(X) & 15) || J >= (1LL << 31) ||
      O >= (1LL << 31))
    return false;
  cuuint64_t dims[3] = {(cuuint64_t)J, (cuuint64_t)I, (cuuint64_t)O};
  cuuint64_t strides[2] = {(cuuint64_t)J * 8, (cuuint64_t)I * J * 8};
  cuuint32_t box[3] = {16, (cuuint32_t)kb, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(X), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// k_ttm_mid3 with the X tiles moved by tensor-map TMA: one 3-D box (16 columns x kMid5KB
// rows x 1, SWIZZLE_128B) per consumer warp and stage, 8 boxes per stage issued by one lane
// of the producer warp (k_ttm_mid3 issues one bulk copy per row: ~64 per stage, serialised
// in the producer, which bounded that kernel). Rows past I arrive zero-filled. Conflict-free
// B fragments of the swizzled box come from relabelling the reduction index: slot
// kappa = 4 ks + t of each 16-row block reads X row sigma(kappa) = 2 t + (ks & 1) + 8 (ks >> 1)
// (rows 2t + b sit in distinct 16-byte chunk pairs after the XOR), and A^T is staged with its
// columns in the same order.
// Rank 32 (C5): A^T (32 x I) takes 132 KB of shared memory at I = 512, so the ring holds five
// stages of 16-row boxes (KB = 16) instead of four of 32.
template <int RP, int KB = kMid5KB, int S = kMid5St>
__global__ void __launch_bounds__(288, 1) k_ttm_mid5(const __grid_constant__ CUtensorMap xmap,
                                                     long long O, int I, long long J,
                                                     const double* __restrict__ A, int R,
                                                     double* __restrict__ out) {
  constexpr int kBox = KB * 16;  // doubles per box
  extern __shared__ __align__(1024) double sm5m[];
  double* xs = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sm5m) + 1023) & ~uintptr_t(1023));
  double* at = xs + (size_t)S * 8 * kBox;  // [RP][LDT], columns in sigma order
  __shared__ __align__(8) unsigned long long full[S], empty[S];
  const int Ip = ceil_div(I, KB) * KB;
  const int LDT = Ip + 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long ntiles = O * J / BJ2;
  const int nchunks = ceil_div(I, KB);
  for (int e = tid; e < RP * LDT; e += blockDim.x) {
    const int r = e / LDT, i = e - r * LDT;
    const int kap = i & 15;
    const int src = (i & ~15) | (2 * (kap & 3) + ((kap >> 2) & 1) + 8 * ((kap >> 3) & 1));
    at[e] = (i < Ip && src < I && r < R) ? A[(size_t)src * R + r] : 0.0;
  }
  if (tid == 0) {
    for (int s2 = 0; s2 < S; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], 8);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const long long my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nitems = my_tiles * nchunks;
  if (warp == 8) {
    if (lane == 0) {
      for (long long q = 0; q < nitems; ++q) {
        const int st = (int)(q % S);
        if (q >= S) mbar_wait(&empty[st], (unsigned)(((q / S) - 1) & 1));
        const long long tile = blockIdx.x + (q / nchunks) * gridDim.x;
        const int c = (int)(q % nchunks);
        const long long c0 = tile * BJ2;
        const long long o = c0 / J, j0 = c0 - o * J;
        double* dst = xs + (size_t)st * 8 * kBox;
        mbar_arrive_expect_tx(&full[st], 8u * kBox * 8u);
        for (int w = 0; w < 8; ++w)
          tma_load_3d(dst + w * kBox, &xmap, (int)(j0 + 16 * w), c * KB, (int)o, &full[st]);
      }
    }
    return;
  }
  double acc[RP / 8][2][2];
  for (long long q = 0; q < nitems; ++q) {
    const int st = (int)(q % S);
    const int c = (int)(q % nchunks);
    if (c == 0) {
#pragma unroll
      for (int mt = 0; mt < RP / 8; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    }
    mbar_wait(&full[st], (unsigned)((q / S) & 1));
    const double* xb = xs + (size_t)st * 8 * kBox + warp * kBox;
    const int i0 = c * KB;
#pragma unroll
    for (int ks = 0; ks < KB / 4; ++ks) {
      double af[RP / 8];
#pragma unroll
      for (int mt = 0; mt < RP / 8; ++mt) af[mt] = at[(size_t)(mt * 8 + g) * LDT + i0 + ks * 4 + t];
      const int ksl = ks & 3;
      const int row = 16 * (ks >> 2) + 2 * t + (ksl & 1) + 8 * (ksl >> 1);
      const int sw = row & 7;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const double bf = xb[row * 16 + (((4 * nt + (g >> 1)) ^ sw) << 1) + (g & 1)];
#pragma unroll
        for (int mt = 0; mt < RP / 8; ++mt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (c == nchunks - 1) {
      const long long tile = blockIdx.x + (q / nchunks) * gridDim.x;
      const long long c0 = tile * BJ2;
      const long long o = c0 / J, j0 = c0 - o * J + warp * 16;
#pragma unroll
      for (int mt = 0; mt < RP / 8; ++mt) {
        const int r = mt * 8 + g;
        if (r >= R) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          double2 v2;
          v2.x = acc[mt][nt][0];
          v2.y = acc[mt][nt][1];
          *reinterpret_cast<double2*>(out + (o * R + r) * J + j0 + nt * 8 + 2 * t) = v2;
        }
      }
    }
  }
}
static size_t mid5_smem(int I, int rp, int kb = kMid5KB, int st = kMid5St) {
  const size_t ip = (size_t)ceil_div(I, kb) * kb;
  return (size_t)st * 8 * kb * 16 * 8 + 1024 + (size_t)rp * (ip + 4) * 8;
}

static size_t mid3_smem(int I, int rp) {
  const size_t ip = (size_t)ceil_div(I, kMidKB) * kMidKB;
  return ((size_t)rp * (ip + 4) + (size_t)kMidStages * kMidKB * (BJ2 + 8)) * 8;
}
static size_t mid2_smem(int I, int rp) {
  const size_t ip = (size_t)ceil_div(I, kBK) * kBK;
  return ((size_t)rp * (ip + 4) + (size_t)kStagesMid * kBK * (BJ2 + 8)) * 8;
}

__global__ void k_sum_splits(const double* __restrict__ part, long long n, int splits,
                             double* __restrict__ out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = 0.0;
  for (int k = 0; k < splits; ++k) s += part[(long long)k * n + e];
  out[e] = s;
}

// ---------------------------------------------------------------------------
// Scalar fallback: out[o,r,j] = sum_i W[r*wr + i*wi] X[o,i,j].
__global__ void k_ttm_generic(const double* __restrict__ X, long long O, int I, long long J,
                              const double* __restrict__ W, long long wr, long long wi, int R,
                              double* __restrict__ out, const int* __restrict__ need) {
  RTB_GUARD()
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = O * R * J;
  if (e >= total) return;
  const long long j = e % J;
  const int r = (int)((e / J) % R);
  const long long o = e / (J * R);
  const double* x = X + o * I * J + j;
  double s = 0.0;
  for (int i = 0; i < I; ++i) s += W[r * wr + i * wi] * x[(long long)i * J];
  out[e] = s;
}

// M[i,r] = sum_{o,j} Y[o,i,j] G[o,r,j]; Y (O,I,J), G (O,R,J).
// One block per i; threads stride over (o,j), accumulate all r in registers,
// then a fixed-order smem reduction (deterministic).
template <int RM>
__global__ void __launch_bounds__(128) k_contract_except(const double* __restrict__ Y,
                                                         const double* __restrict__ G,
                                                         long long O, int I, int R, long long J,
                                                         double* __restrict__ M) {
  __shared__ double part[128][RM + 1];
  const int i = blockIdx.x, tid = threadIdx.x;
  double acc[RM];
#pragma unroll
  for (int r = 0; r < RM; ++r) acc[r] = 0.0;
  const long long n = O * J;
  for (long long t = tid; t < n; t += 128) {
    const long long o = t / J, j = t % J;
    const double y = Y[(o * I + i) * J + j];
    const double* g = G + o * R * J + j;
#pragma unroll
    for (int r = 0; r < RM; ++r)
      if (r < R) acc[r] += y * g[(long long)r * J];
  }
#pragma unroll
  for (int r = 0; r < RM; ++r) part[tid][r] = acc[r];
  __syncthreads();
  if (tid < R) {
    double s = 0.0;
    for (int k = 0; k < 128; ++k) s += part[k][tid];
    M[(long long)i * R + tid] = s;
  }
}

// scalar fallback for R > 32: one thread per (i, r)
__global__ void k_contract_except_scalar(const double* __restrict__ Y,
                                         const double* __restrict__ G, long long O, int I, int R,
                                         long long J, double* __restrict__ M) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)I * R) return;
  const int i = (int)(e / R), r = (int)(e % R);
  double s = 0.0;
  for (long long o = 0; o < O; ++o) {
    const double* y = Y + (o * I + i) * J;
    const double* gg = G + (o * R + r) * J;
    for (long long j = 0; j < J; ++j) s += y[j] * gg[j];
  }
  M[e] = s;
}

// out[o,r,j] = sum_i A[i,r] X[o,i,j] for a short contiguous tail J (<= 32):
// one block per o, i streamed in chunks of 32 through smem, one thread per
// (r, j) output (R*J <= 1024).
__global__ void __launch_bounds__(256) k_ttm_smallj(const double* __restrict__ X, int I, int J,
                                                   const double* __restrict__ A, int R,
                                                   double* __restrict__ out) {
  __shared__ double xs[32][33];
  __shared__ double as[32][33];
  const long long o = blockIdx.x;
  const double* Xo = X + o * (long long)I * J;
  const int tid = threadIdx.x;
  const int nout = R * J;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i0 = 0; i0 < I; i0 += 32) {
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += 256) {
      const int ii = e >> 5, c = e & 31;
      xs[ii][c] = (i0 + ii < I && c < J) ? Xo[(long long)(i0 + ii) * J + c] : 0.0;
      as[ii][c] = (i0 + ii < I && c < R) ? A[(long long)(i0 + ii) * R + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + q * 256;
      if (e < nout) {
        const int r = e / J, j = e % J;
        double sacc = acc[q];
#pragma unroll 8
        for (int ii = 0; ii < 32; ++ii) sacc += as[ii][r] * xs[ii][j];
        acc[q] = sacc;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = tid + q * 256;
    if (e < nout) out[o * nout + e] = acc[q];
  }
}

// Up-projection out[o,i,j] = sum_r A[i,r] Y[o,r,j] (R small): Y[o] and the
// block's A rows staged in smem; grid (ceil(I/ICH), O), threads over (i, j).
__global__ void __launch_bounds__(256) k_ttm_expand(const double* __restrict__ Y, int R,
                                                   long long J, const double* __restrict__ A,
                                                   int I, int ich, double* __restrict__ out,
                                                   const int* __restrict__ need) {
  RTB_GUARD()
  extern __shared__ double ys[];  // R x J, then ich x R
  double* as = ys + (long long)R * J;
  const long long o = blockIdx.y;
  const int i0 = blockIdx.x * ich;
  const double* Yo = Y + o * R * J;
  for (long long e = threadIdx.x; e < (long long)R * J; e += 256) ys[e] = Yo[e];
  for (int e = threadIdx.x; e < ich * R; e += 256) {
    const int ii = e / R;
    as[e] = (i0 + ii < I) ? A[(long long)(i0 + ii) * R + e % R] : 0.0;
  }
  __syncthreads();
  const int Ji = (int)J;  // R * J fits shared memory, so J is small
  const int n = ich * Ji;
  for (int e = threadIdx.x; e < n; e += 256) {
    const int ii = e / Ji;
    const int j = e - ii * Ji;
    const int i = i0 + ii;
    if (i >= I) continue;
    const double* a = as + ii * R;
    double s0 = 0.0, s1 = 0.0;
    int r = 0;
    for (; r + 1 < R; r += 2) {
      s0 = fma(a[r], ys[r * Ji + j], s0);
      s1 = fma(a[r + 1], ys[(r + 1) * Ji + j], s1);
    }
    if (r < R) s0 = fma(a[r], ys[r * Ji + j], s0);
    out[(o * I + i) * J + j] = s0 + s1;
  }
}

// Same up-projection for R, J <= 16 on the FP64 tensor cores: per o, a warp's 16 output rows x 16
// columns are out = A[rows, :] (16 x R) x Y[o] (R x J) as two m16n8k16 DMMAs, the A fragment
// loaded once per warp, Y[o] staged in shared memory per CTA. The row-owner kernel below was
// bound by shared-memory instruction throughput (two LDS per FMA pair; L1/TEX 80% at 28 us).
__global__ void __launch_bounds__(256) k_ttm_expand_dmma(const double* __restrict__ Y, int R, int J,
                                                        const double* __restrict__ A, int I,
                                                        long long O, int och,
                                                        double* __restrict__ out,
                                                        const int* __restrict__ need) {
  RTB_GUARD()
  __shared__ double ys[16 * 16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int i0 = blockIdx.x * 128 + warp * 16;
  double a[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int row = i0 + g + 8 * (v & 1), k = t + 4 * (v >> 1);
    a[v] = (row < I && k < R) ? A[(long long)row * R + k] : 0.0;
  }
  const long long o0 = (long long)blockIdx.y * och;
  const long long o1 = o0 + och < O ? o0 + och : O;
  for (long long o = o0; o < o1; ++o) {
    __syncthreads();
    {
      const int e = threadIdx.x;  // 256 = 16 x 16
      const int k = e >> 4, j = e & 15;
      ys[e] = (k < R && j < J) ? Y[(o * R + k) * J + j] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      double b[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) b[v] = ys[(t + 4 * v) * 16 + nt * 8 + g];
      double c[4] = {0.0, 0.0, 0.0, 0.0};
      dmma_16x8x16(c, a, b);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int row = i0 + g + 8 * (v >> 1), col = nt * 8 + 2 * t + (v & 1);
        if (row < I && col < J) out[(o * I + row) * J + col] = c[v];
      }
    }
  }
}

// Same up-projection for R, J <= 16 (P = W x_2 A_2 at C2: 512 o x 512 i x 16 j): a thread owns
// one output row i (A[i, :] in registers) and all J outputs of it, for och consecutive o; Y[o]
// (R x J) is staged in shared memory and read as broadcasts. The general kernel above reads two
// shared operands per FMA and was bound by shared-memory wavefronts there (40 us).
template <int RM, int JM>
__global__ void __launch_bounds__(256) k_ttm_expand_rows(const double* __restrict__ Y, int R, int J,
                                                        const double* __restrict__ A, int I,
                                                        long long O, int och,
                                                        double* __restrict__ out,
                                                        const int* __restrict__ need) {
  RTB_GUARD()
  __shared__ __align__(16) double ys[RM * JM];
  __shared__ __align__(16) double ot[8][32 * (JM + 1)];  // per warp: 32 rows of outputs
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double a[RM];
#pragma unroll
  for (int r = 0; r < RM; ++r) a[r] = (i < I && r < R) ? A[(long long)i * R + r] : 0.0;
  const long long o0 = (long long)blockIdx.y * och;
  const long long o1 = o0 + och < O ? o0 + och : O;
  for (long long o = o0; o < o1; ++o) {
    __syncthreads();
    for (int e = threadIdx.x; e < RM * JM; e += 256) {
      const int r = e / JM, j = e - r * JM;
      ys[e] = (r < R && j < J) ? Y[(o * R + r) * J + j] : 0.0;
    }
    __syncthreads();
    double acc[JM];
#pragma unroll
    for (int j = 0; j < JM; ++j) acc[j] = 0.0;
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
      for (int j = 0; j < JM; j += 2) {
        const double2 y2 = *reinterpret_cast<const double2*>(ys + r * JM + j);  // broadcast
        acc[j] = fma(a[r], y2.x, acc[j]);
        acc[j + 1] = fma(a[r], y2.y, acc[j + 1]);
      }
    // the warp's 32 rows x J outputs are one contiguous run: stage them and store coalesced
    double* ow = ot[warp];
#pragma unroll
    for (int j = 0; j < JM; ++j) ow[lane * (JM + 1) + j] = acc[j];
    __syncwarp();
    const int wi0 = blockIdx.x * 256 + warp * 32;
    const int nr = min(32, I - wi0);
    double* op = out + (o * I + wi0) * J;
    for (int e = lane; e < nr * J; e += 32) {
      const int rr = e / J, j = e - rr * J;
      op[e] = ow[rr * (JM + 1) + j];
    }
    __syncwarp();
  }
}

// Deterministic sum of per-block partials (fixed order), one block.
__global__ void k_sum_partials(const double* __restrict__ partial, long long n,
                               double* __restrict__ out, const int* __restrict__ need) {
  RTB_GUARD()
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
  s = block_sum<1024>(s, red);
  if (threadIdx.x == 0) *out = s;
}

// ---------------------------------------------------------------------------
// Host launchers.

// grid of the last partial-producing last-mode launch of this host thread (ttm_last_blocks)
static thread_local long long t_last_parts = -1;

template <int RP, int VEC, bool FUSED>
static void launch_last(const double* X, long long O, int I, const double* A, int R, double* T,
                        const double* P, double* partial, cudaStream_t st) {
  constexpr int smem = kStages * 64 * (kBK + kPadX) * sizeof(double);
  auto k = k_ttm_last<RP, VEC, FUSED>;
  set_max_smem(k, (int)smem);
  const long long blocks = ceil_div<long long>(O, 64);
  k<<<(unsigned)blocks, 128, smem, st>>>(X, O, I, A, R, T, P, partial, g_need);
  t_last_parts = blocks;
  RTB_LAUNCH_CHECK();
}

void set_ttm_guard(const int* need) { g_need = need; }

// Same pass with m16n8k16 DMMA (R <= 16): per 32-column chunk a T warp issues 4 MMAs
// (2 k-steps x 2 n-tiles over the rank) and a residual warp 4 (one per 8 columns, K =
// rank), each fed straight from shared memory, instead of 32 m8n8k4 each.
template <bool FUSED, int BK, int ST>
__global__ void __launch_bounds__(512, 1) k_ttm_last3(const double* __restrict__ X, long long O,
                                                      int I, const double* __restrict__ A, int R,
                                                      double* __restrict__ T,
                                                      const double* __restrict__ P,
                                                      double* __restrict__ partial,
                                                      const int* __restrict__ need) {
  RTB_GUARD()
  constexpr int RP = 16;
  constexpr int LD = BK + kPadX;
  constexpr int LDA = RP + 4;
  constexpr int ROWS = 16;  // rows per warp (m16)
  extern __shared__ __align__(16) double sm2[];
  const int Ip = ceil_div(I, BK) * BK;
  double* as = sm2;                        // [Ip][LDA]
  double* xs = as + (size_t)Ip * LDA;      // [ST][BM2][LD]
  __shared__ double red[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  // FUSED: warps 0-7 T, 8-15 residual, 16 rows each; else 8 warps (128 rows) of T
  const bool rwarp = FUSED && warp >= 8;
  const int wrow = warp & 7;
  const bool idle = !FUSED && warp >= 8;
  const long long nrb = ceil_div<long long>(O, BM2);
  const int nchunks = ceil_div(I, BK);
  for (int e = tid; e < Ip * LDA; e += 512) {
    const int i = e / LDA, r = e - i * LDA;
    as[e] = (i < I && r < R) ? A[(size_t)i * R + r] : 0.0;
  }
  const long long my_blocks = blockIdx.x < nrb ? (nrb - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nitems = my_blocks * nchunks;
  auto load_item = [&](long long q, int stage) {
    const long long rb = blockIdx.x + (q / nchunks) * gridDim.x;
    const int c = (int)(q % nchunks);
    const long long o0 = rb * BM2;
    const int i0 = c * BK;
    double* dst = xs + (size_t)stage * BM2 * LD;
    for (int e = tid; e < BM2 * (BK / 2); e += 512) {
      const int r = e / (BK / 2), col = (e % (BK / 2)) * 2;
      const long long o = o0 + r;
      const bool ok = (o < O) && (i0 + col < I);
      cp_async16(dst + r * LD + col, ok ? X + o * I + i0 + col : X, ok);
    }
  };
#pragma unroll
  for (int sidx = 0; sidx < ST - 1; ++sidx) {
    if (sidx < nitems) load_item(sidx, sidx);
    cp_async_commit();
  }
  double acc[2][4];   // T: two n-tiles (rank 0-7, 8-15) of the 16 x 16 block
  double pa[8];       // residual: P rows as the A fragment (constant per row block)
  double resid0 = 0.0, resid1 = 0.0;
  for (long long q = 0; q < nitems; ++q) {
    const int c = (int)(q % nchunks);
    const long long rb = blockIdx.x + (q / nchunks) * gridDim.x;
    const long long o0 = rb * BM2 + wrow * ROWS;
    if (c == 0) {
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[n][v] = 0.0;
      if (rwarp) {
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const long long o = o0 + g + 8 * (v & 1);
          const int k = t + 4 * (v >> 1);
          pa[v] = (o < O && k < R) ? P[o * R + k] : 0.0;
        }
      }
    }
    cp_async_wait<ST - 2>();
    __syncthreads();
    if (q + ST - 1 < nitems) load_item(q + ST - 1, (int)((q + ST - 1) % ST));
    cp_async_commit();
    const double* xt = xs + (size_t)(q % ST) * BM2 * LD + wrow * ROWS * LD;
    const int i0 = c * BK;
    if (idle) {
    } else if (!rwarp) {
#pragma unroll
      for (int kb = 0; kb < BK; kb += 16) {
        double a[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) a[v] = xt[(g + 8 * (v & 1)) * LD + kb + t + 4 * (v >> 1)];
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          double b[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) b[v] = as[(size_t)(i0 + kb + t + 4 * v) * LDA + n * 8 + g];
          dmma_16x8x16(acc[n], a, b);
        }
      }
      if (c == nchunks - 1) {
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const long long o = o0 + g + 8 * (v >> 1);
            const int r = n * 8 + 2 * t + (v & 1);
            if (o < O && r < R) T[o * R + r] = acc[n][v];
          }
      }
    } else {
#pragma unroll
      for (int nb = 0; nb < BK; nb += 8) {
        double b[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) b[v] = as[(size_t)(i0 + nb + g) * LDA + t + 4 * v];
        double cx[4] = {0.0, 0.0, 0.0, 0.0};
        dmma_16x8x16(cx, pa, b);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 xv = *reinterpret_cast<const double2*>(xt + (g + 8 * h) * LD + nb + 2 * t);
          const double d0 = xv.x - cx[2 * h], d1 = xv.y - cx[2 * h + 1];
          resid0 = fma(d0, d0, resid0);  // zero-filled tails contribute exactly 0
          resid1 = fma(d1, d1, resid1);
        }
      }
    }
  }
  cp_async_wait<0>();
  if (FUSED) {
    const double s = block_sum<512>(resid0 + resid1, red);
    if (tid == 0) partial[blockIdx.x] = s;
  }
}

// k_ttm_last3 without CTA-wide barriers: the X ring is filled by TMA bulk row copies and
// handed over by mbarriers. T warp w (rows 16 w .. 16 w + 15 of the row block) also stages
// those 16 rows of every chunk: before computing item q it refills the slot of item q - 1
// (freed when all 16 warps arrived on that slot's `empty` barrier) with item q + ST - 1,
// each of its lanes 0-15 copying one row segment onto the slot's `full` barrier (8 arrivals
// + transaction bytes). Residual warp w + 8 reads the same rows. The warps of a CTA drift by
// up to ST - 1 chunks, so the DMMA pipe is not drained at every chunk boundary.
template <bool FUSED, int BK, int ST>
__global__ void __launch_bounds__(512, 1) k_ttm_last4(const double* __restrict__ X, long long O,
                                                      int I, const double* __restrict__ A, int R,
                                                      double* __restrict__ T,
                                                      const double* __restrict__ P,
                                                      double* __restrict__ partial,
                                                      const int* __restrict__ need) {
  RTB_GUARD()
  constexpr int RP = 16;
  constexpr int LD = BK + kPadX;
  constexpr int LDA = RP + 4;
  constexpr int ROWS = 16;  // rows per warp (m16)
  extern __shared__ __align__(16) double sm4[];
  const int Ip = ceil_div(I, BK) * BK;
  double* as = sm4;                        // [Ip][LDA]
  double* xs = as + (size_t)Ip * LDA;      // [ST][BM2][LD]
  __shared__ double red[32];
  __shared__ __align__(8) unsigned long long full[ST], empty[ST];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const bool rwarp = FUSED && warp >= 8;
  const int wrow = warp & 7;
  const bool idle = !FUSED && warp >= 8;
  const long long nrb = ceil_div<long long>(O, BM2);
  const int nchunks = ceil_div(I, BK);
  for (int e = tid; e < Ip * LDA; e += 512) {
    const int i = e / LDA, r = e - i * LDA;
    as[e] = (i < I && r < R) ? A[(size_t)i * R + r] : 0.0;
  }
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 8);
      mbar_init(&empty[i], FUSED ? 16 : 8);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const long long my_blocks = blockIdx.x < nrb ? (nrb - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nitems = my_blocks * nchunks;
  // T warp: stage its 16 rows of item q into slot q % ST
  auto stage_rows = [&](long long q) {
    const int slot = (int)(q % ST);
    const long long rb = blockIdx.x + (q / nchunks) * gridDim.x;
    const int c = (int)(q % nchunks);
    const long long o = rb * BM2 + wrow * ROWS + lane;
    const int i0 = c * BK;
    const int cols = min(BK, I - i0);
    const long long rem = O - (rb * BM2 + wrow * ROWS);
    const int rows_ok = rem < ROWS ? (rem > 0 ? (int)rem : 0) : ROWS;
    double* dst = xs + ((size_t)slot * BM2 + wrow * ROWS + lane) * LD;
    if (lane < ROWS) {  // zero what the copies do not cover (row / column tails)
      if (lane >= rows_ok) {
        for (int k = 0; k < BK; ++k) dst[k] = 0.0;
      } else {
        for (int k = cols; k < BK; ++k) dst[k] = 0.0;
      }
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0)
      mbar_arrive_expect_tx(&full[slot], (unsigned)rows_ok * cols * 8u);
    __syncwarp();
    if (lane < rows_ok) bulk_g2s(dst, X + o * I + i0, (unsigned)cols * 8u, &full[slot]);
  };
  if (!rwarp && !idle) {
    for (long long q = 0; q < ST - 1 && q < nitems; ++q) stage_rows(q);
  }
  double acc[2][4];
  double pa[8];
  double resid0 = 0.0, resid1 = 0.0;
  for (long long q = 0; q < nitems; ++q) {
    const int c = (int)(q % nchunks);
    const long long rb = blockIdx.x + (q / nchunks) * gridDim.x;
    const long long o0 = rb * BM2 + wrow * ROWS;
    if (idle) continue;
    if (!rwarp && q + ST - 1 < nitems) {
      const long long qn = q + ST - 1;
      if (qn >= ST) mbar_wait(&empty[qn % ST], (unsigned)(((qn / ST) - 1) & 1));
      stage_rows(qn);
    }
    if (c == 0) {
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[n][v] = 0.0;
      if (rwarp) {
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const long long o = o0 + g + 8 * (v & 1);
          const int k = t + 4 * (v >> 1);
          pa[v] = (o < O && k < R) ? P[o * R + k] : 0.0;
        }
      }
    }
    const int slot = (int)(q % ST);
    mbar_wait(&full[slot], (unsigned)((q / ST) & 1));
    const double* xt = xs + (size_t)slot * BM2 * LD + wrow * ROWS * LD;
    const int i0 = c * BK;
    if (!rwarp) {
#pragma unroll
      for (int kb = 0; kb < BK; kb += 16) {
        double a[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) a[v] = xt[(g + 8 * (v & 1)) * LD + kb + t + 4 * (v >> 1)];
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          double b[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) b[v] = as[(size_t)(i0 + kb + t + 4 * v) * LDA + n * 8 + g];
          dmma_16x8x16(acc[n], a, b);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (c == nchunks - 1) {
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const long long o = o0 + g + 8 * (v >> 1);
            const int r = n * 8 + 2 * t + (v & 1);
            if (o < O && r < R) T[o * R + r] = acc[n][v];
          }
      }
    } else {
#pragma unroll
      for (int nb = 0; nb < BK; nb += 8) {
        double b[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) b[v] = as[(size_t)(i0 + nb + g) * LDA + t + 4 * v];
        double cx[4] = {0.0, 0.0, 0.0, 0.0};
        dmma_16x8x16(cx, pa, b);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 xv = *reinterpret_cast<const double2*>(xt + (g + 8 * h) * LD + nb + 2 * t);
          const double d0 = xv.x - cx[2 * h], d1 = xv.y - cx[2 * h + 1];
          resid0 = fma(d0, d0, resid0);  // zero-filled tails contribute exactly 0
          resid1 = fma(d1, d1, resid1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
  }
  if (FUSED) {
    const double s = block_sum<512>(resid0 + resid1, red);
    if (tid == 0) partial[blockIdx.x] = s;
  }
}

// The last-mode pass with the X tiles moved by tensor-map TMA. A stage is one 128-row x 32-
// column chunk of X as two 128 x 16 boxes (128 B rows, SWIZZLE_128B: the 16-byte chunk j of
// row r sits at chunk j ^ (r & 7)); out-of-range rows / columns arrive zero-filled. One thread
// issues both boxes of a stage (full barrier: 1 arrival + 32 KB); the 16 warps release a
// stage on its `empty` barrier. Conflict-free fragment reads of the swizzled tile come from
// two free relabellings, applied consistently to every operand:
//  * the k16 reduction order of the T GEMM: fragment slot kappa = t + 4 vh reads X column
//    pi(kappa) = (t & 1) + 2 vh + 8 (t >> 1) of the 16-column half, and the A_3 rows are
//    staged in the same order (smem row kappa holds A_3 row pi(kappa)), so the B fragments and
//    the residual GEMM's columns (A_3 rows) keep their plain addressing;
//  * the rows of a warp's 16-row tile: MMA row m reads X row rho(m) = (m & 8) | s(m & 7),
//    s = swap of bits 0 and 1, for the T output rows, the P rows and the residual alike.
__device__ __forceinline__ int l5_rho(int m) {
  return (m & 12) | ((m & 1) << 1) | ((m >> 1) & 1);
}
// RONLY (with FUSED): residual only, no T -- all 16 warps take residual column groups
template <bool FUSED, int ST, bool PW, bool RONLY = false>
__global__ void __launch_bounds__(PW ? 544 : 512, 1) k_ttm_last5(const __grid_constant__ CUtensorMap xmap,
                                                      long long O, int I,
                                                      const double* __restrict__ A, int R,
                                                      double* __restrict__ T,
                                                      const double* __restrict__ P,
                                                      double* __restrict__ partial,
                                                      const int* __restrict__ need) {
  RTB_GUARD()
  constexpr int BK = 32;
  constexpr int LDA = 20;
  constexpr int ROWS = 16;
  constexpr int kHalf = BM2 * 16;  // doubles per 128 x 16 box
  extern __shared__ __align__(1024) double sm5[];
  // the dynamic smem base is 16-byte aligned only: round up to the 1 KB swizzle atom
  double* xs = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sm5) + 1023) & ~uintptr_t(1023));
  double* as = xs + (size_t)ST * 2 * kHalf;  // [Ip][LDA], rows in pi order per 16-block
  __shared__ double red[32];
  __shared__ __align__(8) unsigned long long full[ST], empty[ST];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const bool rwarp = FUSED && (RONLY || warp >= 8);
  // residual column groups of this warp (8-column steps within the 32-column chunk)
  const int nb_lo = RONLY ? 16 * (warp >> 3) : 0, nb_hi = RONLY ? nb_lo + 16 : 32;
  const int wrow = warp & 7;
  const bool idle = !FUSED && warp >= 8;
  const long long nrb = ceil_div<long long>(O, BM2);
  const int nchunks = ceil_div(I, BK);
  const int Ip = nchunks * BK;
  for (int e = tid; e < Ip * LDA; e += 512) {
    const int i = e / LDA, r = e - i * LDA;
    const int kap = i & 15;
    const int src = (i & ~15) | ((kap & 1) + 2 * (kap >> 2) + 8 * ((kap >> 1) & 1));
    as[e] = (src < I && r < R) ? A[(size_t)src * R + r] : 0.0;
  }
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], FUSED ? 16 : 8);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const long long my_blocks = blockIdx.x < nrb ? (nrb - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long nitems = my_blocks * nchunks;
  // PW: a dedicated producer warp (warp 16) runs ahead of the ring; else thread 0 of warp 0
  const bool producer = PW ? tid == 512 : tid == 0;
  auto issue = [&](long long q) {
    const int slot = (int)(q % ST);
    const long long rb = blockIdx.x + (q / nchunks) * gridDim.x;
    const int c = (int)(q % nchunks);
    double* dst = xs + (size_t)slot * 2 * kHalf;
    mbar_arrive_expect_tx(&full[slot], 2u * kHalf * 8u);
    tma_load_2d(dst, &xmap, c * BK, (int)(rb * BM2), &full[slot]);
    tma_load_2d(dst + kHalf, &xmap, c * BK + 16, (int)(rb * BM2), &full[slot]);
  };
  if (PW && warp == 16) {
    if (producer) {
      for (long long q = 0; q < nitems; ++q) {
        if (q >= ST) mbar_wait(&empty[q % ST], (unsigned)(((q / ST) - 1) & 1));
        issue(q);
      }
    }
    return;
  }
  if (!PW && producer)
    for (long long q = 0; q < ST - 1 && q < nitems; ++q) issue(q);
  // this lane's tile rows (rho of MMA rows g and g + 8)
  const int ra = l5_rho(g), rb8 = l5_rho(g + 8);
  const int sw = ra & 7;  // = rb8 & 7
  double acc[2][4];
  double pa[8];
  double resid0 = 0.0, resid1 = 0.0;
  for (long long q = 0; q < nitems; ++q) {
    const int c = (int)(q % nchunks);
    const long long rbk = blockIdx.x + (q / nchunks) * gridDim.x;
    const long long o0 = rbk * BM2 + wrow * ROWS;
    if (idle) continue;
    if (!PW && producer && q + ST - 1 < nitems) {
      const long long qn = q + ST - 1;
      if (qn >= ST) mbar_wait(&empty[qn % ST], (unsigned)(((qn / ST) - 1) & 1));
      issue(qn);
    }
    __syncwarp();
    if (c == 0) {
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[n][v] = 0.0;
      if (rwarp) {
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const long long o = o0 + ((v & 1) ? rb8 : ra);
          const int k = t + 4 * (v >> 1);
          pa[v] = (o < O && k < R) ? P[o * R + k] : 0.0;
        }
      }
    }
    const int slot = (int)(q % ST);
    mbar_wait(&full[slot], (unsigned)((q / ST) & 1));
    const double* xt = xs + (size_t)slot * 2 * kHalf + (size_t)wrow * ROWS * 16;
    const int i0 = c * BK;
    if (!rwarp) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double* xh = xt + h * kHalf;
        double a[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const int row = (v & 1) ? rb8 : ra;
          const int chunk = ((v >> 1) + 4 * (t >> 1)) ^ sw;
          a[v] = xh[row * 16 + chunk * 2 + (t & 1)];
        }
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          double b[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) b[v] = as[(size_t)(i0 + 16 * h + t + 4 * v) * LDA + n * 8 + g];
          dmma_16x8x16(acc[n], a, b);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (c == nchunks - 1) {
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const long long o = o0 + ((v >> 1) ? rb8 : ra);
            const int r = n * 8 + 2 * t + (v & 1);
            if (o < O && r < R) T[o * R + r] = acc[n][v];
          }
      }
    } else {
#pragma unroll
      for (int nb = 0; nb < BK; nb += 8) {
        if (RONLY && (nb < nb_lo || nb >= nb_hi)) continue;
        double b[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) b[v] = as[(size_t)(i0 + nb + g) * LDA + t + 4 * v];
        double cx[4] = {0.0, 0.0, 0.0, 0.0};
        dmma_16x8x16(cx, pa, b);
        // output columns 2t, 2t + 1 of this 8-column group = smem A rows nb + 2t (+1) = X
        // columns pi(kappa), pi(kappa + 1) (adjacent): chunk (kappa >> 2) + 4 (t & 1)
        const double* xh = xt + (nb >> 4) * kHalf;
        const int chunk = ((((nb & 15) + 2 * t) >> 2) + 4 * (t & 1)) ^ sw;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int row = hh ? rb8 : ra;
          const double2 xv = *reinterpret_cast<const double2*>(xh + row * 16 + chunk * 2);
          const double d0 = xv.x - cx[2 * hh], d1 = xv.y - cx[2 * hh + 1];
          resid0 = fma(d0, d0, resid0);  // zero-filled tails contribute exactly 0
          resid1 = fma(d1, d1, resid1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
  }
  if (FUSED) {
    // (a producer warp has exited: a named barrier over the 16 compute warps)
    double v = resid0 + resid1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    asm volatile("bar.sync 1, 512;" ::: "memory");
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < 16; ++w) tot += red[w];
      partial[blockIdx.x] = tot;
    }
  }
}

static int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : kNumSMs;
  }();
  return n;
}

// the persistent kernel applies when A fits next to the X pipeline in shared memory
static bool last2_ok(int I, int R) {
  const int rp = R <= 8 ? 8 : R <= 16 ? 16 : R <= 24 ? 24 : 32;
  const size_t ip = (size_t)ceil_div(I, kBK) * kBK;
  const size_t smem = (ip * (rp + 4) + (size_t)kStages2 * BM2 * (kBK + kPadX)) * 8;
  return (I % 2) == 0 && smem <= 220 * 1024;
}

template <int RP, bool FUSED>
static void launch_last2(const double* X, long long O, int I, const double* A, int R, double* T,
                         const double* P, double* partial, cudaStream_t st, PGen pg) {
  const size_t ip = (size_t)ceil_div(I, kBK) * kBK;
  const size_t smem = (ip * lda2<RP>() + (size_t)kStages2 * BM2 * (kBK + kPadX)) * 8;
  auto k = k_ttm_last2<RP, FUSED>;
  set_max_smem(k, 220 * 1024);
  const long long nrb = ceil_div<long long>(O, BM2);
  const int grid = (int)std::min<long long>(nrb, sm_count());
  k<<<grid, 512, smem, st>>>(X, O, I, A, R, T, P, partial, g_need, pg);
  t_last_parts = grid;
  RTB_LAUNCH_CHECK();
}

bool ttm_last_resid(const double* X, long long O, int I, const double* A, int R, const double* P,
                    double* partial, cudaStream_t st) {
  static const bool no_l5 = std::getenv("RTB_NO_LAST5") != nullptr;
  constexpr int kL5St = 4;
  const size_t smem5 = (size_t)kL5St * 2 * BM2 * 16 * 8 + 1024 +
                       (size_t)ceil_div(I, 32) * 32 * 20 * 8;
  CUtensorMap xmap;
  if (no_l5 || R > 16 || smem5 > 227 * 1024 || !x_tensor_map(&xmap, X, O, I)) return false;
  auto k = k_ttm_last5<true, kL5St, true, true>;
  set_max_smem(k, (int)smem5);
  const long long nrb = ceil_div<long long>(O, BM2);
  const int grid = (int)std::min<long long>(nrb, sm_count());
  k<<<grid, 544, smem5, st>>>(xmap, O, I, A, R, nullptr, P, partial, g_need);
  t_last_parts = grid;
  RTB_LAUNCH_CHECK();
  count_variant("k_ttm_last5_resid");
  return true;
}

bool ttm_last_pgen_ok(int I, int R) { return R <= 32 && last2_ok(I, R); }

long long ttm_last_parts_bound(long long O, int I, int R) {
  (void)I;
  (void)R;
  return std::max(ceil_div<long long>(O, 64), std::min<long long>(ceil_div<long long>(O, BM2),
                                                                   sm_count()));
}

long long ttm_last_blocks(long long O, int I, int R) {
  if (t_last_parts >= 0) return t_last_parts;  // the launch just made by this thread
  if (last2_ok(I, R)) return std::min<long long>(ceil_div<long long>(O, BM2), sm_count());
  return ceil_div<long long>(O, 64);
}

void ttm_last(const double* X, long long O, int I, const double* A, int R, double* T,
              const double* P, double* partial, cudaStream_t st, const double* W,
              const double* A2, int I2, int R2) {
  const bool fused = P != nullptr || W != nullptr;
  const PGen pg{W, A2, I2, R2};
  if (W) throw Error(4, "ttm_last: in-pass P generation is disabled (slower than materialised P)");
  const bool v2 = (I % 2) == 0;
  const int rp = R <= 8 ? 8 : R <= 16 ? 16 : R <= 24 ? 24 : 32;
  if (R > 32) throw Error(4, "ttm_last: rank > 32 not supported by the DMMA path");
  const size_t ip3 = (size_t)ceil_div(I, kL3BK) * kL3BK;
  const size_t smem3 = (ip3 * lda2<16>() + (size_t)kL3Stages * BM2 * (kL3BK + kPadX)) * 8;
  static const bool no_l5 = std::getenv("RTB_NO_LAST5") != nullptr;
  constexpr int kL5St = 4;
  const size_t smem5 = (size_t)kL5St * 2 * BM2 * 16 * 8 + 1024 +
                       (size_t)ceil_div(I, 32) * 32 * 20 * 8;
  CUtensorMap xmap;
  if (!no_l5 && R <= 16 && smem5 <= 227 * 1024 && x_tensor_map(&xmap, X, O, I)) {
    static const bool pw = std::getenv("RTB_L5_NO_PW") == nullptr;
    auto k = fused ? (pw ? k_ttm_last5<true, kL5St, true> : k_ttm_last5<true, kL5St, false>)
                   : (pw ? k_ttm_last5<false, kL5St, true> : k_ttm_last5<false, kL5St, false>);
    set_max_smem(k, (int)smem5);
    const long long nrb = ceil_div<long long>(O, BM2);
    const int grid = (int)std::min<long long>(nrb, sm_count());
    k<<<grid, pw ? 544 : 512, smem5, st>>>(xmap, O, I, A, R, T, P, partial, g_need);
    t_last_parts = grid;
    RTB_LAUNCH_CHECK();
    count_variant(fused ? "k_ttm_last3_fused" : "k_ttm_last3");
    count_variant(fused ? "k_ttm_last5_fused" : "k_ttm_last5");
    return;
  }
  static const bool no_l4 = std::getenv("RTB_NO_LAST4") != nullptr;
  const size_t smem4 = (ip3 * lda2<16>() + (size_t)kL4Stages * BM2 * (kL4BK + kPadX)) * 8;
  if (!no_l4 && R <= 16 && (I % 2) == 0 && I % kL4BK == 0 && smem4 <= 227 * 1024 - 1024) {
    auto k = fused ? k_ttm_last4<true, kL4BK, kL4Stages> : k_ttm_last4<false, kL4BK, kL4Stages>;
    set_max_smem(k, (int)smem4);
    const long long nrb = ceil_div<long long>(O, BM2);
    const int grid = (int)std::min<long long>(nrb, sm_count());
    k<<<grid, 512, smem4, st>>>(X, O, I, A, R, T, P, partial, g_need);
    t_last_parts = grid;
    RTB_LAUNCH_CHECK();
    count_variant(fused ? "k_ttm_last3_fused" : "k_ttm_last3");
    count_variant(fused ? "k_ttm_last4_fused" : "k_ttm_last4");
    return;
  }
  if (R <= 16 && (I % 2) == 0 && smem3 <= 227 * 1024 - 1024) {
    const size_t smem = smem3;
    auto k = fused ? k_ttm_last3<true, kL3BK, kL3Stages> : k_ttm_last3<false, kL3BK, kL3Stages>;
    set_max_smem(k, 227 * 1024 - 1024);
    const long long nrb = ceil_div<long long>(O, BM2);
    const int grid = (int)std::min<long long>(nrb, sm_count());
    k<<<grid, 512, smem, st>>>(X, O, I, A, R, T, P, partial, g_need);
    t_last_parts = grid;
    RTB_LAUNCH_CHECK();
    count_variant(fused ? "k_ttm_last3_fused" : "k_ttm_last3");
    return;
  }
  if (last2_ok(I, R)) {
#define RTB_L2(RPV)                                                     \
  case RPV:                                                             \
    if (fused) launch_last2<RPV, true>(X, O, I, A, R, T, P, partial, st, pg); \
    else launch_last2<RPV, false>(X, O, I, A, R, T, P, partial, st, pg);      \
    break;
    switch (rp) {
      RTB_L2(8)
      RTB_L2(16)
      RTB_L2(24)
      RTB_L2(32)
    }
#undef RTB_L2
    return;
  }
#define RTB_L(RPV)                                                                       \
  case RPV:                                                                              \
    if (fused) {                                                                         \
      if (v2) launch_last<RPV, 2, true>(X, O, I, A, R, T, P, partial, st);               \
      else launch_last<RPV, 1, true>(X, O, I, A, R, T, P, partial, st);                  \
    } else {                                                                             \
      if (v2) launch_last<RPV, 2, false>(X, O, I, A, R, T, P, partial, st);              \
      else launch_last<RPV, 1, false>(X, O, I, A, R, T, P, partial, st);                 \
    }                                                                                    \
    break;
  switch (rp) {
    RTB_L(8)
    RTB_L(16)
    RTB_L(24)
    RTB_L(32)
  }
#undef RTB_L
}

// per-thread, per-device scratch for split-K partial sums (grown on demand,
// stream-ordered; thread-local so concurrent host threads on their own streams never
// share it)
static double* splits_scratch(size_t bytes, cudaStream_t st) {
  thread_local double* buf[16] = {};
  thread_local size_t cap[16] = {};
  int dev = 0;
  RTB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) throw Error(4, "ttm_mid: device index");
  if (cap[dev] < bytes) {
    if (buf[dev]) RTB_CUDA(cudaFreeAsync(buf[dev], st));
    RTB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf[dev]), bytes, st));
    cap[dev] = bytes;
  }
  return buf[dev];
}

template <int RP, int VEC>
static void launch_mid(const double* X, long long O, int I, long long J, const double* A, int R,
                       double* out, cudaStream_t st) {
  constexpr int smem = kStages * kBK * (64 + kPadX) * sizeof(double);
  auto k = k_ttm_mid<RP, VEC>;
  set_max_smem(k, (int)smem);
  const long long tiles = ceil_div<long long>(O * J, 64);
  // split the reduction when the column tiles alone cannot fill the GPU
  int splits = 1;
  while (tiles * splits < 6LL * kNumSMs && I / (splits * 2) >= 2 * kBK) splits *= 2;
  const int ich = ceil_div(ceil_div(I, splits), kBK) * kBK;
  splits = ceil_div(I, ich);
  const long long n = O * R * J;
  double* dst = splits > 1 ? splits_scratch((size_t)splits * n * 8, st) : out;
  dim3 grid((unsigned)tiles, (unsigned)splits);
  k<<<grid, 128, smem, st>>>(X, O, I, J, A, R, dst, ich);
  RTB_LAUNCH_CHECK();
  if (splits > 1) {
    k_sum_splits<<<(unsigned)ceil_div<long long>(n, 256), 256, 0, st>>>(dst, n, splits, out);
    RTB_LAUNCH_CHECK();
  }
}

template <int RP>
static void launch_mid2(const double* X, long long O, int I, long long J, const double* A, int R,
                        double* out, cudaStream_t st) {
  const size_t smem = mid2_smem(I, RP);
  static const bool probe = std::getenv("RTB_TTM_STREAM_ONLY") != nullptr;
  static const bool pc = std::getenv("RTB_TTM_NO_PRODUCER") == nullptr;
  const size_t smem3 = mid3_smem(I, RP);
  static const bool no_m5 = std::getenv("RTB_NO_MID5") != nullptr;
  const size_t smem5 = mid5_smem(I, RP);
  CUtensorMap xmap;
  if (!no_m5 && !probe && smem5 <= 227 * 1024 - 2048 && mid_tensor_map(&xmap, X, O, I, J)) {
    set_max_smem(k_ttm_mid5<RP>, (int)smem5);
    const long long ntiles = O * J / BJ2;
    const int grid = (int)std::min<long long>(ntiles, sm_count());
    k_ttm_mid5<RP><<<grid, 288, smem5, st>>>(xmap, O, I, J, A, R, out);
    RTB_LAUNCH_CHECK();
    count_variant("k_ttm_mid3");
    count_variant("k_ttm_mid5");
    return;
  }
  if constexpr (RP > 16) {
    // rank 32: 16-row boxes, five stages
    const size_t smem6 = mid5_smem(I, RP, 16, 5);
    if (!no_m5 && !probe && smem6 <= 227 * 1024 - 2048 && mid_tensor_map(&xmap, X, O, I, J, 16)) {
      set_max_smem(k_ttm_mid5<RP, 16, 5>, (int)smem6);
      const long long ntiles = O * J / BJ2;
      const int grid = (int)std::min<long long>(ntiles, sm_count());
      k_ttm_mid5<RP, 16, 5><<<grid, 288, smem6, st>>>(xmap, O, I, J, A, R, out);
      RTB_LAUNCH_CHECK();
      count_variant("k_ttm_mid5<32>");
      return;
    }
  }
  if (pc && smem3 <= 227 * 1024 - 2048) {
    auto k3 = probe ? k_ttm_mid3<RP, false> : k_ttm_mid3<RP, true>;
    set_max_smem(k3, 227 * 1024 - 2048);
    const long long ntiles = O * J / BJ2;
    const int grid = (int)std::min<long long>(ntiles, sm_count());
    k3<<<grid, 288, smem3, st>>>(X, O, I, J, A, R, out);
    RTB_LAUNCH_CHECK();
    count_variant("k_ttm_mid3");
    return;
  }
  auto k = probe ? k_ttm_mid2<RP, false> : k_ttm_mid2<RP, true>;
  set_max_smem(k, 220 * 1024);
  const long long ntiles = O * J / BJ2;
  const int grid = (int)std::min<long long>(ntiles, sm_count());
  k<<<grid, 256, smem, st>>>(X, O, I, J, A, R, out);
  RTB_LAUNCH_CHECK();
  count_variant("k_ttm_mid2");
}

void ttm_mid(const double* X, long long O, int I, long long J, const double* A, int R, double* out,
             cudaStream_t st) {
  const bool v2 = (J % 2) == 0;
  const int rp = R <= 8 ? 8 : R <= 16 ? 16 : R <= 24 ? 24 : 32;
  if (R > 32) throw Error(4, "ttm_mid: rank > 32 not supported by the DMMA path");
  {
    // persistent path: whole 128-column tiles, enough of them to keep every SM busy,
    // and A resident next to the pipeline
    const size_t smem = mid2_smem(I, rp);
    const bool tiles_ok = J % BJ2 == 0 && O * J / BJ2 >= 4LL * sm_count();
    // rank 32 with I beyond k_ttm_mid2's shared memory (C5: I = 512): the 16-row-box mid5 only
    static const bool no_m5 = std::getenv("RTB_NO_MID5") != nullptr;
    CUtensorMap probe_map;
    if (tiles_ok && smem > 220 * 1024 && rp == 32 && !no_m5 &&
        mid5_smem(I, 32, 16, 5) <= 227 * 1024 - 2048 && mid_tensor_map(&probe_map, X, O, I, J, 16)) {
      launch_mid2<32>(X, O, I, J, A, R, out, st);
      return;
    }
    if (tiles_ok && smem <= 220 * 1024) {
      switch (rp) {
        case 8: launch_mid2<8>(X, O, I, J, A, R, out, st); return;
        case 16: launch_mid2<16>(X, O, I, J, A, R, out, st); return;
        case 24: launch_mid2<24>(X, O, I, J, A, R, out, st); return;
        default: launch_mid2<32>(X, O, I, J, A, R, out, st); return;
      }
    }
  }
#define RTB_M(RPV)                                        \
  case RPV:                                               \
    if (v2) launch_mid<RPV, 2>(X, O, I, J, A, R, out, st); \
    else launch_mid<RPV, 1>(X, O, I, J, A, R, out, st);    \
    break;
  switch (rp) {
    RTB_M(8)
    RTB_M(16)
    RTB_M(24)
    RTB_M(32)
  }
#undef RTB_M
}

void ttm_generic(const double* X, long long O, int I, long long J, const double* W, long long wr,
                 long long wi, int R, double* out, cudaStream_t st) {
  const long long total = O * R * J;
  if (total == 0) return;
  k_ttm_generic<<<(unsigned)ceil_div<long long>(total, 256), 256, 0, st>>>(X, O, I, J, W, wr, wi,
                                                                          R, out, g_need);
  RTB_LAUNCH_CHECK();
}

bool ttm_smallj(const double* X, long long O, int I, int J, const double* A, int R, double* out,
                cudaStream_t st) {
  if (R * J > 1024 || J > 32 || R > 32) return false;
  k_ttm_smallj<<<(unsigned)O, 256, 0, st>>>(X, I, J, A, R, out);
  RTB_LAUNCH_CHECK();
  return true;
}

// F_1 / F_2 of an order-3 exact factor update from T = X x_3 A_3^T (I_1 x I_2 x R_3, L2-resident)
// in ONE launch: per unit u of mode n (a warp), Y_u = A_m^T S_u (R_m x R_3, S_u the I_m x R_3
// slice of T at u; m the other non-last mode) on the DMMA pipe (m16n8k16, K = I_m), then
// M[u, :] = G_(n) vec(Y_u) from shared memory. Replaces the mode product, its split-K sum and
// the core contraction (3 launches, ~30 us at C2). R_m, R_3, R_n <= 16.
__global__ void __launch_bounds__(256) k_fu_proj3(const double* __restrict__ T, int I1, int I2,
                                                  int R3, const double* __restrict__ Am, int Rm,
                                                  const double* __restrict__ G, int R1, int R2,
                                                  int n, double* __restrict__ M) {
  // a CTA per unit u (persistent over units); its 8 warps split the K = I_m contraction
  // (all of a warp's loads issued before its DMMAs), partial Y summed in shared memory
  extern __shared__ double fps[];
  double* Gs = fps;               // [16 rn][16 rm][16 r3]
  double* Yp = Gs + 4096;         // [8 warps][256]
  double* Y = Yp + 8 * 256;       // [256]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int Rn = n == 0 ? R1 : R2;
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) {
    const int rn = e >> 8, rm = (e >> 4) & 15, r3 = e & 15;
    double v = 0.0;
    if (rn < Rn && rm < Rm && r3 < R3) {
      const int r1 = n == 0 ? rn : rm, r2 = n == 0 ? rm : rn;
      v = G[((size_t)r1 * R2 + r2) * R3 + r3];
    }
    Gs[e] = v;
  }
  const int In = n == 0 ? I1 : I2, Im = n == 0 ? I2 : I1;
  const long long su = n == 0 ? (long long)I2 * R3 : (long long)R3;  // stride of u
  const long long sk = n == 0 ? (long long)R3 : (long long)I2 * R3;  // stride of k
  const int kper = ((Im + 7) / 8 + 15) / 16 * 16;                      // k range per warp
  for (int u = blockIdx.x; u < In; u += gridDim.x) {
    const double* S = T + (long long)u * su;
    double c[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
    const int kw0 = warp * kper, kw1 = min(Im, kw0 + kper);
    for (int kb = kw0; kb < kw1; kb += 64) {
      double a[4][8], b[4][2][4];
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const int k0 = kb + 16 * s4;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const int k = k0 + t + 4 * (v >> 1), r = g + 8 * (v & 1);
          a[s4][v] = (k < kw1 && r < Rm) ? __ldg(Am + (size_t)k * Rm + r) : 0.0;
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int k = k0 + t + 4 * v, r3 = nt * 8 + g;
            b[s4][nt][v] = (k < kw1 && r3 < R3) ? __ldcg(S + (long long)k * sk + r3) : 0.0;
          }
      }
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma_16x8x16(c[nt], a[s4], b[s4][nt]);
    }
    double* yw = Yp + warp * 256;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int v = 0; v < 4; ++v) yw[(g + 8 * (v >> 1)) * 16 + nt * 8 + 2 * t + (v & 1)] = c[nt][v];
    __syncthreads();
    {
      const int e = threadIdx.x;  // 256 = 16 rm x 16 r3
      double y = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) y += Yp[w * 256 + e];
      Y[e] = y;
    }
    __syncthreads();
    // M[u, rn] = sum_{rm, r3} G_(n)[rn][rm][r3] Y[rm][r3]: warp w takes rn = w, w + 8
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int rn = warp + 8 * q;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = fma(Gs[rn * 256 + lane + 32 * j], Y[lane + 32 * j], acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0 && rn < Rn) M[(size_t)u * Rn + rn] = acc;
    }
    __syncthreads();  // Yp / Y reused by the next unit
  }
}

bool fu_proj3(const double* T, int I1, int I2, int R3, const double* Am, int Rm, const double* G,
              int R1, int R2, int n, double* M, cudaStream_t st) {
  static const bool off = std::getenv("RTB_NO_FU_PROJ3") != nullptr;  // experiments
  if (off || n > 1 || R1 > 16 || R2 > 16 || R3 > 16) return false;
  const int In = n == 0 ? I1 : I2;
  const int grid = std::max(1, std::min(In, 2 * sm_count()));
  const size_t smem = (size_t)(4096 + 8 * 256 + 256) * 8;
  set_max_smem(k_fu_proj3, (int)smem);
  k_fu_proj3<<<grid, 256, smem, st>>>(T, I1, I2, R3, Am, Rm, G, R1, R2, n, M);
  RTB_LAUNCH_CHECK();
  return true;
}

bool ttm_expand(const double* Y, long long O, int R, long long J, const double* A, int I,
                double* out, cudaStream_t st) {
  // big i chunks (A rows staged once per CTA, several outputs per thread), shrunk
  // until there are enough blocks to fill the GPU
  // (each CTA stages all of Y[o] (R x J): when that is large, about one wave of CTAs
  // amortises it better than many small ones -- W = G x_1 A_1 at C2: 512 CTAs each staging
  // 32 KB took 23 us)
  int ich = 128;
  const long long minb = (long long)R * J >= 2048 ? kNumSMs / 2 : 4LL * kNumSMs;
  while (ich > 1 && O * ceil_div(I, ich) < minb) ich >>= 1;
  static const bool no_dx = std::getenv("RTB_NO_EXPAND_DMMA") != nullptr;  // experiments
  if (!no_dx && R <= 16 && J <= 16 && I >= 128) {
    const long long ib = ceil_div(I, 128);
    int och = (int)std::max<long long>(1, (O * ib) / (2LL * kNumSMs));
    if (ceil_div<long long>(O, och) > 65535) och = (int)ceil_div<long long>(O, 65535);
    const dim3 grid((unsigned)ib, (unsigned)ceil_div<long long>(O, och));
    k_ttm_expand_dmma<<<grid, 256, 0, st>>>(Y, R, (int)J, A, I, O, och, out, g_need);
    RTB_LAUNCH_CHECK();
    return true;
  }
  if (R <= 16 && J <= 16 && (J % 2) == 0 && I >= 256) {
    // row-owner kernel: about two CTAs per SM over (i blocks) x (o ranges)
    const long long ib = ceil_div(I, 256);
    int och = (int)std::max<long long>(1, (O * ib) / (2LL * kNumSMs));
    if (ceil_div<long long>(O, och) > 65535) och = (int)ceil_div<long long>(O, 65535);
    const dim3 grid((unsigned)ib, (unsigned)ceil_div<long long>(O, och));
    if (J <= 8)
      k_ttm_expand_rows<16, 8><<<grid, 256, 0, st>>>(Y, R, (int)J, A, I, O, och, out, g_need);
    else
      k_ttm_expand_rows<16, 16><<<grid, 256, 0, st>>>(Y, R, (int)J, A, I, O, och, out, g_need);
    RTB_LAUNCH_CHECK();
    return true;
  }
  const size_t smem = ((size_t)R * J + (size_t)ich * R) * sizeof(double);
  if (smem > 48 * 1024 || O > 65535) return false;
  k_ttm_expand<<<dim3((unsigned)ceil_div(I, ich), (unsigned)O), 256, smem, st>>>(Y, R, J, A, I,
                                                                                 ich, out, g_need);
  RTB_LAUNCH_CHECK();
  return true;
}

void contract_except(const double* Y, const double* G, long long O, int I, int R, long long J,
                     double* M, cudaStream_t st) {
  if (R <= 8) {
    k_contract_except<8><<<I, 128, 0, st>>>(Y, G, O, I, R, J, M);
  } else if (R <= 16) {
    k_contract_except<16><<<I, 128, 0, st>>>(Y, G, O, I, R, J, M);
  } else if (R <= 32) {
    k_contract_except<32><<<I, 128, 0, st>>>(Y, G, O, I, R, J, M);
  } else {
    const long long total = (long long)I * R;
    k_contract_except_scalar<<<(unsigned)ceil_div<long long>(total, 128), 128, 0, st>>>(
        Y, G, O, I, R, J, M);
  }
  RTB_LAUNCH_CHECK();
}

void sum_partials(const double* partial, long long n, double* out, cudaStream_t st) {
  k_sum_partials<<<1, 1024, 0, st>>>(partial, n, out, g_need);
  RTB_LAUNCH_CHECK();
}

}  // namespace rtb
