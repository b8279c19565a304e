// k_fsketch.cu -- the sketched factor update's normal equations (perf mode).
//
// Not in the reference (BASELINE's "samples per factor update").
// The mode-n subproblem  min ||K a_i - x_i||^2 + lambda ||a_i||^2  over the rows i of
// A_n, with K = (kron_{m!=n} A_m) G_(n)^T (ref tucker.cpp:31-43,70-89), is sketched ONCE
// for all rows: s draws from the product of the other modes' leverage distributions
// with the sqrt(lambda) augmentation over R_n (the core's draw machinery, k_draw.cu,
// with d = R_n), then
//   data draw t (other-mode indices j):  k_t = G_(n) z_t, z_t = kron_m A_m[j_m, :]
//                                        fiber x_t = X(j_1, .., :, .., j_N)   (I_n values)
//   Gram = sum_t w_t^2 k_t k_t^T + sum_aug w^2 lambda e_j e_j^T                (R_n x R_n)
//   M    = sum_t w_t^2 x_t k_t^T                                               (I_n x R_n)
// and A_n = M pinv(Gram) (the caller). The oracle restatement is
// orc_update_factor_sketched (oracle/rtucker_oracle.c).
//
// Kernels:
//   k_fsk_unfold G_(n)^T as W x R rows (W = prod_{m!=n} R_m) + packed digits of each q
//   k_fsk_rows   8 draws per warp: Kw = Z Gt as m8n8k4 DMMAs, Z generated from the draws'
//                factor rows in shared memory (each Gt element serves 8 draws);
//                stores w_t k_t and the fiber's base offset (-1 - j for augmented row j)
//   k_fsk_accum  (draw chunk, 256-column tile) CTAs: the fiber GATHER (the HBM part:
//                8 I_n useful bytes per data draw; one 32 B sector per value when the
//                mode is not the last, since fibers of random draws share no sectors)
//                and register accumulation of M; tile-0 CTAs also sum the chunk's Gram
//   k_fsk_reduce fixed-order sums over chunks (deterministic)
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace rtb {

namespace {

constexpr int kSub = 64;       // draws staged per shared-memory round
constexpr int kTile = 256;     // fiber columns per CTA (one per thread)

struct FskDev {
  int order, mode, rn, nother;
  int orow[8], orank[8];            // other modes, ascending
  long long oxstride[8];            // X stride of each other mode
  int ocstride[8];                  // core stride of each other mode
  const double* ofac[8];
  int cstride_n;                    // core stride of mode n
  long long xstride_n;              // X stride of mode n
  int width;                        // prod_{m!=n} R_m
  int in;                           // I_n
  unsigned long long total_other;
  double root_lambda;
  int o0_lo, o0_hi;                 // sharded, n > 0: mode-1 rows owned (o0_hi = 0: all)
  int skip_aug;                     // sharded, n > 0: augmented rows counted elsewhere
};

// Gt[q][r] = G_(n)[r][q] (W x RM, zero-padded) and the digit offsets of q over the
// other modes' ranks packed 5 bits per mode (R_m <= 32): one coalesced row per q.
template <int RM>
__global__ void k_fsk_unfold(FskDev f, const double* __restrict__ core, double* __restrict__ gt,
                             unsigned long long* __restrict__ qdig) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= f.width) return;
  int rem = q, coff = 0;
  unsigned long long packed = 0;
  for (int m = f.nother - 1; m >= 0; --m) {
    const int dgt = rem % f.orank[m];
    rem /= f.orank[m];
    coff += dgt * f.ocstride[m];
    packed |= (unsigned long long)dgt << (5 * m);
  }
  qdig[q] = packed;
  for (int r = 0; r < RM; ++r) gt[(size_t)q * RM + r] = r < f.rn ? core[coff + r * f.cstride_n] : 0.0;
}

// k_t for 8 draws per warp on the FP64 tensor cores: Kw (8 draws x R) = Z (8 x W) Gt (W x R)
// as m8n8k4 DMMAs over q (4 per step), Z generated on the fly: lane (g, t) = (lane / 4,
// lane % 4) forms z_g(q0 + t) = prod_m A_m[j_m(draw g), digit_m(q0 + t)] from the draw's
// factor rows staged in shared memory (product in ascending mode order, as kron_row),
// and reads Gt[q0 + t][8 nt + g] (L1-resident) as the B fragment. Each Gt element now
// serves 8 draws. Augmented draws get z = 0 (k = 0) and base = -1 - j.
template <int RM>
__global__ void __launch_bounds__(256) k_fsk_rows(FskDev f, const double* __restrict__ gt,
                                                  const unsigned long long* __restrict__ qdig,
                                                  const unsigned long long* __restrict__ idx,
                                                  const double* __restrict__ wts,
                                                  unsigned long long s, int srow,
                                                  double* __restrict__ kw,
                                                  long long* __restrict__ base) {
  extern __shared__ double rows_s[];  // [warp][8 draws][srow]: other modes' rows, concatenated
  int* isdata = reinterpret_cast<int*>(rows_s + (size_t)(blockDim.x >> 5) * 8 * srow);
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 8;
  if (t0 >= (long long)s) return;
  double* rs = rows_s + (size_t)wib * 8 * srow;
  int* dflag = isdata + wib * 8;
  int* sj = isdata + (blockDim.x >> 5) * 8 + wib * 64;  // [draw][mode] other-mode indices
  const int g = lane >> 2, tq = lane & 3;
  double wg = 0.0;
  // lanes 0..7: delinearize draw t0 + lane (last fastest, ref kronecker.cpp:44-52)
  if (lane < 8) {
    const long long t = t0 + lane;
    long long b = 0;
    int data = 0;
    if (t < (long long)s) {
      const unsigned long long id = idx[t];
      if (id < f.total_other) {
        data = 1;
        unsigned long long rem = id;
#pragma unroll
        for (int m = 7; m >= 0; --m)
          if (m < f.nother) {
            const int jm = (int)(rem % (unsigned long long)f.orow[m]);
            rem /= (unsigned long long)f.orow[m];
            // other mode 0 is mode 1 when n > 0: under sharding only its own rows are in x
            const int jx = (m == 0 && f.o0_hi > 0) ? jm - f.o0_lo : jm;
            if (m == 0 && f.o0_hi > 0 && (jm < f.o0_lo || jm >= f.o0_hi)) data = 0;
            b += (long long)jx * f.oxstride[m];
            sj[lane * 8 + m] = jm;
          }
        if (!data) b = 0;  // another shard's draw: k = 0 at a valid fiber, contributes nothing
      } else {
        b = f.skip_aug ? 0 : -1 - (long long)(id - f.total_other);
      }
      base[t] = b;
    }
    dflag[lane] = data;
  }
  __syncwarp();
  // stage the factor rows: draw d's mode-m row at rs[d * srow + off_m] (independent loads)
  {
    int off = 0;
#pragma unroll
    for (int m = 0; m < 8; ++m)
      if (m < f.nother) {
        const int R = f.orank[m];
        for (int e = lane; e < 8 * R; e += 32) {
          const int d = e / R, c = e - d * R;
          if (dflag[d]) rs[d * srow + off + c] = __ldg(f.ofac[m] + (size_t)sj[d * 8 + m] * R + c);
        }
        off += R;
      }
  }
  __syncwarp();
  const bool gdata = dflag[g] != 0;
  const double* rg = rs + g * srow;
  double c[RM / 8][2];
#pragma unroll
  for (int nt = 0; nt < RM / 8; ++nt) c[nt][0] = c[nt][1] = 0.0;
  // unrolled so that the digit and Gt loads of four k-steps are in flight together (the loop
  // was bound by one L1/L2 round trip per step); the DMMA order is unchanged
#pragma unroll 4
  for (int q0 = 0; q0 < f.width; q0 += 4) {
    const int q = q0 + tq;
    const bool qv = q < f.width;
    double z = 0.0;
    if (qv && gdata) {
      const unsigned long long dg = __ldg(qdig + q);
      z = 1.0;
      int off = 0;
#pragma unroll
      for (int m = 0; m < 8; ++m)
        if (m < f.nother) {
          z *= rg[off + (int)((dg >> (5 * m)) & 31)];
          off += f.orank[m];
        }
    }
#pragma unroll
    for (int nt = 0; nt < RM / 8; ++nt) {
      const double bv = qv ? __ldg(gt + (size_t)q * RM + nt * 8 + g) : 0.0;
      dmma_8x8x4(c[nt][0], c[nt][1], z, bv);
    }
  }
  // C[g][2 tq + e] of n-tile nt: draw t0 + g, r = 8 nt + 2 tq + e
  const long long t = t0 + g;
  if (t < (long long)s) {
    wg = wts[t];
#pragma unroll
    for (int nt = 0; nt < RM / 8; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = nt * 8 + 2 * tq + e;
        kw[t * RM + r] = r < f.rn ? wg * c[nt][e] : 0.0;
      }
  }
}

template <int RM>
__global__ void __launch_bounds__(kTile) k_fsk_accum(FskDev f, const double* __restrict__ x,
                                                     const double* __restrict__ kw,
                                                     const long long* __restrict__ base,
                                                     const double* __restrict__ wts,
                                                     unsigned long long s, long long chunk,
                                                     double* __restrict__ part,
                                                     double* __restrict__ gpart) {
  __shared__ __align__(16) double skw[kSub][RM];
  __shared__ long long sb[kSub];
  __shared__ double sw[kSub];
  const long long t0 = (long long)blockIdx.x * chunk;
  const long long t1 = min((long long)s, t0 + chunk);
  const int i = blockIdx.y * kTile + threadIdx.x;
  const bool col = i < f.in;
  const double* xcol = x + (col ? (long long)i * f.xstride_n : 0);
  const bool do_gram = blockIdx.y == 0;
  const int rn = f.rn;
  double acc[RM];
#pragma unroll
  for (int r = 0; r < RM; ++r) acc[r] = 0.0;
  // Gram pairs of this thread (tile-0 CTAs): (p, q) = e / rn, e % rn for e = tid, tid + 256..
  double gacc[(RM * RM + kTile - 1) / kTile];
#pragma unroll
  for (int k = 0; k < (RM * RM + kTile - 1) / kTile; ++k) gacc[k] = 0.0;
  for (long long ts = t0; ts < t1; ts += kSub) {
    const int n = (int)min((long long)kSub, t1 - ts);
    __syncthreads();
    for (int e = threadIdx.x; e < n * RM; e += kTile) skw[e / RM][e % RM] = kw[(ts + e / RM) * RM + e % RM];
    for (int e = threadIdx.x; e < n; e += kTile) {
      sb[e] = base[ts + e];
      sw[e] = wts[ts + e];
    }
    __syncthreads();
    if (col) {
#pragma unroll 8
      for (int tt = 0; tt < n; ++tt) {
        const long long bb = sb[tt];
        const double v = bb >= 0 ? sw[tt] * __ldg(xcol + bb) : 0.0;
#pragma unroll
        for (int r = 0; r < RM; ++r) acc[r] = fma(skw[tt][r], v, acc[r]);
      }
    }
    if (do_gram) {
#pragma unroll
      for (int k = 0; k < (RM * RM + kTile - 1) / kTile; ++k) {
        const int e = threadIdx.x + k * kTile;
        if (e < rn * rn) {
          const int p = e / rn, q = e - p * rn;
          double g = gacc[k];
          for (int tt = 0; tt < n; ++tt) {
            const long long bb = sb[tt];
            if (bb >= 0) {
              g = fma(skw[tt][p], skw[tt][q], g);
            } else if (p == q && (int)(-1 - bb) == p) {
              const double w2 = sw[tt] * sw[tt];
              g = fma(w2 * f.root_lambda, f.root_lambda, g);
            }
          }
          gacc[k] = g;
        }
      }
    }
  }
  if (col) {
    double* o = part + ((size_t)blockIdx.x * f.in + i) * RM;
#pragma unroll
    for (int r = 0; r < RM; ++r) o[r] = acc[r];
  }
  if (do_gram) {
#pragma unroll
    for (int k = 0; k < (RM * RM + kTile - 1) / kTile; ++k) {
      const int e = threadIdx.x + k * kTile;
      if (e < rn * rn) gpart[(size_t)blockIdx.x * rn * rn + e] = gacc[k];
    }
  }
}

// Contiguous fibers (x is the mode-n-last copy, or n is the last mode) and even I_n: each of
// 128 threads owns TWO adjacent columns of the 256-column tile (16-byte loads of the gathered
// fiber values, 16 draws unrolled so ~32 KB per SM are in flight), otherwise as
// k_fsk_accum (same chunking by the caller, same Gram partials from the tile-0 CTAs).
constexpr int kT2 = 128;
template <int RM>
__global__ void __launch_bounds__(kT2) k_fsk_accum2(FskDev f, const double* __restrict__ x,
                                                   const double* __restrict__ kw,
                                                   const long long* __restrict__ base,
                                                   const double* __restrict__ wts,
                                                   unsigned long long s, long long chunk,
                                                   double* __restrict__ part,
                                                   double* __restrict__ gpart) {
  __shared__ __align__(16) double skw[kSub][RM];
  __shared__ long long sb[kSub];
  __shared__ double sw[kSub];
  const long long t0 = (long long)blockIdx.x * chunk;
  const long long t1 = min((long long)s, t0 + chunk);
  const int i = blockIdx.y * kTile + 2 * threadIdx.x;
  const bool col = i < f.in;
  const double2* xcol = reinterpret_cast<const double2*>(x + (col ? i : 0));
  const bool do_gram = blockIdx.y == 0;
  const int rn = f.rn;
  double acc0[RM], acc1[RM];
#pragma unroll
  for (int r = 0; r < RM; ++r) acc0[r] = acc1[r] = 0.0;
  constexpr int NG = (RM * RM + kT2 - 1) / kT2;
  double gacc[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) gacc[k] = 0.0;
  for (long long ts = t0; ts < t1; ts += kSub) {
    const int n = (int)min((long long)kSub, t1 - ts);
    __syncthreads();
    for (int e = threadIdx.x; e < n * RM; e += kT2) skw[e / RM][e % RM] = kw[(ts + e / RM) * RM + e % RM];
    for (int e = threadIdx.x; e < n; e += kT2) {
      sb[e] = base[ts + e];
      sw[e] = wts[ts + e];
    }
    __syncthreads();
    if (col) {
#pragma unroll 16
      for (int tt = 0; tt < n; ++tt) {
        const long long bb = sb[tt];
        double2 v = make_double2(0.0, 0.0);
        if (bb >= 0) {
          const double2 xv = __ldg(xcol + (bb >> 1));  // bb is a multiple of I_n (even)
          v.x = sw[tt] * xv.x;
          v.y = sw[tt] * xv.y;
        }
#pragma unroll
        for (int r = 0; r < RM; r += 2) {
          const double2 k2 = *reinterpret_cast<const double2*>(&skw[tt][r]);
          acc0[r] = fma(k2.x, v.x, acc0[r]);
          acc0[r + 1] = fma(k2.y, v.x, acc0[r + 1]);
          acc1[r] = fma(k2.x, v.y, acc1[r]);
          acc1[r + 1] = fma(k2.y, v.y, acc1[r + 1]);
        }
      }
    }
    if (do_gram) {
#pragma unroll
      for (int k = 0; k < NG; ++k) {
        const int e = threadIdx.x + k * kT2;
        if (e < rn * rn) {
          const int p = e / rn, q = e - p * rn;
          double g = gacc[k];
          for (int tt = 0; tt < n; ++tt) {
            const long long bb = sb[tt];
            if (bb >= 0) {
              g = fma(skw[tt][p], skw[tt][q], g);
            } else if (p == q && (int)(-1 - bb) == p) {
              const double w2 = sw[tt] * sw[tt];
              g = fma(w2 * f.root_lambda, f.root_lambda, g);
            }
          }
          gacc[k] = g;
        }
      }
    }
  }
  if (col) {
    double* o = part + ((size_t)blockIdx.x * f.in + i) * RM;
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      o[r] = acc0[r];
      o[RM + r] = acc1[r];
    }
  }
  if (do_gram) {
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      const int e = threadIdx.x + k * kT2;
      if (e < rn * rn) gpart[(size_t)blockIdx.x * rn * rn + e] = gacc[k];
    }
  }
}

// Contiguous fibers, TMA-staged: one CTA per chunk of draws. Warp 0 scans the chunk's draws
// (32 at a time, ballot on "data draw") and bulk-copies each data draw's fiber (I_n values,
// contiguous in the mode-n-last copy) and its w k row into a kFq-deep ring of kFg-fiber
// stages (full mbarrier with the byte count, empty mbarrier per consumer warp); 8 consumer
// warps, thread = 2 adjacent columns of up to 512 (I_n <= 2 * 256 * kFcols), accumulate
// M[i] += x_t[i] (w_t k_t) from shared memory. The bytes in flight per SM are the ring, not
// registers, so the gather runs at HBM speed. The chunk's Gram partial comes from the same
// staged w k rows (one entry per consumer thread, R_n^2 <= 256) plus the augmented diagonal
// (count per column x the common weight^2 x lambda).
constexpr int kFg = 8;       // fibers per stage
constexpr int kFq = 4;       // stages
constexpr int kFthreads = 9 * 32;
template <int RM>
__global__ void __launch_bounds__(kFthreads, 1) k_fsk_accum3(FskDev f, const double* __restrict__ x,
                                                           const double* __restrict__ kw,
                                                           const long long* __restrict__ base,
                                                           const double* __restrict__ wts,
                                                           unsigned long long s, long long chunk,
                                                           double* __restrict__ part,
                                                           double* __restrict__ gpart) {
  extern __shared__ __align__(16) double fsm[];
  const int in = f.in;
  const int ldf = in + 2;                              // fiber row stride (16-byte aligned)
  double* fib = fsm;                                   // [kFq][kFg][ldf]
  double* kws = fib + (size_t)kFq * kFg * ldf;         // [kFq][kFg][RM]  (w k)
  __shared__ __align__(8) unsigned long long full[kFq], empty[kFq];
  __shared__ int cnt[kFq];                             // fibers in the stage (0: end)
  __shared__ double wfib[kFq][kFg];                    // w_t of each staged fiber
  __shared__ int aug_cnt[RM];                          // augmented draws per column
  __shared__ double aug_w2;                            // their (common) weight^2
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < RM) aug_cnt[tid] = 0;
  if (tid == 0) aug_w2 = 0.0;
  const long long t0 = (long long)blockIdx.x * chunk;
  const long long t1 = min((long long)s, t0 + chunk);
  if (tid == 0) {
    for (int q = 0; q < kFq; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kFthreads / 32 - 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 0) {  // producer
    unsigned q = 0;
    int fill = 0;
    long long my_t = 0, my_b = 0;  // lane k holds the k-th fiber of the stage being filled
    auto flush = [&](bool last) {
      const int sb = (int)(q % kFq);
      if (q >= kFq) mbar_wait(&empty[sb], ((q / kFq) - 1) & 1);
      if (lane == 0) cnt[sb] = last && fill == 0 ? 0 : fill;
      if (lane < fill) wfib[sb][lane] = wts[my_t];
      __syncwarp();
      const unsigned bytes = (unsigned)fill * ((unsigned)in * 8u + RM * 8u);
      if (lane == 0) mbar_arrive_expect_tx(&full[sb], bytes);
      __syncwarp();
      if (lane < fill) {
        bulk_g2s(fib + ((size_t)sb * kFg + lane) * ldf, x + my_b, in * 8, &full[sb]);
        bulk_g2s(kws + ((size_t)sb * kFg + lane) * RM, kw + my_t * RM, RM * 8, &full[sb]);
      }
      ++q;
      fill = 0;
    };
    for (long long tb = t0; tb < t1; tb += 32) {
      const long long t = tb + lane;
      const long long bb = t < t1 ? base[t] : 0;
      if (t < t1 && bb < 0) {  // augmented draw of column -1 - bb (all share one weight)
        atomicAdd(&aug_cnt[(int)(-1 - bb)], 1);
        aug_w2 = wts[t] * wts[t];
      }
      unsigned m = __ballot_sync(0xffffffffu, t < t1 && bb >= 0);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const long long b_src = __shfl_sync(0xffffffffu, bb, src);
        if (lane == fill) {
          my_b = b_src;
          my_t = tb + src;
        }
        ++fill;
        if (fill == kFg) flush(false);
      }
    }
    if (fill) flush(false);
    flush(true);  // end marker
    return;
  }
  // consumers: thread (warp - 1, lane) owns columns 2 c, 2 c + 1 for c = tid - 32 + 256 j
  const int c0 = tid - 32;
  constexpr int kCols = 2;  // column pairs per thread: I_n <= 2 * 256 * kCols
  double acc[kCols][2][RM];
#pragma unroll
  for (int a = 0; a < kCols; ++a)
#pragma unroll
    for (int r = 0; r < RM; ++r) acc[a][0][r] = acc[a][1][r] = 0.0;
  // Gram entry (gp, gq) of this thread over the data draws (w k staged with the fibers)
  const int rn = f.rn;
  const bool gth = c0 < rn * rn;
  const int gp = gth ? c0 / rn : 0, gq = gth ? c0 - gp * rn : 0;
  double gacc = 0.0;
  for (unsigned q = 0;; ++q) {
    const int sb = (int)(q % kFq);
    mbar_wait(&full[sb], (q / kFq) & 1);
    const int n = cnt[sb];
    if (n == 0) break;
    for (int j = 0; j < n; ++j) {
      const double* fr = fib + ((size_t)sb * kFg + j) * ldf;
      const double* kr = kws + ((size_t)sb * kFg + j) * RM;
      const double wj = wfib[sb][j];
      if (gth) gacc = fma(kr[gp], kr[gq], gacc);
#pragma unroll
      for (int a = 0; a < kCols; ++a) {
        const int i = 2 * (c0 + 256 * a);
        if (i < in) {
          double2 xv = *reinterpret_cast<const double2*>(fr + i);
          xv.x *= wj;  // M += (w x)(w k)^T, as k_fsk_accum
          xv.y *= wj;
#pragma unroll
          for (int r = 0; r < RM; r += 2) {
            const double2 k2 = *reinterpret_cast<const double2*>(kr + r);
            acc[a][0][r] = fma(k2.x, xv.x, acc[a][0][r]);
            acc[a][0][r + 1] = fma(k2.y, xv.x, acc[a][0][r + 1]);
            acc[a][1][r] = fma(k2.x, xv.y, acc[a][1][r]);
            acc[a][1][r + 1] = fma(k2.y, xv.y, acc[a][1][r + 1]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sb]);
  }
  if (gth) {
    if (gp == gq && aug_cnt[gp]) gacc += (double)aug_cnt[gp] * ((aug_w2 * f.root_lambda) * f.root_lambda);
    gpart[(size_t)blockIdx.x * rn * rn + c0] = gacc;
  }
#pragma unroll
  for (int a = 0; a < kCols; ++a) {
    const int i = 2 * (c0 + 256 * a);
    if (i < in) {
      double* o = part + ((size_t)blockIdx.x * in + i) * RM;
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        o[r] = acc[a][0][r];
        o[RM + r] = acc[a][1][r];
      }
    }
  }
}

// One warp per output entry: lanes stride over the chunk partials, a fixed butterfly sums
// the lanes (deterministic; the chunk partials of one entry are read in parallel).
template <int RM>
__global__ void k_fsk_reduce(const double* __restrict__ part, const double* __restrict__ gpart,
                             int nchunks, int in, int rn, double* __restrict__ M,
                             double* __restrict__ gram) {
  const long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nm = (long long)in * rn;
  if (e >= nm + (long long)rn * rn) return;
  double acc = 0.0;
  if (e < nm) {
    const long long i = e / rn, r = e - i * rn;
    for (int c = lane; c < nchunks; c += 32) acc += __ldg(part + ((size_t)c * in + i) * RM + r);
  } else {
    const long long g = e - nm;
    for (int c = lane; c < nchunks; c += 32) acc += __ldg(gpart + (size_t)c * rn * rn + g);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    if (e < nm) M[e] = acc;
    else gram[e - nm] = acc;
  }
}

int rm_of(int rn) { return rn <= 8 ? 8 : rn <= 16 ? 16 : 32; }

size_t tma_smem(int in, int rm) { return ((size_t)kFq * kFg * (in + 2) + (size_t)kFq * kFg * rm) * 8; }

struct FskLayout {
  int nchunks;
  long long chunk;
  double* gt;
  unsigned long long* qdig;
  double* kw;
  long long* base;
  double* part;
  double* gpart;
  size_t bytes;
};

// the TMA-staged gather applies: contiguous fibers of even length <= 1024, R_n^2 <= 256
// fiber length in x: mode 1 under sharding holds this shard's rows only
int fsk_in(const FactorSketchSpec& sp) {
  return (sp.mode == 0 && sp.shard_rows > 0) ? sp.shard_rows : sp.rows[sp.mode];
}

bool fsk_tma(const FactorSketchSpec& sp) {
  const int n = sp.mode, in = fsk_in(sp), rn = sp.ranks[n];
  const bool contiguous = (sp.x_mode_last || n == sp.order - 1) && in % 2 == 0 &&
                          std::getenv("RTB_NO_FSK2") == nullptr;
  return contiguous && in <= 1024 && rn * rn <= 256 && tma_smem(in, rm_of(rn)) <= 220 * 1024 &&
         std::getenv("RTB_NO_FSK3") == nullptr;
}

FskLayout fsk_layout(const FactorSketchSpec& sp, void* work) {
  const int RM = rm_of(sp.ranks[sp.mode]);
  const int in = fsk_in(sp), rn = sp.ranks[sp.mode];
  const int tiles = ceil_div(in, kTile);
  const long long s = (long long)sp.s;
  // one wave of work units: the TMA gather runs one CTA per SM (fewer chunk partials too)
  const int units = fsk_tma(sp) ? kNumSMs : 4 * kNumSMs / tiles;
  int nchunks = std::max(1, std::min<int>((int)ceil_div<long long>(s, kSub), units));
  long long chunk = ceil_div<long long>(ceil_div<long long>(s, nchunks), kSub) * kSub;
  nchunks = (int)ceil_div<long long>(s, chunk);
  FskLayout l{};
  l.nchunks = nchunks;
  l.chunk = chunk;
  char* p = static_cast<char*>(work);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = p ? p + off : nullptr;
    off += (bytes + 255) & ~size_t(255);
    return r;
  };
  int width = 1;
  for (int m = 0; m < sp.order; ++m)
    if (m != sp.mode) width *= sp.ranks[m];
  l.gt = reinterpret_cast<double*>(take((size_t)width * RM * 8));
  l.qdig = reinterpret_cast<unsigned long long*>(take((size_t)width * 8));
  l.kw = reinterpret_cast<double*>(take((size_t)s * RM * 8));
  l.base = reinterpret_cast<long long*>(take((size_t)s * 8));
  l.part = reinterpret_cast<double*>(take((size_t)nchunks * in * RM * 8));
  l.gpart = reinterpret_cast<double*>(take((size_t)nchunks * rn * rn * 8));
  l.bytes = off;
  return l;
}

}  // namespace

size_t factor_sketch_work_bytes(const FactorSketchSpec& sp) { return fsk_layout(sp, nullptr).bytes; }

namespace {
// [A][In][B] -> [A][B][In]: 32 x 32 tiles through shared memory, batch a = blockIdx.z
__global__ void k_move_axis_last(const double* __restrict__ x, int In, long long B,
                                 double* __restrict__ out) {
  __shared__ double tile[32][33];
  const long long a = blockIdx.z;
  const int i0 = blockIdx.y * 32;
  const long long b0 = (long long)blockIdx.x * 32;
  const double* xa = x + a * In * B;
  double* oa = out + a * In * B;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + r;
    const long long b = b0 + threadIdx.x;
    if (i < In && b < B) tile[r][threadIdx.x] = xa[(long long)i * B + b];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const long long b = b0 + r;
    const int i = i0 + threadIdx.x;
    if (i < In && b < B) oa[b * In + i] = tile[threadIdx.x][r];
  }
}
}  // namespace

void move_axis_last(const double* x, long long A, int In, long long B, double* out,
                    cudaStream_t st) {
  if (A > 65535) throw Error(4, "move_axis_last: batch too large");
  const dim3 grid((unsigned)ceil_div<long long>(B, 32), (unsigned)ceil_div(In, 32), (unsigned)A);
  k_move_axis_last<<<grid, dim3(32, 8), 0, st>>>(x, In, B, out);
  RTB_LAUNCH_CHECK();
}

void factor_sketch_normal_eq(const FactorSketchSpec& sp, const unsigned long long* idx,
                             const double* w, void* work, double* gram, double* M,
                             cudaStream_t st) {
  if (sp.order < 2 || sp.order > 8 || sp.mode < 0 || sp.mode >= sp.order)
    throw Error(1, "factor_sketch: bad order/mode");
  const int n = sp.mode, rn = sp.ranks[n];
  if (rn < 1 || rn > 32) throw Error(1, "factor_sketch: R_n must be in [1, 32]");
  FskDev f{};
  f.order = sp.order;
  f.mode = n;
  f.rn = rn;
  f.in = fsk_in(sp);
  const bool sharded = sp.shard_rows > 0;
  if (sharded && (sp.shard_lo < 0 || sp.shard_lo + sp.shard_rows > sp.rows[0]))
    throw Error(1, "factor_sketch: bad shard rows");
  long long xs[8];
  int cs[8];
  {
    // X strides over the rows x actually holds (mode 1: this shard's)
    int xr[8];
    for (int m = 0; m < sp.order; ++m) xr[m] = (m == 0 && sharded) ? sp.shard_rows : sp.rows[m];
    long long a = 1;
    int c = 1;
    for (int m = sp.order - 1; m >= 0; --m) {
      xs[m] = a;
      cs[m] = c;
      a *= xr[m];
      c *= sp.ranks[m];
    }
    if (sp.x_mode_last) {  // axes: other modes ascending, then mode n (stride 1)
      a = xr[n];
      xs[n] = 1;
      for (int m = sp.order - 1; m >= 0; --m) {
        if (m == n) continue;
        xs[m] = a;
        a *= xr[m];
      }
    }
  }
  f.o0_lo = (sharded && n > 0) ? sp.shard_lo : 0;
  f.o0_hi = (sharded && n > 0) ? sp.shard_lo + sp.shard_rows : 0;
  f.skip_aug = (sharded && n > 0 && !sp.count_aug) ? 1 : 0;
  f.cstride_n = cs[n];
  f.xstride_n = xs[n];
  f.width = 1;
  f.total_other = 1;
  int k = 0;
  for (int m = 0; m < sp.order; ++m) {
    if (m == n) continue;
    f.orow[k] = sp.rows[m];
    f.orank[k] = sp.ranks[m];
    f.oxstride[k] = xs[m];
    f.ocstride[k] = cs[m];
    f.ofac[k] = sp.factors[m];
    f.width *= sp.ranks[m];
    f.total_other *= (unsigned long long)sp.rows[m];
    ++k;
  }
  f.nother = k;
  f.root_lambda = std::sqrt(sp.lambda);
  if (sp.s == 0) throw Error(1, "solve_sketched_ridge: sample count must be positive");
  FskLayout l = fsk_layout(sp, work);
  const int RM = rm_of(rn);
  const bool contiguous = f.xstride_n == 1 && f.in % 2 == 0 &&
                          std::getenv("RTB_NO_FSK2") == nullptr;
  // TMA-staged gather: one CTA per chunk, one chunk per SM (fsk_layout)
  const bool tma = fsk_tma(sp);
  // 8 draws per warp, 8 warps per block
  const unsigned rows_blocks = (unsigned)ceil_div<unsigned long long>(sp.s, 64ULL);
  int srow = 0;
  for (int m = 0; m < f.nother; ++m) srow += f.orank[m];
  const size_t rows_smem = (size_t)8 * 8 * srow * 8 + 8 * 8 * sizeof(int) + 8 * 64 * sizeof(int);
  const dim3 agrid(l.nchunks, ceil_div(f.in, kTile));
  const long long tot = (long long)f.in * rn + (long long)rn * rn;
  const unsigned rblocks = (unsigned)ceil_div<long long>(tot * 32, 256);
#define RTB_FSK(RMV)                                                                             \
  k_fsk_unfold<RMV><<<ceil_div(f.width, 128), 128, 0, st>>>(f, sp.core, l.gt, l.qdig);          \
  RTB_LAUNCH_CHECK();                                                                            \
  if (rows_smem > 48 * 1024)                                                                     \
    set_max_smem(k_fsk_rows<RMV>, (int)rows_smem);                                               \
  k_fsk_rows<RMV><<<rows_blocks, 256, rows_smem, st>>>(f, l.gt, l.qdig, idx, w, sp.s, srow, l.kw, \
                                                       l.base);                                \
  RTB_LAUNCH_CHECK();                                                                            \
  if (tma) {                                                                                     \
    set_max_smem(k_fsk_accum3<RMV>, (int)tma_smem(f.in, RMV));                                   \
    k_fsk_accum3<RMV><<<l.nchunks, kFthreads, tma_smem(f.in, RMV), st>>>(                        \
        f, sp.x, l.kw, l.base, w, sp.s, l.chunk, l.part, l.gpart);                               \
  } else if (contiguous)                                                                         \
    k_fsk_accum2<RMV><<<agrid, kT2, 0, st>>>(f, sp.x, l.kw, l.base, w, sp.s, l.chunk, l.part,   \
                                             l.gpart);                                           \
  else                                                                                           \
    k_fsk_accum<RMV><<<agrid, kTile, 0, st>>>(f, sp.x, l.kw, l.base, w, sp.s, l.chunk, l.part,  \
                                              l.gpart);                                          \
  RTB_LAUNCH_CHECK();                                                                            \
  k_fsk_reduce<RMV><<<rblocks, 256, 0, st>>>(l.part, l.gpart, l.nchunks, f.in, rn, M, gram);    \
  RTB_LAUNCH_CHECK();
  if (RM == 8) {
    RTB_FSK(8)
  } else if (RM == 16) {
    RTB_FSK(16)
  } else {
    RTB_FSK(32)
  }
#undef RTB_FSK
}

}  // namespace rtb
