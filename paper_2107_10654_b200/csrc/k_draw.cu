// k_draw.cu -- the reference's sequential sketch draw stream, decoded in parallel.
//
// solve_sketched_ridge draws s rows one after another from ONE SplitMix64
// stream (ref sketch_ridge.cpp:80-90) with ProductLeverageSampler::draw
// (ref kronecker.cpp:172-181):
//   coin = next_double() < 1/2                      (1 output; bit 63 == 0)
//   data: N x [next_double() * S_n -> upper_bound]  (N outputs)
//   aug : next_below(d)                             (1 output + rejections)
// so the stream position of draw t depends on every earlier coin. SplitMix64 is
// counter based (output k = mix(seed + (k+1) gamma)), so we
//   1. k_draw_submaps: for every sub-chunk of SUB stream positions and every
//      possible entry offset e < L (L = longest rejection-free draw) simulate
//      the draw boundaries inside the sub-chunk -> exit offset + draw count;
//   2. k_draw_group / k_draw_scan / k_draw_fix: the small maps are composed per
//      group of GS sub-chunks (walks in shared memory), one CTA composes the group
//      maps with a block scan, then each group re-walks its sub-chunks from its true
//      entry: every sub-chunk's entry offset and first draw id;
//   3. k_draw_emit:    each sub-chunk re-walks from its true entry and records
//      the stream position of each of its draws;
//   4. k_draw_eval:    one thread per draw evaluates it exactly as the
//      reference does (same IEEE operations, no FMA contraction), giving
//      bit-identical indices and weights for identical CDFs.
// A draw longer than L (a next_below rejection, probability ~ (2^64 mod d)/2^64
// per augmented draw, zero when d is a power of two) trips a flag and the scan
// CTA falls back to an exact serial walk on the device.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace rtb {

namespace {
constexpr int SUB = 128;
constexpr int LMAX = 9;  // order <= 8

struct StreamCfg {
  unsigned long long seed;
  const unsigned long long* seed_ptr;  // non-null: the seed is read from device memory
  unsigned long long thr;  // (2^64 - d) % d: next_below rejection threshold
  int data_step;           // 1 + order
};

__device__ __forceinline__ long long step_at(const StreamCfg& c, long long pos) {
  const uint64_t u = sm_at(c.seed, (uint64_t)pos);
  if ((u >> 63) == 0) return c.data_step;  // next_double() < 0.5
  long long q = pos + 1;
  while (sm_at(c.seed, (uint64_t)q) < c.thr) ++q;  // rejection (rare)
  return q + 1 - pos;
}

constexpr int GS = 16;   // sub-chunks per group (first level of the map composition)
constexpr int GCTA = 64;   // groups (threads) per CTA in k_draw_group / k_draw_fix

struct Layout {
  long long nsub, ngrp;
  unsigned char* gexit;  // [ngrp][L] composed group maps
  int* gcnt;             // [ngrp][L]
  int* gentry;           // [ngrp]
  long long* gbase;      // [ngrp]
  unsigned char* exitm;  // [nsub][L]
  unsigned short* cnt;   // [nsub][L]
  int* entry;            // [nsub]
  long long* base;       // [nsub]
  long long* start;      // [s] stream position of each draw
  int* overflow;         // [1]
};

Layout layout(const DrawSpec& spec, void* base) {
  const int L = spec.order + 1 > 2 ? spec.order + 1 : 2;
  const long long positions = (long long)spec.s * (spec.order + 1) + 2 * SUB;
  Layout l;
  l.nsub = ceil_div<long long>(positions, SUB);
  l.ngrp = ceil_div<long long>(l.nsub, GS);
  char* p = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  l.exitm = reinterpret_cast<unsigned char*>(take(l.nsub * L));
  l.cnt = reinterpret_cast<unsigned short*>(take(l.nsub * L * sizeof(unsigned short)));
  l.entry = reinterpret_cast<int*>(take(l.nsub * sizeof(int)));
  l.base = reinterpret_cast<long long*>(take(l.nsub * sizeof(long long)));
  l.start = reinterpret_cast<long long*>(take(spec.s * sizeof(long long)));
  l.overflow = reinterpret_cast<int*>(take(sizeof(int)));
  l.gexit = reinterpret_cast<unsigned char*>(take(l.ngrp * L));
  l.gcnt = reinterpret_cast<int*>(take(l.ngrp * L * sizeof(int)));
  l.gentry = reinterpret_cast<int*>(take(l.ngrp * sizeof(int)));
  l.gbase = reinterpret_cast<long long*>(take(l.ngrp * sizeof(long long)));
  return l;
}
}  // namespace

size_t draw_work_bytes(const DrawSpec& spec) {
  const int L = spec.order + 1 > 2 ? spec.order + 1 : 2;
  const long long positions = (long long)spec.s * (spec.order + 1) + 2 * SUB;
  const long long nsub = ceil_div<long long>(positions, SUB);
  size_t b = 0;
  auto add = [&](size_t bytes) { b += (bytes + 255) & ~size_t(255); };
  add(nsub * L);
  add(nsub * L * sizeof(unsigned short));
  add(nsub * sizeof(int));
  add(nsub * sizeof(long long));
  add(spec.s * sizeof(long long));
  add(sizeof(int));
  const long long ngrp = ceil_div<long long>(nsub, GS);
  add(ngrp * L);
  add(ngrp * L * sizeof(int));
  add(ngrp * sizeof(int));
  add(ngrp * sizeof(long long));
  return b;
}

__global__ void k_draw_submaps(StreamCfg c, int L, long long nsub, unsigned char* exitm,
                               unsigned short* cnt, int* overflow) {
  if (c.seed_ptr) c.seed = *c.seed_ptr;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nsub * L) return;
  const long long j = e / L;
  const int entry = (int)(e % L);
  const long long end = (j + 1) * SUB;
  long long pos = j * SUB + entry;
  int n = 0;
  while (pos < end) {
    pos += step_at(c, pos);
    ++n;
  }
  const long long ex = pos - end;
  if (ex >= L) {
    atomicExch(overflow, 1);
    exitm[e] = 0;
  } else {
    exitm[e] = (unsigned char)ex;
  }
  cnt[e] = (unsigned short)n;
}

// Stage the sub-chunk maps of GCTA groups (GCTA * GS sub-chunks) in shared memory, so the
// per-group walks below are chains of shared-memory loads, not of global loads.
__device__ __forceinline__ long long stage_maps(int L, long long nsub, const unsigned char* exitm,
                                                const unsigned short* cnt, unsigned char* sx,
                                                unsigned short* sc) {
  const long long j0 = (long long)blockIdx.x * GCTA * GS;
  const long long n = min((long long)GCTA * GS, nsub - j0) * L;
  for (long long e = threadIdx.x; e < n; e += blockDim.x) {
    sx[e] = exitm[j0 * L + e];
    sc[e] = cnt[j0 * L + e];
  }
  __syncthreads();
  return j0;
}

// First level: compose the maps of each group of GS sub-chunks (thread = group).
__global__ void __launch_bounds__(GCTA) k_draw_group(int L, long long nsub, long long ngrp,
                                                     const unsigned char* exitm,
                                                     const unsigned short* cnt,
                                                     unsigned char* gexit, int* gcnt) {
  __shared__ unsigned char sx[GCTA * GS * LMAX];
  __shared__ unsigned short sc[GCTA * GS * LMAX];
  const long long j0 = stage_maps(L, nsub, exitm, cnt, sx, sc);
  const long long g = (long long)blockIdx.x * GCTA + threadIdx.x;
  if (g >= ngrp) return;
  const int k0 = threadIdx.x * GS, k1 = (int)min((long long)k0 + GS, nsub - j0);
  for (int e = 0; e < L; ++e) {
    int cur = e, n = 0;
    for (int k = k0; k < k1; ++k) {
      n += sc[k * L + cur];
      cur = sx[k * L + cur];
    }
    gexit[g * L + e] = (unsigned char)cur;
    gcnt[g * L + e] = n;
  }
}

// Single CTA of 1024 threads: compose the group maps with a block scan and fix each
// group's true entry offset and first draw id.
// (CT = unsigned short: applied to the sub-chunk maps directly, when there are few)
template <typename CT>
__global__ void __launch_bounds__(1024) k_draw_scan(StreamCfg c, int L, long long nsub,
                                                   long long ngrp, const unsigned char* gexit,
                                                   const CT* gcnt, int* gentry, long long* gbase,
                                                   long long* base, const int* overflow,
                                                   long long* start, long long s) {
  if (c.seed_ptr) c.seed = *c.seed_ptr;
  __shared__ unsigned char mx[1024][LMAX];
  __shared__ int mc[1024][LMAX];  // draws per range (< 2^31)
  const int tid = threadIdx.x;
  if (*overflow) {
    // exact serial fallback: thread 0 walks the whole stream
    if (tid == 0) {
      long long pos = 0;
      for (long long t = 0; t < s; ++t) {
        start[t] = pos;
        pos += step_at(c, pos);
      }
      for (long long j = 0; j < nsub; ++j) base[j] = -1;  // tells emit to skip
    }
    return;
  }
  const long long per = ceil_div<long long>(ngrp, 1024);
  const long long j0 = tid * per, j1 = min(ngrp, j0 + per);
  // this thread's composed map over groups [j0, j1)
  unsigned char fx[LMAX];
  long long fc[LMAX];
  for (int e = 0; e < L; ++e) {
    int cur = e;
    long long n = 0;
    for (long long j = j0; j < j1; ++j) {
      n += gcnt[j * L + cur];
      cur = gexit[j * L + cur];
    }
    fx[e] = (unsigned char)cur;
    fc[e] = n;
  }
  for (int e = 0; e < L; ++e) {
    mx[tid][e] = fx[e];
    mc[tid][e] = (int)fc[e];
  }
  __syncthreads();
  // inclusive Hillis-Steele scan: P_i <- P_i o P_{i-d}
  for (int d = 1; d < 1024; d <<= 1) {
    unsigned char nx[LMAX];
    int nc[LMAX];
    if (tid >= d) {
      for (int e = 0; e < L; ++e) {
        const int mid = mx[tid - d][e];
        nx[e] = mx[tid][mid];
        nc[e] = mc[tid - d][e] + mc[tid][mid];
      }
    }
    __syncthreads();
    if (tid >= d)
      for (int e = 0; e < L; ++e) {
        mx[tid][e] = nx[e];
        mc[tid][e] = nc[e];
      }
    __syncthreads();
  }
  // exclusive prefix applied to entry 0
  int cur = tid == 0 ? 0 : mx[tid - 1][0];
  long long n = tid == 0 ? 0 : mc[tid - 1][0];
  for (long long j = j0; j < j1; ++j) {
    gentry[j] = cur;
    gbase[j] = n;
    n += gcnt[j * L + cur];
    cur = gexit[j * L + cur];
  }
}

// Second level: each group walks its GS sub-chunks from its true entry (thread = group).
__global__ void __launch_bounds__(GCTA) k_draw_fix(int L, long long nsub, long long ngrp,
                                                   const unsigned char* exitm,
                                                   const unsigned short* cnt, const int* gentry,
                                                   const long long* gbase, const int* overflow,
                                                   int* entry, long long* base) {
  __shared__ unsigned char sx[GCTA * GS * LMAX];
  __shared__ unsigned short sc[GCTA * GS * LMAX];
  if (*overflow) return;
  const long long j0 = stage_maps(L, nsub, exitm, cnt, sx, sc);
  const long long g = (long long)blockIdx.x * GCTA + threadIdx.x;
  if (g >= ngrp) return;
  const int k0 = threadIdx.x * GS, k1 = (int)min((long long)k0 + GS, nsub - j0);
  int cur = gentry[g];
  long long n = gbase[g];
  for (int k = k0; k < k1; ++k) {
    entry[j0 + k] = cur;
    base[j0 + k] = n;
    n += sc[k * L + cur];
    cur = sx[k * L + cur];
  }
}

__global__ void k_draw_emit(StreamCfg c, long long nsub, const int* entry, const long long* base,
                            long long* start, long long s) {
  if (c.seed_ptr) c.seed = *c.seed_ptr;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nsub) return;
  long long t = base[j];
  if (t < 0 || t >= s) return;
  const long long end = (j + 1) * SUB;
  long long pos = j * SUB + entry[j];
  while (pos < end && t < s) {
    start[t++] = pos;
    pos += step_at(c, pos);
  }
}

// Evaluate draw t at stream position start[t] (ref kronecker.cpp:125-144,
// 172-181; sketch_ridge.cpp:88: w = sqrt((1/s)/prob)).
__global__ void k_draw_eval(DrawSpec spec, StreamCfg c, const long long* start,
                            const double* scores, const double* cdfs, const double* sums,
                            unsigned long long* idx_out, double* w_out, int* flag) {
  if (c.seed_ptr) c.seed = *c.seed_ptr;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)spec.s) return;
  const long long pos = start[t];
  const uint64_t coin = sm_at(c.seed, (uint64_t)pos);
  const double p_data = 0.5;  // 1 / (1 + min(1, d - 0)), d >= 1
  const double inv_s = __ddiv_rn(1.0, (double)spec.s);
  double prob;
  unsigned long long index;
  if ((coin >> 63) == 0) {
    double probability = 1.0;
    unsigned long long flat = 0;
    for (int n = 0; n < spec.order; ++n) {
      const long long I = spec.rows[n];
      const double S = sums[n];
      if (!(S > 0.0)) atomicExch(flag, 1);  // ref kronecker.cpp:128-131 throws
      const double* cdf = cdfs + spec.cdf_off[n];
      const double* sc = scores + spec.cdf_off[n];
      const double u = __dmul_rn(u64_to_unit(sm_at(c.seed, (uint64_t)(pos + 1 + n))), S);
      // upper_bound: first i with cdf[i] > u
      long long lo = 0, len = I;
      while (len > 0) {
        const long long half = len >> 1;
        if (!(u < cdf[lo + half])) {
          lo += half + 1;
          len -= half + 1;
        } else {
          len = half;
        }
      }
      long long i = lo >= I ? I - 1 : lo;
      while (i > 0 && sc[i] == 0.0) --i;
      flat = flat * (unsigned long long)I + (unsigned long long)i;
      probability = __dmul_rn(probability, __ddiv_rn(sc[i], S));
    }
    index = flat;
    prob = __dmul_rn(probability, p_data);
  } else {
    long long q = pos + 1;
    uint64_t r = sm_at(c.seed, (uint64_t)q);
    while (r < c.thr) r = sm_at(c.seed, (uint64_t)(++q));
    index = spec.total_rows + (r % spec.d);
    prob = __ddiv_rn(__dadd_rn(1.0, -p_data), (double)spec.d);
  }
  idx_out[t] = index;
  w_out[t] = __dsqrt_rn(__ddiv_rn(inv_s, prob));
}

namespace {
StreamCfg stream_cfg(const DrawSpec& spec) {
  StreamCfg c;
  c.seed = spec.seed;
  c.seed_ptr = spec.seed_dev;
  c.thr = (0ULL - spec.d) % spec.d;
  c.data_step = 1 + spec.order;
  return c;
}
}  // namespace

// Steps 1-3: the stream position of every draw. Depends on the seed, s, d and the order only
// (not on the CDFs), so a sweep runs it as a side branch next to the factor updates.
void draw_decode(const DrawSpec& spec, DrawWork work, cudaStream_t st) {
  if (spec.s == 0) return;
  const int L = spec.order + 1 > 2 ? spec.order + 1 : 2;
  Layout l = layout(spec, work.base);
  const StreamCfg c = stream_cfg(spec);
  RTB_CUDA(cudaMemsetAsync(l.overflow, 0, sizeof(int), st));
  // test hook: take the exact serial walk (the path a next_below rejection triggers, which
  // real seeds reach with probability ~ (2^64 mod d) / 2^64 per augmented draw)
  static const bool force_serial = std::getenv("RTB_DRAW_FORCE_SERIAL") != nullptr;
  if (force_serial) RTB_CUDA(cudaMemsetAsync(l.overflow, 1, 1, st));
  const long long n1 = l.nsub * L;
  k_draw_submaps<<<(unsigned)ceil_div<long long>(n1, 256), 256, 0, st>>>(c, L, l.nsub, l.exitm,
                                                                       l.cnt, l.overflow);
  RTB_LAUNCH_CHECK();
  if (l.nsub <= 8 * 1024) {  // few sub-chunks: one scan CTA composes them directly
    k_draw_scan<unsigned short><<<1, 1024, 0, st>>>(c, L, l.nsub, l.nsub, l.exitm, l.cnt, l.entry,
                                                    l.base, l.base, l.overflow, l.start,
                                                    (long long)spec.s);
    RTB_LAUNCH_CHECK();
  } else {
    const unsigned gb = (unsigned)ceil_div<long long>(l.ngrp, GCTA);
    k_draw_group<<<gb, GCTA, 0, st>>>(L, l.nsub, l.ngrp, l.exitm, l.cnt, l.gexit, l.gcnt);
    RTB_LAUNCH_CHECK();
    k_draw_scan<int><<<1, 1024, 0, st>>>(c, L, l.nsub, l.ngrp, l.gexit, l.gcnt, l.gentry, l.gbase,
                                         l.base, l.overflow, l.start, (long long)spec.s);
    RTB_LAUNCH_CHECK();
    k_draw_fix<<<gb, GCTA, 0, st>>>(L, l.nsub, l.ngrp, l.exitm, l.cnt, l.gentry, l.gbase,
                                    l.overflow, l.entry, l.base);
    RTB_LAUNCH_CHECK();
  }
  k_draw_emit<<<(unsigned)ceil_div<long long>(l.nsub, 128), 128, 0, st>>>(
      c, l.nsub, l.entry, l.base, l.start, (long long)spec.s);
  RTB_LAUNCH_CHECK();
}

// Step 4 on the positions draw_decode left in the workspace.
void draw_evaluate(const DrawSpec& spec, const double* scores, const double* cdfs,
                   const double* sums, DrawWork work, unsigned long long* idx_out, double* w_out,
                   int* flag_dev, cudaStream_t st) {
  if (spec.s == 0) return;
  Layout l = layout(spec, work.base);
  const StreamCfg c = stream_cfg(spec);
  k_draw_eval<<<(unsigned)ceil_div<unsigned long long>(spec.s, 256ULL), 256, 0, st>>>(
      spec, c, l.start, scores, cdfs, sums, idx_out, w_out, flag_dev);
  RTB_LAUNCH_CHECK();
}

// The first-mode half of k_draw_eval fused with k_sketch_keys (k_gram.cu): a data draw's i_1
// is fixed by its first uniform and A_1's CDF alone (modes are drawn in order, ref
// kronecker.cpp:125-144), so the bucket keys, the bucket histogram and the augmented-row
// histogram -- exactly what k_sketch_keys derives from the evaluated indices -- can be made
// as soon as A_1 is final, while A_2 and A_3 are still being updated.
__global__ void k_draw_keys(DrawSpec spec, StreamCfg c, const long long* start,
                            const double* scores, const double* cdfs, const double* sums,
                            int i1_lo, int i1_hi, unsigned* keys, unsigned* vals, int* counts,
                            int* aug_count, unsigned long long* data_draws) {
  if (c.seed_ptr) c.seed = *c.seed_ptr;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)spec.s) return;
  const long long pos = start[t];
  const uint64_t coin = sm_at(c.seed, (uint64_t)pos);
  const unsigned I1 = (unsigned)spec.rows[0];
  vals[t] = (unsigned)t;
  if ((coin >> 63) == 0) {
    const long long I = spec.rows[0];
    const double S = sums[0];
    const double* cdf = cdfs + spec.cdf_off[0];
    const double* sc = scores + spec.cdf_off[0];
    const double u = __dmul_rn(u64_to_unit(sm_at(c.seed, (uint64_t)(pos + 1))), S);
    long long lo = 0, len = I;
    while (len > 0) {
      const long long half = len >> 1;
      if (!(u < cdf[lo + half])) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    long long i = lo >= I ? I - 1 : lo;
    while (i > 0 && sc[i] == 0.0) --i;
    if (i1_hi > 0 && ((int)i < i1_lo || (int)i >= i1_hi)) {
      keys[t] = I1;  // another shard's draw
      return;
    }
    keys[t] = (unsigned)i;
    atomicAdd(&counts[i], 1);
    atomicAdd(data_draws, 1ULL);
  } else {
    long long q = pos + 1;
    uint64_t r = sm_at(c.seed, (uint64_t)q);
    while (r < c.thr) r = sm_at(c.seed, (uint64_t)(++q));
    keys[t] = I1;
    atomicAdd(&aug_count[r % spec.d], 1);
  }
}

void draw_keys(const DrawSpec& spec, const double* scores, const double* cdfs, const double* sums,
               DrawWork work, int i1_lo, int i1_hi, unsigned* keys, unsigned* vals, int* counts,
               int* aug_count, unsigned long long* data_draws, cudaStream_t st) {
  if (spec.s == 0) return;
  Layout l = layout(spec, work.base);
  const StreamCfg c = stream_cfg(spec);
  k_draw_keys<<<(unsigned)ceil_div<unsigned long long>(spec.s, 256ULL), 256, 0, st>>>(
      spec, c, l.start, scores, cdfs, sums, i1_lo, i1_hi, keys, vals, counts, aug_count,
      data_draws);
  RTB_LAUNCH_CHECK();
}

void draw_sketch(const DrawSpec& spec, const double* scores, const double* cdfs,
                 const double* sums, DrawWork work, unsigned long long* idx_out, double* w_out,
                 int* flag_dev, cudaStream_t st) {
  draw_decode(spec, work, st);
  draw_evaluate(spec, scores, cdfs, sums, work, idx_out, w_out, flag_dev, st);
}

}  // namespace rtb
