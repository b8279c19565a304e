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
// The Gram is the core-Gram machinery of k_gram.cu with order 2 (vech/Kronecker
// factored). The RHS is factored the same way: draws sorted by (j2, j3), so for each j2
// bucket D_b = sum_{t in b} w^2 a3(j3_t) x_t^T (R3 x I1) and RHS = sum_b a2(b) (x) D_b:
// 2 R3 I1 flops per data draw instead of 2 W I1.
//
// k_c4_fiber_rhs: one CTA per 16-column tile of the fiber index i (I1 / 16 CTAs); see
// the kernel comment for the pipeline.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace rtb {

namespace {

constexpr int kC4Tile = 16;    // fiber columns per CTA

__global__ void k_c4_keys(const unsigned long long* __restrict__ idx, unsigned long long s,
                          unsigned long long total, int I3, unsigned long long* keys,
                          unsigned* vals, int* counts) {
  const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  const unsigned long long id = idx[t];
  const bool data = id < total;
  keys[t] = data ? id : total;
  vals[t] = (unsigned)t;
  if (data) atomicAdd(counts + (int)(id / (unsigned long long)I3), 1);
}

// sorted draw records: j3 and w^2 of each data draw in (j2, j3) order (one gather of w)
__global__ void k_c4_records(const unsigned long long* __restrict__ keys_s,
                             const unsigned* __restrict__ vals_s, const double* __restrict__ w,
                             unsigned long long n, int I3, int* __restrict__ j3s,
                             double* __restrict__ w2s) {
  const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double wt = w[vals_s[t]];
  j3s[t] = (int)(keys_s[t] % (unsigned long long)I3);
  w2s[t] = wt * wt;
}

// exclusive scan of the I2 bucket counts (one block)
__global__ void __launch_bounds__(1024) k_c4_scan(int n, const int* counts, int* start) {
  __shared__ int part[1024];
  const int per = (n + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  int s = 0;
  for (int i = 0; i < per; ++i)
    if (b0 + i < n) s += counts[b0 + i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int run = threadIdx.x > 0 ? part[threadIdx.x - 1] : 0;
  for (int i = 0; i < per; ++i)
    if (b0 + i < n) {
      start[b0 + i] = run;
      run += counts[b0 + i];
    }
}

__global__ void k_c4_chunk_counts(int I2, const int* __restrict__ counts, int* __restrict__ ccnt) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < I2) ccnt[b] = (counts[b] + 255) / 256;
}
__global__ void k_c4_total(int I2, const int* ccnt, const int* cstart, int* total) {
  *total = I2 > 0 ? cstart[I2 - 1] + ccnt[I2 - 1] : 0;
}

// chunk descriptors: chunk c covers draws [start, start + len) of bucket b (len <= kQC)
constexpr int kQC = 256;  // draws per pipelined chunk
__global__ void k_c4_chunks(int I2, const int* __restrict__ bstart, const int* __restrict__ bcount,
                            const int* __restrict__ cstart, int4* __restrict__ chunks) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= I2) return;
  const int n = bcount[b], c0 = cstart[b];
  for (int k = 0; k * kQC < n; ++k) chunks[c0 + k] = make_int4(b, bstart[b] + k * kQC, min(kQC, n - k * kQC), 0);
}

// Pipelined RHS: the CTA's RHS tile (W x 16) lives in registers -- thread (q, i) =
// (tid / 16, tid % 16) holds RHS[(p, q), i] for all p. Chunks of <= 256 draws of one j2
// bucket flow through a two-buffer cp.async pipeline (a3 rows by 16 B copies, the
// tile's 16 fiber values per draw by 4 B copies -- FP32 kept in shared memory, upcast
// and scaled by w^2 at the fragment load -- and the next chunk's records), so the
// gathers of chunk c + 1 are in flight while warps 0-7 run chunk c's DMMAs into
// D (32 x 16). The limit is the cp.async issue rate of the staging (8 B a3 copies and
// 4 B fiber copies: ~12k per 256-draw chunk), not the DMMAs. At each bucket end D goes through shared memory and every thread folds
// RHS[(p, q), i] += a2(b)[p] D[q][i]. Fixed order: deterministic.
constexpr int kQLDT = 36;   // a3 rows, draw-major [k][q]: conflict-free A fragments
constexpr int kQLDB = 24;   // fiber values (floats) [k][i]: conflict-free B fragments
__global__ void __launch_bounds__(512, 1) k_c4_fiber_rhs(
    const float* __restrict__ X, int I1, int I2, int I3, const double* __restrict__ A2, int R2,
    const double* __restrict__ A3, int R3, const int* __restrict__ j3s,
    const double* __restrict__ w2s, const int4* __restrict__ chunks, const int* __restrict__ nchunks_p,
    double* __restrict__ rhs) {
  extern __shared__ __align__(16) double c4s[];
  double* At = c4s;                                    // [2][kQC][kQLDT]
  float* Bf = reinterpret_cast<float*>(At + 2 * kQC * kQLDT);  // [2][kQC][kQLDB]
  double* W2 = reinterpret_cast<double*>(Bf + 2 * kQC * kQLDB);  // [2][kQC]
  int* J3 = reinterpret_cast<int*>(W2 + 2 * kQC);      // [2][kQC]
  double* Ds = reinterpret_cast<double*>(J3 + 2 * kQC);  // [32][17]: D of the bucket
  double* a2s = Ds + 32 * 17;                          // [32]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int i0 = blockIdx.x * kC4Tile;
  const long long slab = (long long)I2 * I3;
  const int nch = *nchunks_p;
  const int mq = tid >> 4, mi = tid & 15;              // this thread's RHS column (q, i)
  const bool mma_warp = warp < 8;
  const int mt = warp >> 1, nt = warp & 1;
  double acc[32];
#pragma unroll
  for (int p = 0; p < 32; ++p) acc[p] = 0.0;
  // records of chunk c into record buffer c & 1
  auto load_records = [&](int c) {
    if (c >= nch) return;
    const int4 ch = chunks[c];
    const int rb = c & 1;
    for (int k = tid; k < kQC; k += blockDim.x) {
      const bool v = k < ch.z;
      cp_async4(J3 + rb * kQC + k, j3s + (v ? ch.y + k : 0), v);
      cp_async8(W2 + rb * kQC + k, w2s + (v ? ch.y + k : 0), v);
    }
  };
  // data of chunk c (its records landed) into data buffer c & 1
  auto load_data = [&](int c) {
    if (c >= nch) return;
    const int4 ch = chunks[c];
    const int db = c & 1;
    const int* j3 = J3 + db * kQC;
    const int kpad = (ch.z + 3) & ~3;
    // a3 rows: kpad x 32 doubles, 8 B copies (rows >= len and columns >= R3 zero-filled)
    for (int e = tid; e < kpad * 32; e += blockDim.x) {
      const int k = e >> 5, q = e & 31;
      const bool v = k < ch.z && q < R3;
      cp_async8(At + ((size_t)db * kQC + k) * kQLDT + q, A3 + (v ? (size_t)j3[k] * R3 + q : 0), v);
    }
    const long long rowb = (long long)ch.x * I3;
    for (int e = tid; e < kpad * kC4Tile; e += blockDim.x) {
      const int k = e >> 4, i = e & 15;
      const bool v = k < ch.z && i0 + i < I1;
      cp_async4(Bf + ((size_t)db * kQC + k) * kQLDB + i,
                X + (v ? (long long)(i0 + i) * slab + rowb + j3[k] : 0), v);
    }
  };
  load_records(0);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  load_data(0);
  load_records(1);
  cp_async_commit();
  double c0 = 0.0, c1 = 0.0;
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<0>();
    __syncthreads();  // chunk c's data and chunk c+1's records are in; buffers of c-1 free
    load_data(c + 1);
    // records of chunk c + 2 go to record buffer c & 1, whose chunk c is still read
    // below -- so they are issued after this chunk's DMMAs (next iteration's head)
    cp_async_commit();
    const int4 ch = chunks[c];
    const int db = c & 1;
    if (mma_warp) {
      const double* at = At + (size_t)db * kQC * kQLDT;
      const float* bf = Bf + (size_t)db * kQC * kQLDB;
      const double* w2 = W2 + db * kQC;
      const int kpad = (ch.z + 3) & ~3;
      for (int ks = 0; ks < kpad; ks += 4) {
        const int k = ks + t;
        const double a = at[k * kQLDT + mt * 8 + g];
        const double b = (double)bf[k * kQLDB + nt * 8 + g] * w2[k];
        dmma_8x8x4(c0, c1, a, b);
      }
    }
    const bool last_of_bucket = (c + 1 >= nch) || (chunks[c + 1].x != ch.x);
    if (last_of_bucket) {
      if (mma_warp) {
        Ds[(mt * 8 + g) * 17 + nt * 8 + 2 * t] = c0;
        Ds[(mt * 8 + g) * 17 + nt * 8 + 2 * t + 1] = c1;
      }
      if (tid < 32) a2s[tid] = tid < R2 ? A2[(size_t)ch.x * R2 + tid] : 0.0;
      c0 = c1 = 0.0;
      __syncthreads();
      const double dv = Ds[mq * 17 + mi];
#pragma unroll
      for (int p = 0; p < 32; ++p) acc[p] = fma(a2s[p], dv, acc[p]);
    }
    __syncthreads();  // record buffer c & 1 (chunk c) no longer read
    load_records(c + 2);
    cp_async_commit();
  }
  cp_async_wait<0>();
  if (mq < R3 && i0 + mi < I1) {
#pragma unroll
    for (int p = 0; p < 32; ++p)
      if (p < R2) rhs[(size_t)(p * R3 + mq) * I1 + i0 + mi] = acc[p];
  }
}

}  // namespace

size_t c4_fiber_work_bytes(unsigned long long s, int I2) {
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs<unsigned long long, unsigned>(
      nullptr, cub_bytes, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
      (const unsigned*)nullptr, (unsigned*)nullptr, (int)s);
  return (size_t)s * (8 + 8 + 4 + 4 + 4 + 8) + (size_t)I2 * 16 + cub_bytes +
         ((size_t)s / 256 + (size_t)I2 + 1) * 16 + 8192;
}

void c4_fiber_rhs(const float* x, int I1, int I2, int I3, const double* A2, int R2,
                  const double* A3, int R3, const unsigned long long* idx, const double* w,
                  unsigned long long s, void* work, size_t work_bytes, double* rhs,
                  cudaStream_t st) {
  if (R3 > 32 || R2 > 32) throw Error(1, "c4_fiber_rhs: ranks must be <= 32");
  if (work_bytes < c4_fiber_work_bytes(s, I2)) throw Error(4, "c4_fiber_rhs: workspace");
  char* p = static_cast<char*>(work);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  auto* keys = reinterpret_cast<unsigned long long*>(take(s * 8));
  auto* keys_s = reinterpret_cast<unsigned long long*>(take(s * 8));
  auto* vals = reinterpret_cast<unsigned*>(take(s * 4));
  auto* vals_s = reinterpret_cast<unsigned*>(take(s * 4));
  auto* counts = reinterpret_cast<int*>(take((size_t)I2 * 4));
  auto* start = reinterpret_cast<int*>(take((size_t)I2 * 4));
  auto* j3s = reinterpret_cast<int*>(take(s * 4));
  auto* w2s = reinterpret_cast<double*>(take(s * 8));
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs<unsigned long long, unsigned>(
      nullptr, cub_bytes, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
      (const unsigned*)nullptr, (unsigned*)nullptr, (int)s);
  void* cub_tmp = take(cub_bytes);
  const unsigned long long total = (unsigned long long)I2 * I3;
  int bits = 1;
  while ((1ULL << bits) <= total) ++bits;
  RTB_CUDA(cudaMemsetAsync(counts, 0, (size_t)I2 * 4, st));
  k_c4_keys<<<(unsigned)ceil_div<unsigned long long>(s, 256ULL), 256, 0, st>>>(idx, s, total, I3,
                                                                             keys, vals, counts);
  RTB_LAUNCH_CHECK();
  RTB_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, keys, keys_s, vals, vals_s, (int)s,
                                           0, bits, st));
  k_c4_scan<<<1, 1024, 0, st>>>(I2, counts, start);
  RTB_LAUNCH_CHECK();
  // records for the data draws (they sort first: aug draws carry the sentinel key)
  k_c4_records<<<(unsigned)ceil_div<unsigned long long>(s, 256ULL), 256, 0, st>>>(keys_s, vals_s, w,
                                                                                s, I3, j3s, w2s);
  RTB_LAUNCH_CHECK();
  // chunk descriptors (<= kQC draws, one bucket each)
  auto* ccnt = reinterpret_cast<int*>(take((size_t)I2 * 4));
  auto* cstart = reinterpret_cast<int*>(take((size_t)I2 * 4));
  auto* nch = reinterpret_cast<int*>(take(64));
  auto* chunks = reinterpret_cast<int4*>(take(((size_t)s / kQC + (size_t)I2 + 1) * 16));
  k_c4_chunk_counts<<<ceil_div(I2, 256), 256, 0, st>>>(I2, counts, ccnt);
  RTB_LAUNCH_CHECK();
  k_c4_scan<<<1, 1024, 0, st>>>(I2, ccnt, cstart);
  RTB_LAUNCH_CHECK();
  k_c4_total<<<1, 1, 0, st>>>(I2, ccnt, cstart, nch);
  RTB_LAUNCH_CHECK();
  k_c4_chunks<<<ceil_div(I2, 256), 256, 0, st>>>(I2, start, counts, cstart, chunks);
  RTB_LAUNCH_CHECK();
  const size_t smem = (size_t)2 * kQC * kQLDT * 8 + (size_t)2 * kQC * kQLDB * 4 +
                      (size_t)2 * kQC * 8 + (size_t)2 * kQC * 4 + (2 * 32 * 17 + 32) * 8;
  static bool attr = false;
  if (!attr) {
    RTB_CUDA(cudaFuncSetAttribute(k_c4_fiber_rhs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    attr = true;
  }
  k_c4_fiber_rhs<<<ceil_div(I1, kC4Tile), 512, smem, st>>>(x, I1, I2, I3, A2, R2, A3, R3, j3s,
                                                             w2s, chunks, nch, rhs);
  RTB_LAUNCH_CHECK();
}

}  // namespace rtb
