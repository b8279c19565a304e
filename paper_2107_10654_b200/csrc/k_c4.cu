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
// k_c4_fiber_rhs: one CTA per 16-column tile of the fiber index i (I1 / 16 CTAs) holds
// its RHS tile (W x 16) in shared memory; per bucket, 64-draw chunks are staged from
// precomputed sorted records (j3, w^2): A = a3 rows, B = w^2 times the gathered fiber
// values of the tile (16 sectors per draw, shared by neighbouring j3 after the sort),
// and 8 warps run m8n8k4 DMMAs into D (R3 x 16); at the bucket end D is folded into
// the tile with a2(b). Fixed order: deterministic.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace rtb {

namespace {

constexpr int kC4Tile = 16;    // fiber columns per CTA
constexpr int kC4Chunk = 64;   // draws staged per round
constexpr int kC4LDA = kC4Chunk + 4;
constexpr int kC4LDB = kC4Tile + 4;
constexpr int kC4LDR = kC4Tile + 1;

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

__global__ void __launch_bounds__(512, 1) k_c4_fiber_rhs(
    const float* __restrict__ X, int I1, int I2, int I3, const double* __restrict__ A2, int R2,
    const double* __restrict__ A3, int R3, const int* __restrict__ j3s,
    const double* __restrict__ w2s, const int* __restrict__ bstart, const int* __restrict__ bcount,
    double* __restrict__ rhs) {
  extern __shared__ __align__(16) double c4s[];
  const int W = R2 * R3;
  double* rt = c4s;                             // [W][kC4LDR] RHS tile
  double* As = rt + (size_t)W * kC4LDR;         // [32][kC4LDA]: a3 rows (q x draw)
  double* Bs = As + 32 * kC4LDA;                // [kC4Chunk][kC4LDB]: fiber values
  double* a2s = Bs + kC4Chunk * kC4LDB;         // [32]: a2 row of the bucket
  double* sw2 = a2s + 32;                       // [kC4Chunk]: w^2 of the chunk's draws
  int* sj3 = reinterpret_cast<int*>(sw2 + kC4Chunk);  // [kC4Chunk]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int i0 = blockIdx.x * kC4Tile;
  const long long slab = (long long)I2 * I3;    // X stride of mode 1
  for (int e = tid; e < W * kC4LDR; e += blockDim.x) rt[e] = 0.0;
  const bool mma_warp = warp < 8;
  const int mt = warp >> 1, nt = warp & 1;       // q rows 8 mt.., fiber columns 8 nt..
  for (int b = 0; b < I2; ++b) {
    const int n = bcount[b];
    if (n == 0) continue;
    const int st0 = bstart[b];
    if (tid < 32) a2s[tid] = tid < R2 ? A2[(size_t)b * R2 + tid] : 0.0;
    double c0 = 0.0, c1 = 0.0;
    for (int k0 = 0; k0 < n; k0 += kC4Chunk) {
      const int kn = min(kC4Chunk, n - k0);
      __syncthreads();
      // stage the chunk's records, then A[q][k] = a3(j3_t)[q] and B[k][i] = w_t^2 X[i0 + i, j2, j3_t]
      if (tid < kC4Chunk) {
        const int pos = st0 + k0 + tid;
        sj3[tid] = tid < kn ? j3s[pos] : 0;
        sw2[tid] = tid < kn ? w2s[pos] : 0.0;
      }
      __syncthreads();
      for (int e = tid; e < 32 * kC4Chunk; e += blockDim.x) {
        const int k = e / 32, q = e - k * 32;
        As[q * kC4LDA + k] = (k < kn && q < R3) ? __ldg(A3 + (size_t)sj3[k] * R3 + q) : 0.0;
      }
      const long long rowb = (long long)b * I3;
      for (int e = tid; e < kC4Chunk * kC4Tile; e += blockDim.x) {
        const int k = e / kC4Tile, i = e - k * kC4Tile;
        double v = 0.0;
        if (k < kn && i0 + i < I1)
          v = sw2[k] * (double)__ldg(X + (long long)(i0 + i) * slab + rowb + sj3[k]);
        Bs[k * kC4LDB + i] = v;
      }
      __syncthreads();
      if (mma_warp) {
        const int kk = (kn + 3) & ~3;
        for (int ks = 0; ks < kk; ks += 4) {
          const double a = As[(mt * 8 + g) * kC4LDA + ks + t];
          const double bv = Bs[(ks + t) * kC4LDB + nt * 8 + g];
          dmma_8x8x4(c0, c1, a, bv);
        }
      }
    }
    // fold D (this warp: q = 8 mt + g, i = 8 nt + 2t + e) into the tile with a2(b)
    __syncthreads();
    if (mma_warp) {
      const int q = mt * 8 + g;
      if (q < R3) {
        const int ic = nt * 8 + 2 * t;
        for (int p = 0; p < R2; ++p) {
          const double ap = a2s[p];
          double* row = rt + (size_t)(p * R3 + q) * kC4LDR + ic;
          row[0] = fma(ap, c0, row[0]);
          row[1] = fma(ap, c1, row[1]);
        }
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < W * kC4Tile; e += blockDim.x) {
    const int r = e / kC4Tile, i = e - r * kC4Tile;
    if (i0 + i < I1) rhs[(size_t)r * I1 + i0 + i] = rt[r * kC4LDR + i];
  }
}

}  // namespace

size_t c4_fiber_work_bytes(unsigned long long s, int I2) {
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs<unsigned long long, unsigned>(
      nullptr, cub_bytes, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
      (const unsigned*)nullptr, (unsigned*)nullptr, (int)s);
  return (size_t)s * (8 + 8 + 4 + 4 + 4 + 8) + (size_t)I2 * 8 + cub_bytes + 4096;
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
  const int W = R2 * R3;
  const size_t smem =
      ((size_t)W * kC4LDR + 32 * kC4LDA + kC4Chunk * kC4LDB + 32 + 2 * kC4Chunk) * sizeof(double);
  if (smem > 227 * 1024) throw Error(4, "c4_fiber_rhs: R2 R3 too large for the shared tile");
  static bool attr = false;
  if (!attr) {
    RTB_CUDA(cudaFuncSetAttribute(k_c4_fiber_rhs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    attr = true;
  }
  k_c4_fiber_rhs<<<ceil_div(I1, kC4Tile), 512, smem, st>>>(x, I1, I2, I3, A2, R2, A3, R3, j3s,
                                                             w2s, start, counts, rhs);
  RTB_LAUNCH_CHECK();
}

}  // namespace rtb
