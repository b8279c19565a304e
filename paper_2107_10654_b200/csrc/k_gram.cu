// k_gram.cu -- sketched normal equations of the augmented Kronecker design.
//
// The reference streams every sampled row r_t = a1(i1) (x) a2(i2) (x) ... and
// rank-1-updates the d x d upper triangle (ref sketch_ridge.cpp:105-128):
// s_data * d^2 / 2 multiply-adds (C2: 8.4e11). We use the Kronecker structure:
//
//   G = sum_t w_t^2 r_t r_t^T
//     = sum_{i1} (a1(i1) a1(i1)^T) (x) H_{i1},   H_{i1} = sum_{t: i1(t)=i1} w_t^2 z_t z_t^T
//
// with z_t = a2(i2) (x) ... (x) aN(iN) of width d' = d / R1. So
//   (A) bucket the data draws by i1 (stable radix sort of (i1, t)),
//   (B) k_bucket_syrk: per nonempty bucket, H_{i1} (d' x d', upper 64x64 tiles)
//       plus h_{i1} = sum w^2 x_t z_t, FP64 tensor cores (DMMA.8x8x4),
//   (C) k_bucket_contract: S[(p1<=q1), e] = sum_{i1} a1(i1)_p1 a1(i1)_q1 H_{i1}[e],
//       a (R1(R1+1)/2) x (#H entries) x (#buckets) DMMA GEMM,
//   (D) k_expand_gram: scatter S into the full d x d Gram and add the
//       augmented rows' diagonal sum_{aug draws of j} (w^2 sqrt(l)) sqrt(l),
//   (E) k_rhs: rhs = sum_{i1} a1(i1) (x) h_{i1}.
// C2 (d=4096, R1=16, s_data~1e5, 512 buckets): (B) 3.3e9 + (C) 2.3e9 MACs
// instead of 8.4e11. Summation order differs from the reference, so entries
// agree to rounding (parity ladder rung 3 in SURVEY.md 8(c)), not bitwise.
#include "common.cuh"
#include "kernels.h"

#include <cub/cub.cuh>

namespace rtb {

namespace {
constexpr int TS = 64;        // H / S tile edge
constexpr int KC = 32;        // samples (or buckets) per K chunk
constexpr int LDS = TS + 4;   // padded smem row

struct GramLayout {
  unsigned* keys;
  unsigned* vals;
  unsigned* keys_sorted;
  unsigned* vals_sorted;
  int* counts;         // [I1]
  int* bstart;         // [I1] compacted bucket start in sorted order
  int* blen;           // [I1]
  int* bi1;            // [I1] i1 of compacted bucket
  int* nbuckets;       // [1]
  int* aug_count;      // [d]
  double* H;           // [I1][ntp][TS*TS]
  double* h;           // [I1][d']
  double* S;           // [npair1][ntp*TS*TS]
  void* cub_tmp;
  size_t cub_bytes;
};

__host__ __device__ inline int tiles_of(int dprime) { return (dprime + TS - 1) / TS; }
int tile_pairs(int dprime) {
  const int T = tiles_of(dprime);
  return T * (T + 1) / 2;
}
int key_bits(int I1) {
  int b = 1;
  while ((1 << b) <= I1) ++b;
  return b;
}

size_t cub_sort_bytes(unsigned long long s, int bits) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (unsigned*)nullptr, (unsigned*)nullptr,
                                  (unsigned*)nullptr, (unsigned*)nullptr, (int)s, 0, bits);
  return bytes;
}

template <typename F>
size_t carve(const GramSpec& spec, F&& take) {
  const int I1 = spec.rows[0];
  const int R1 = spec.ranks[0];
  const int ntp = tile_pairs(spec.dprime);
  const int npair1 = R1 * (R1 + 1) / 2;
  size_t total = 0;
  auto t = [&](size_t b) {
    const size_t r = (b + 255) & ~size_t(255);
    take(total, b);
    total += r;
  };
  t(spec.s * 4);
  t(spec.s * 4);
  t(spec.s * 4);
  t(spec.s * 4);
  t((size_t)I1 * 4);
  t((size_t)I1 * 4);
  t((size_t)I1 * 4);
  t((size_t)I1 * 4);
  t(4);
  t((size_t)spec.d * 4);
  t((size_t)I1 * ntp * TS * TS * 8);
  t((size_t)I1 * spec.dprime * 8);
  t((size_t)npair1 * ntp * TS * TS * 8);
  t(cub_sort_bytes(spec.s, key_bits(I1)));
  return total;
}

GramLayout layout(const GramSpec& spec, void* base) {
  GramLayout l;
  char* p = static_cast<char*>(base);
  int k = 0;
  carve(spec, [&](size_t off, size_t bytes) {
    void* q = p + off;
    switch (k++) {
      case 0: l.keys = (unsigned*)q; break;
      case 1: l.vals = (unsigned*)q; break;
      case 2: l.keys_sorted = (unsigned*)q; break;
      case 3: l.vals_sorted = (unsigned*)q; break;
      case 4: l.counts = (int*)q; break;
      case 5: l.bstart = (int*)q; break;
      case 6: l.blen = (int*)q; break;
      case 7: l.bi1 = (int*)q; break;
      case 8: l.nbuckets = (int*)q; break;
      case 9: l.aug_count = (int*)q; break;
      case 10: l.H = (double*)q; break;
      case 11: l.h = (double*)q; break;
      case 12: l.S = (double*)q; break;
      case 13: l.cub_tmp = q; l.cub_bytes = bytes; break;
    }
  });
  return l;
}

// pair index of (a <= b) among n items, row-major upper triangle
__host__ __device__ __forceinline__ int upper_pair(int a, int b, int n) {
  return a * n - a * (a - 1) / 2 + (b - a);
}
}  // namespace

size_t gram_work_bytes(const GramSpec& spec) {
  return carve(spec, [](size_t, size_t) {});
}

// (A) keys, augmented-row histogram, data-draw count.
__global__ void k_sketch_keys(GramSpec spec, const unsigned long long* idx, unsigned* keys,
                              unsigned* vals, int* counts, int* aug_count,
                              unsigned long long* data_draws) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)spec.s) return;
  const unsigned long long v = idx[t];
  const int I1 = spec.rows[0];
  vals[t] = (unsigned)t;
  if (v < spec.total_rows) {
    const unsigned long long inner = spec.total_rows / (unsigned long long)I1;
    const unsigned i1 = (unsigned)(v / inner);
    keys[t] = i1;
    atomicAdd(&counts[i1], 1);
    atomicAdd(data_draws, 1ULL);
  } else {
    keys[t] = (unsigned)I1;
    atomicAdd(&aug_count[v - spec.total_rows], 1);
  }
}

// Compact nonempty buckets in i1 order; start offsets = exclusive prefix of counts.
__global__ void __launch_bounds__(1024) k_bucket_scan(int I1, const int* counts, int* bstart,
                                                      int* blen, int* bi1, int* nbuckets) {
  __shared__ int s_cnt[1024], s_nz[1024];
  const int tid = threadIdx.x;
  const int per = ceil_div(I1, 1024);
  const int a = tid * per, b = min(I1, a + per);
  int c = 0, nz = 0;
  for (int i = a; i < b; ++i) {
    c += counts[i];
    nz += counts[i] > 0;
  }
  s_cnt[tid] = c;
  s_nz[tid] = nz;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    const int vc = tid >= d ? s_cnt[tid - d] : 0;
    const int vn = tid >= d ? s_nz[tid - d] : 0;
    __syncthreads();
    s_cnt[tid] += vc;
    s_nz[tid] += vn;
    __syncthreads();
  }
  int off = tid ? s_cnt[tid - 1] : 0;
  int k = tid ? s_nz[tid - 1] : 0;
  for (int i = a; i < b; ++i) {
    if (counts[i] > 0) {
      bstart[k] = off;
      blen[k] = counts[i];
      bi1[k] = i;
      ++k;
    }
    off += counts[i];
  }
  if (tid == 1023) *nbuckets = s_nz[1023];
}

// (B) per-bucket SYRK tiles. grid = (tile pairs, buckets), block 256.
__global__ void __launch_bounds__(256) k_bucket_syrk(GramSpec spec, const double* __restrict__ x,
                                                     const unsigned long long* __restrict__ idx,
                                                     const double* __restrict__ w,
                                                     const unsigned* __restrict__ order,
                                                     const int* __restrict__ bstart,
                                                     const int* __restrict__ blen,
                                                     const int* __restrict__ nbuckets,
                                                     double* __restrict__ H, double* __restrict__ h) {
  __shared__ __align__(16) double zp[KC][LDS];
  __shared__ __align__(16) double zq[KC][LDS];
  __shared__ double xs[KC];
  __shared__ int modes[KC][kMaxOrder];
  const int b = blockIdx.y;
  if (b >= *nbuckets) return;
  const int T = tiles_of(spec.dprime);
  // tile pair -> (P, Q), P <= Q
  int P = 0, rem = blockIdx.x;
  while (rem >= T - P) {
    rem -= T - P;
    ++P;
  }
  const int Q = P + rem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int mbase = 16 * (warp >> 1), nbase = 32 * (warp & 1);
  const int start = bstart[b], len = blen[b];
  const int N = spec.order;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double hacc = 0.0;  // threads 0..63 of diagonal tiles

  for (int k0 = 0; k0 < len; k0 += KC) {
    __syncthreads();
    if (tid < KC) {
      const int k = k0 + tid;
      if (k < len) {
        const unsigned tt = order[start + k];
        unsigned long long flat = idx[tt];
        xs[tid] = x[flat];
        for (int n = N - 1; n >= 0; --n) {
          modes[tid][n] = (int)(flat % (unsigned long long)spec.rows[n]);
          flat /= (unsigned long long)spec.rows[n];
        }
        const double wt = w[tt];
        zp[tid][TS] = wt * wt;  // stash w^2 in the pad column
      } else {
        xs[tid] = 0.0;
        zp[tid][TS] = 0.0;
        for (int n = 0; n < N; ++n) modes[tid][n] = 0;
      }
    }
    __syncthreads();
    // z values: entry p' = (p_2..p_N), last fastest; product over modes >= 2
    for (int e = tid; e < 2 * KC * TS; e += 256) {
      const int which = e / (KC * TS);
      const int k = (e / TS) % KC, c = e % TS;
      const int p = (which == 0 ? P : Q) * TS + c;
      double z = 0.0;
      if (p < spec.dprime && k0 + k < len) {
        z = 1.0;
        int rem2 = p;
        for (int n = N - 1; n >= 1; --n) {
          const int R = spec.ranks[n];
          const int pn = rem2 % R;
          rem2 /= R;
          z *= spec.factors[n][(size_t)modes[k][n] * R + pn];
        }
      }
      if (which == 0) zp[k][c] = z * zp[k][TS];
      else zq[k][c] = z;
    }
    __syncthreads();
    if (P == Q && tid < TS) {
      for (int k = 0; k < KC; ++k) hacc += zp[k][tid] * xs[k];
    }
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      double af[2], bf[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) af[mt] = zp[ks * 4 + t4][mbase + mt * 8 + g];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = zq[ks * 4 + t4][nbase + nt * 8 + g];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
  }
  const int ntp = gridDim.x;
  double* Ht = H + ((size_t)b * ntp + blockIdx.x) * TS * TS;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int r = mbase + mt * 8 + g, c = nbase + nt * 8 + 2 * t4;
      *reinterpret_cast<double2*>(Ht + r * TS + c) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
    }
  if (P == Q && tid < TS && P * TS + tid < spec.dprime)
    h[(size_t)b * spec.dprime + P * TS + tid] = hacc;
}

// (C) S[m, n] = sum_b V1[b, m] H[b, n]; m = (p1 <= q1) pair, n over H entries.
// grid = (ceil(ncols / 64), ceil(npair1 / 64)), block 256.
__global__ void __launch_bounds__(256) k_bucket_contract(GramSpec spec,
                                                         const double* __restrict__ H,
                                                         const int* __restrict__ bi1,
                                                         const int* __restrict__ nbuckets,
                                                         long long ncols, double* __restrict__ S) {
  __shared__ __align__(16) double vs[KC][LDS];
  __shared__ __align__(16) double hs[KC][LDS];
  __shared__ int pq[TS][2];
  const int R1 = spec.ranks[0];
  const int npair1 = R1 * (R1 + 1) / 2;
  const int nb = *nbuckets;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int mbase = 16 * (warp >> 1), nbase = 32 * (warp & 1);
  const long long n0 = (long long)blockIdx.x * TS;
  const int m0 = blockIdx.y * TS;
  if (tid < TS) {
    int m = m0 + tid, p1 = 0;
    if (m < npair1) {
      while (m >= R1 - p1) {
        m -= R1 - p1;
        ++p1;
      }
      pq[tid][0] = p1;
      pq[tid][1] = p1 + m;
    } else {
      pq[tid][0] = pq[tid][1] = -1;
    }
  }
  const double* A1 = spec.factors[0];
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < nb; k0 += KC) {
    __syncthreads();
    for (int e = tid; e < KC * (TS / 2); e += 256) {
      const int k = e / (TS / 2), c = (e % (TS / 2)) * 2;
      const bool ok = (k0 + k < nb) && (n0 + c < ncols);
      const double* src = ok ? H + (size_t)(k0 + k) * ncols + n0 + c : H;
      cp_async16(&hs[k][c], src, ok);
    }
    cp_async_commit();
    for (int e = tid; e < KC * TS; e += 256) {
      const int k = e / TS, c = e % TS;
      double v = 0.0;
      if (k0 + k < nb && pq[c][0] >= 0) {
        const double* a = A1 + (size_t)bi1[k0 + k] * R1;
        v = a[pq[c][0]] * a[pq[c][1]];
      }
      vs[k][c] = v;
    }
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      double af[2], bf[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) af[mt] = vs[ks * 4 + t4][mbase + mt * 8 + g];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = hs[ks * 4 + t4][nbase + nt * 8 + g];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int m = m0 + mbase + mt * 8 + g;
      const long long n = n0 + nbase + nt * 8 + 2 * t4;
      if (m < npair1 && n < ncols)
        *reinterpret_cast<double2*>(S + (size_t)m * ncols + n) =
            make_double2(acc[mt][nt][0], acc[mt][nt][1]);
    }
}

// (D) full Gram from S plus the augmented diagonal.
__global__ void k_expand_gram(GramSpec spec, const double* __restrict__ S, long long ncols,
                              const int* __restrict__ aug_count, double aug_term,
                              double* __restrict__ G) {
  const int d = spec.d, dp = spec.dprime, R1 = spec.ranks[0];
  const int T = tiles_of(dp);
  const long long total = (long long)d * d;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / d), j = (int)(e % d);
    const int p1 = i / dp, pp = i % dp, q1 = j / dp, qp = j % dp;
    const int m = upper_pair(min(p1, q1), max(p1, q1), R1);
    const int a = min(pp, qp), bq = max(pp, qp);
    const int tp = upper_pair(a / TS, bq / TS, T);
    double v = S[(size_t)m * ncols + (size_t)tp * TS * TS + (a % TS) * TS + (bq % TS)];
    if (i == j && aug_count[i] > 0) v += (double)aug_count[i] * aug_term;
    G[e] = v;
  }
}

// (E) rhs[p1 * d' + p'] = sum_b A1[i1_b, p1] h[b, p'].
// grid = (ceil(d'/64), R1); 64 outputs x 4 bucket groups per block.
__global__ void __launch_bounds__(256) k_rhs(GramSpec spec, const double* __restrict__ h,
                                             const int* __restrict__ bi1,
                                             const int* __restrict__ nbuckets,
                                             double* __restrict__ rhs) {
  __shared__ double part[4][64];
  const int R1 = spec.ranks[0], dp = spec.dprime;
  const int p1 = blockIdx.y;
  const int c = threadIdx.x & 63, q = threadIdx.x >> 6;
  const int pp = blockIdx.x * 64 + c;
  const int nb = *nbuckets;
  double s = 0.0;
  if (pp < dp)
    for (int b = q; b < nb; b += 4)
      s += spec.factors[0][(size_t)bi1[b] * R1 + p1] * h[(size_t)b * dp + pp];
  part[q][c] = s;
  __syncthreads();
  if (q == 0 && pp < dp)
    rhs[(size_t)p1 * dp + pp] = (part[0][c] + part[1][c]) + (part[2][c] + part[3][c]);
}

void sketch_normal_eq(const GramSpec& spec, const double* x, const unsigned long long* idx,
                      const double* w, void* work, size_t work_bytes, double* gram, double* rhs,
                      unsigned long long* data_draws_dev, cudaStream_t st) {
  if (work_bytes < gram_work_bytes(spec)) throw Error(4, "sketch_normal_eq: workspace too small");
  GramLayout l = layout(spec, work);
  const int I1 = spec.rows[0];
  const int ntp = tile_pairs(spec.dprime);
  const int R1 = spec.ranks[0];
  const int npair1 = R1 * (R1 + 1) / 2;
  const long long ncols = (long long)ntp * TS * TS;
  RTB_CUDA(cudaMemsetAsync(l.counts, 0, (size_t)I1 * 4, st));
  RTB_CUDA(cudaMemsetAsync(l.aug_count, 0, (size_t)spec.d * 4, st));
  RTB_CUDA(cudaMemsetAsync(data_draws_dev, 0, 8, st));
  const unsigned sb = (unsigned)ceil_div<unsigned long long>(spec.s, 256ULL);
  k_sketch_keys<<<sb, 256, 0, st>>>(spec, idx, l.keys, l.vals, l.counts, l.aug_count,
                                    data_draws_dev);
  RTB_LAUNCH_CHECK();
  size_t cb = l.cub_bytes;
  RTB_CUDA(cub::DeviceRadixSort::SortPairs(l.cub_tmp, cb, l.keys, l.keys_sorted, l.vals,
                                           l.vals_sorted, (int)spec.s, 0, key_bits(I1), st));
  k_bucket_scan<<<1, 1024, 0, st>>>(I1, l.counts, l.bstart, l.blen, l.bi1, l.nbuckets);
  RTB_LAUNCH_CHECK();
  // Every bucket slot up to I1 is launched; blocks beyond *nbuckets exit.
  dim3 g1(ntp, I1);
  k_bucket_syrk<<<g1, 256, 0, st>>>(spec, x, idx, w, l.vals_sorted, l.bstart, l.blen, l.nbuckets,
                                    l.H, l.h);
  RTB_LAUNCH_CHECK();
  dim3 g2((unsigned)ceil_div<long long>(ncols, TS), (unsigned)ceil_div(npair1, TS));
  k_bucket_contract<<<g2, 256, 0, st>>>(spec, l.H, l.bi1, l.nbuckets, ncols, l.S);
  RTB_LAUNCH_CHECK();
  // augmented rows: each adds (w^2 sqrt(lambda)) sqrt(lambda) to its diagonal,
  // w = sqrt((1/s) / (0.5/d)) (ref sketch_ridge.cpp:88, 18-36, 115-120)
  const double inv_s = 1.0 / (double)spec.s;
  const double prob = (1.0 - 0.5) / (double)spec.d;
  const double wa = std::sqrt(inv_s / prob);
  const double rl = std::sqrt(spec.lambda);
  const double aug_term = (wa * wa * rl) * rl;
  k_expand_gram<<<kNumSMs * 8, 256, 0, st>>>(spec, l.S, ncols, l.aug_count, aug_term, gram);
  RTB_LAUNCH_CHECK();
  k_rhs<<<dim3(ceil_div(spec.dprime, 64), R1), 256, 0, st>>>(spec, l.h, l.bi1, l.nbuckets, rhs);
  RTB_LAUNCH_CHECK();
}

}  // namespace rtb
