// k_gram.cu -- sketched normal equations of the augmented Kronecker design.
//
// The reference streams every sampled row r_t = a_1(i_1) (x) ... (x) a_N(i_N)
// and rank-1-updates the d x d upper triangle (ref sketch_ridge.cpp:105-128):
// s_data * d^2 / 2 multiply-adds (C2: 8.4e11). The Gram of Kronecker rows has
// far fewer distinct entries:
//
//   G[(p_n),(q_n)] = sum_t w_t^2 prod_n a_n(i_n)[p_n] a_n(i_n)[q_n]
//
// depends only on the unordered pairs u_n = {p_n, q_n} (vech index, m_n =
// R_n(R_n+1)/2 values per mode): prod m_n distinct entries (C2: 136^3 = 2.5M vs
// 8.4M), and it factors through a bucketing of the draws by i_1:
//   (A) stable radix sort of the data draws by i_1 (CUB),
//   (B) k_vech_bucket: per bucket, H_b[Urow, Ucol] = sum_t w_t^2 v_row(t) v_col(t)^T
//       with v = products of vech(a_n a_n^T) over the modes >= 2 split into a
//       row group and a column group -- a GEMM with generated operands on the
//       FP64 tensor cores (DMMA.8x8x4), 48x48 tiles (136 = 3 x 48 - 8),
//   (C) k_vech_contract: S[u_1, U] = sum_b vech(a_1 a_1^T)(i_1(b))[u_1] H_b[U],
//       a DMMA GEMM with K = #buckets,
//   (D) k_vech_expand: scatter S into the full d x d Gram, plus the augmented
//       rows' diagonal (w^2 sqrt(l)) sqrt(l) per draw,
//   (E) k_bucket_h + k_rhs: rhs = sum_b a_1(b) (x) h_b, h_b = sum w^2 x_t z_t.
// C2 (d = 4096, s_data ~ 1e5, 512 buckets): (B) 1.85e9 + (C) 1.3e9 MACs.
// Summation order differs from the reference, so entries agree to rounding
// (parity ladder rung 3 in SURVEY.md 8(c)), not bitwise.
#include "common.cuh"
#include "kernels.h"

#include <cub/cub.cuh>

#include <cmath>

namespace rtb {

namespace {
constexpr int TB = 48;          // phase B/C output tile (6 x 8 rows)
constexpr int TNC = 64;         // phase C output tile columns
constexpr int KC = 32;          // samples (or buckets) per K chunk
constexpr int LDB = TB + 4;     // padded smem rows (phase B operands)
constexpr int LDC = TNC + 4;    // padded smem rows (phase C H chunk)
constexpr int kTh = 192;        // 6 warps, one 8-row m-tile each
constexpr int kMaxRow = 256;    // max concatenated factor-row length (modes >= 2)

// Vech/split description shared by the kernels.
struct VechSpec {
  int N;
  int R[kMaxOrder];
  int m[kMaxOrder];      // R(R+1)/2
  int msplit;            // row group = modes 1..msplit, column group = msplit+1..N-1
  long long Mrow, Ncol;  // product of m over the row / column group (1 if empty)
  long long Hsz;         // Mrow * Ncol
  int roff[kMaxOrder];   // offset of mode n's factor row in the staged concatenation
  int rowlen;            // sum_{n>=1} R_n
};

VechSpec make_vech(const GramSpec& g) {
  VechSpec v{};
  v.N = g.order;
  int o = 0;
  for (int n = 0; n < g.order; ++n) {
    v.R[n] = g.ranks[n];
    v.m[n] = g.ranks[n] * (g.ranks[n] + 1) / 2;
    if (n >= 1) {
      v.roff[n] = o;
      o += g.ranks[n];
    }
  }
  v.rowlen = o > 0 ? o : 1;
  // split modes 1..N-1 so that Mrow and Ncol are as balanced as possible
  v.msplit = g.order >= 2 ? 1 : 0;
  double best = 1e300;
  for (int ms = 1; ms <= g.order - 1; ++ms) {
    double a = 1, b = 1;
    for (int n = 1; n <= ms; ++n) a *= v.m[n];
    for (int n = ms + 1; n < g.order; ++n) b *= v.m[n];
    const double score = std::fabs(std::log(a / b));
    if (score < best) {
      best = score;
      v.msplit = ms;
    }
  }
  v.Mrow = 1;
  v.Ncol = 1;
  for (int n = 1; n <= v.msplit && n < g.order; ++n) v.Mrow *= v.m[n];
  for (int n = v.msplit + 1; n < g.order; ++n) v.Ncol *= v.m[n];
  v.Hsz = v.Mrow * v.Ncol;
  return v;
}

struct GramLayout {
  unsigned* keys;
  unsigned* vals;
  unsigned* keys_sorted;
  unsigned* vals_sorted;
  int* counts;    // [I1]
  int* bstart;    // [I1] compacted bucket start in sorted order
  int* blen;      // [I1]
  int* bi1;       // [I1] i1 of compacted bucket
  int* nbuckets;  // [1]
  int* aug_count; // [d]
  double* H;      // [I1][Hsz]
  double* h;      // [I1][d']
  double* S;      // [m_1][Hsz]
  void* cub_tmp;
  size_t cub_bytes;
};

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
  const VechSpec v = make_vech(spec);
  const int I1 = spec.rows[0];
  size_t total = 0;
  auto t = [&](size_t b) {
    take(total, b);
    total += (b + 255) & ~size_t(255);
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
  t((size_t)I1 * v.Hsz * 8);
  t((size_t)I1 * spec.dprime * 8);
  t((size_t)v.m[0] * v.Hsz * 8);
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

}  // namespace

size_t gram_work_bytes(const GramSpec& spec) {
  return carve(spec, [](size_t, size_t) {});
}

const int* gram_aug_counts(const GramSpec& spec, void* work) {
  return layout(spec, work).aug_count;
}

double gram_aug_term(const GramSpec& spec) {
  // augmented rows: each adds (w^2 sqrt(lambda)) sqrt(lambda) to its diagonal,
  // w = sqrt((1/s) / (0.5/d)) (ref sketch_ridge.cpp:88, 18-36, 115-120)
  const double inv_s = 1.0 / (double)spec.s;
  const double prob = (1.0 - 0.5) / (double)spec.d;
  const double wa = std::sqrt(inv_s / prob);
  const double rl = std::sqrt(spec.lambda);
  return (wa * wa * rl) * rl;
}

long long gram_block_elems(const GramSpec& spec) {
  const VechSpec v = make_vech(spec);
  long long n = (long long)v.R[v.N - 1] * v.R[v.N - 1];
  for (int k = 0; k < v.N - 1; ++k) n *= v.m[k];
  return n;
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

// decode a group index (modes lo..hi, last fastest) into 2 offsets per mode
__device__ __forceinline__ void decode_group(const VechSpec& v, long long u, int lo, int hi,
                                             short* out /* 2*(hi-lo+1) */) {
  for (int n = hi; n >= lo; --n) {
    const int un = (int)(u % v.m[n]);
    u /= v.m[n];
    int a, b;
    pair_of(un, v.R[n], a, b);
    out[2 * (n - lo)] = (short)(v.roff[n] + a);
    out[2 * (n - lo) + 1] = (short)(v.roff[n] + b);
  }
}

// (B) per bucket b and 48x48 tile of H_b: H_b[r][c] = sum_t w_t^2 vrow_t[r] vcol_t[c].
// grid = (tiles_row * tiles_col, I1), block 192.
__global__ void __launch_bounds__(kTh) k_vech_bucket(GramSpec spec, VechSpec v,
                                                     const unsigned long long* __restrict__ idx,
                                                     const double* __restrict__ w,
                                                     const unsigned* __restrict__ order,
                                                     const int* __restrict__ bstart,
                                                     const int* __restrict__ blen,
                                                     const int* __restrict__ nbuckets,
                                                     double* __restrict__ H) {
  __shared__ __align__(16) double zr[KC][LDB];
  __shared__ __align__(16) double zc[KC][LDB];
  __shared__ double w2s[KC];
  __shared__ int modes[KC][kMaxOrder];
  __shared__ short rowoff[TB][2 * kMaxOrder];
  __shared__ short coloff[TB][2 * kMaxOrder];
  __shared__ unsigned char qmode[kMaxRow];
  extern __shared__ double frow_dyn[];  // [KC][rowlen]
  const int RL = v.rowlen;
  auto frow = [&](int k, int q) -> double& { return frow_dyn[k * RL + q]; };
  const int b = blockIdx.y;
  if (b >= *nbuckets) return;
  const int N = v.N;
  const int tiles_c = (int)((v.Ncol + TB - 1) / TB);
  const long long r0 = (long long)(blockIdx.x / tiles_c) * TB;
  const long long c0 = (long long)(blockIdx.x % tiles_c) * TB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int nr = v.msplit, nc = N - 1 - v.msplit;  // modes in each group
  for (int e = tid; e < TB; e += kTh) {
    if (r0 + e < v.Mrow && nr > 0) decode_group(v, r0 + e, 1, v.msplit, rowoff[e]);
    if (c0 + e < v.Ncol && nc > 0) decode_group(v, c0 + e, v.msplit + 1, N - 1, coloff[e]);
  }
  for (int q = tid; q < v.rowlen; q += kTh) {
    int n = 1;
    while (n + 1 < N && q >= v.roff[n + 1]) ++n;
    qmode[q] = (unsigned char)n;
  }
  const int start = bstart[b], len = blen[b];
  double acc[6][2];
#pragma unroll
  for (int nt = 0; nt < 6; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  for (int k0 = 0; k0 < len; k0 += KC) {
    __syncthreads();
    if (tid < KC) {
      const int k = k0 + tid;
      if (k < len) {
        const unsigned tt = order[start + k];
        unsigned long long flat = idx[tt];
        for (int n = N - 1; n >= 0; --n) {
          modes[tid][n] = (int)(flat % (unsigned long long)spec.rows[n]);
          flat /= (unsigned long long)spec.rows[n];
        }
        const double wt = w[tt];
        w2s[tid] = wt * wt;
      } else {
        w2s[tid] = 0.0;
        for (int n = 0; n < N; ++n) modes[tid][n] = 0;
      }
    }
    __syncthreads();
    if (N > 1) {
      for (int e = tid; e < KC * v.rowlen; e += kTh) {
        const int k = e / v.rowlen, q = e - k * v.rowlen;
        const int n = qmode[q];
        frow(k, q) = spec.factors[n][(size_t)modes[k][n] * v.R[n] + (q - v.roff[n])];
      }
    }
    __syncthreads();
    for (int e = tid; e < 2 * KC * TB; e += kTh) {
      const int which = e / (KC * TB);
      const int rem = e - which * (KC * TB);
      const int k = rem / TB, c = rem - k * TB;
      double z = 0.0;
      if (which == 0) {
        if (r0 + c < v.Mrow) {
          z = w2s[k];
          for (int j = 0; j < nr; ++j) z *= frow(k, rowoff[c][2 * j]) * frow(k, rowoff[c][2 * j + 1]);
        }
        zr[k][c] = z;
      } else {
        if (c0 + c < v.Ncol) {
          z = 1.0;
          for (int j = 0; j < nc; ++j) z *= frow(k, coloff[c][2 * j]) * frow(k, coloff[c][2 * j + 1]);
        }
        zc[k][c] = z;
      }
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      const double af = zr[ks * 4 + t4][warp * 8 + g];
#pragma unroll
      for (int nt = 0; nt < 6; ++nt)
        dmma_8x8x4(acc[nt][0], acc[nt][1], af, zc[ks * 4 + t4][nt * 8 + g]);
    }
  }
  double* Hb = H + (size_t)b * v.Hsz;
  const long long r = r0 + warp * 8 + g;
  if (r < v.Mrow) {
#pragma unroll
    for (int nt = 0; nt < 6; ++nt) {
      const long long c = c0 + nt * 8 + 2 * t4;
      if (c < v.Ncol) Hb[r * v.Ncol + c] = acc[nt][0];
      if (c + 1 < v.Ncol) Hb[r * v.Ncol + c + 1] = acc[nt][1];
    }
  }
}

// h_b[p'] = sum_{t in b} w_t^2 x_t prod_{n>=1} a_n(i_n)[p_n]  (rhs ingredients)
// grid = I1, block 256.
__global__ void __launch_bounds__(256) k_bucket_h(GramSpec spec, const double* __restrict__ x,
                                                  const unsigned long long* __restrict__ idx,
                                                  const double* __restrict__ w,
                                                  const unsigned* __restrict__ order,
                                                  const int* __restrict__ bstart,
                                                  const int* __restrict__ blen,
                                                  const int* __restrict__ nbuckets,
                                                  double* __restrict__ h) {
  __shared__ double wx[KC];
  __shared__ int modes[KC][kMaxOrder];
  const int b = blockIdx.x;
  if (b >= *nbuckets) return;
  const int N = spec.order, dp = spec.dprime;
  const int start = bstart[b], len = blen[b];
  for (int p0 = 0; p0 < dp; p0 += 256) {
    const int p = p0 + threadIdx.x;
    // mode offsets of p' (last fastest)
    int pn[kMaxOrder];
    {
      int rem = p < dp ? p : 0;
      for (int n = N - 1; n >= 1; --n) {
        pn[n] = rem % spec.ranks[n];
        rem /= spec.ranks[n];
      }
    }
    double acc = 0.0;
    for (int k0 = 0; k0 < len; k0 += KC) {
      __syncthreads();
      if (threadIdx.x < KC) {
        const int k = k0 + threadIdx.x;
        if (k < len) {
          const unsigned tt = order[start + k];
          unsigned long long flat = idx[tt];
          const double xv = x[flat];
          for (int n = N - 1; n >= 0; --n) {
            modes[threadIdx.x][n] = (int)(flat % (unsigned long long)spec.rows[n]);
            flat /= (unsigned long long)spec.rows[n];
          }
          const double wt = w[tt];
          wx[threadIdx.x] = wt * wt * xv;
        } else {
          wx[threadIdx.x] = 0.0;
          for (int n = 0; n < N; ++n) modes[threadIdx.x][n] = 0;
        }
      }
      __syncthreads();
      if (p < dp) {
        const int kmax = min(KC, len - k0);
        for (int k = 0; k < kmax; ++k) {
          double z = wx[k];
          for (int n = 1; n < N; ++n)
            z *= spec.factors[n][(size_t)modes[k][n] * spec.ranks[n] + pn[n]];
          acc += z;
        }
      }
    }
    if (p < dp) h[(size_t)b * dp + p] = acc;
  }
}

// (C) S[u0, U] = sum_b vech(a0 a0^T)(i0_b)[u0] H[b, U]: M = m_0, N = Hsz, K = buckets.
// grid = (ceil(Hsz/64), ceil(m0/48)), block 192: warp w -> m-tile w, 8 n-tiles.
__global__ void __launch_bounds__(kTh) k_vech_contract(GramSpec spec, VechSpec v,
                                                       const double* __restrict__ H,
                                                       const int* __restrict__ bi1,
                                                       const int* __restrict__ nbuckets,
                                                       double* __restrict__ S) {
  __shared__ __align__(16) double vs[KC][LDB];
  __shared__ __align__(16) double hs[2][KC][LDC];
  __shared__ short pq[TB][2];
  const int R0 = v.R[0], m0 = v.m[0];
  const int nb = *nbuckets;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const long long n0 = (long long)blockIdx.x * TNC;
  const int u00 = blockIdx.y * TB;
  if (tid < TB) {
    const int u = u00 + tid;
    int a = -1, bb = -1;
    if (u < m0) pair_of(u, R0, a, bb);
    pq[tid][0] = (short)a;
    pq[tid][1] = (short)bb;
  }
  const double* A0 = spec.factors[0];
  auto load_h = [&](int kc, int stage) {
    for (int e = tid; e < KC * (TNC / 2); e += kTh) {
      const int k = e / (TNC / 2), c = (e % (TNC / 2)) * 2;
      const bool ok = (kc + k < nb) && (n0 + c < v.Hsz);
      const double* src = ok ? H + (size_t)(kc + k) * v.Hsz + n0 + c : H;
      if ((v.Hsz & 1) == 0) {
        cp_async16(&hs[stage][k][c], src, ok);
      } else {
        hs[stage][k][c] = ok ? src[0] : 0.0;
        hs[stage][k][c + 1] = (ok && n0 + c + 1 < v.Hsz) ? src[1] : 0.0;
      }
    }
  };
  double acc[8][2];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  load_h(0, 0);
  cp_async_commit();
  for (int k0 = 0, it = 0; k0 < nb; k0 += KC, ++it) {
    const int cur = it & 1;
    __syncthreads();  // previous chunk's readers of vs / hs[cur^1] are done
    if (k0 + KC < nb) load_h(k0 + KC, cur ^ 1);
    cp_async_commit();
    for (int e = tid; e < KC * TB; e += kTh) {
      const int k = e / TB, c = e - (e / TB) * TB;
      double val = 0.0;
      if (k0 + k < nb && pq[c][0] >= 0) {
        const double* a = A0 + (size_t)bi1[k0 + k] * R0;
        val = a[pq[c][0]] * a[pq[c][1]];
      }
      vs[k][c] = val;
    }
    cp_async_wait<1>();
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      const double af = vs[ks * 4 + t4][warp * 8 + g];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
        dmma_8x8x4(acc[nt][0], acc[nt][1], af, hs[cur][ks * 4 + t4][nt * 8 + g]);
    }
  }
  cp_async_wait<0>();
  const int u = u00 + warp * 8 + g;
  if (u < m0) {
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const long long c = n0 + nt * 8 + 2 * t4;
      if (c < v.Hsz) S[(size_t)u * v.Hsz + c] = acc[nt][0];
      if (c + 1 < v.Hsz) S[(size_t)u * v.Hsz + c + 1] = acc[nt][1];
    }
  }
}

// (D) full Gram from S plus the augmented diagonal.
__global__ void k_vech_expand(GramSpec spec, VechSpec v, const double* __restrict__ S,
                              const int* __restrict__ aug_count, double aug_term,
                              double* __restrict__ G) {
  const int d = spec.d, N = v.N;
  const long long total = (long long)d * d;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / d), j = (int)(e % d);
    int un[kMaxOrder];
    for (int n = N - 1; n >= 0; --n) {
      const int R = v.R[n];
      const int pi = i % R, qj = j % R;
      i /= R;
      j /= R;
      un[n] = upper_pair(min(pi, qj), max(pi, qj), R);
    }
    long long ur = 0, uc = 0;
    for (int n = 1; n <= v.msplit && n < N; ++n) ur = ur * v.m[n] + un[n];
    for (int n = v.msplit + 1; n < N; ++n) uc = uc * v.m[n] + un[n];
    double val = S[(size_t)un[0] * v.Hsz + ur * v.Ncol + uc];
    const int ii = (int)(e / d);
    if (ii == (int)(e % d) && aug_count[ii] > 0) val += (double)aug_count[ii] * aug_term;
    G[e] = val;
  }
}

// (D') the Gram in "last-mode blocks": B[u_1..u_{N-1}][r][c] = G entry whose
// first N-1 modes have vech pairs u_n and whose last-mode indices are (r, c).
// prod_{n<N} m_n blocks of R_N x R_N (C2: 136^2 x 16^2 doubles = 38 MB, vs
// 134 MB for the full Gram); consumed by the CG matvec (k_pcg.cu).
__global__ void k_vech_blocks(GramSpec spec, VechSpec v, const double* __restrict__ S,
                              double* __restrict__ B) {
  // one CTA per block (u_1..u_{N-1}); threads over the R_N x R_N entries
  const int N = v.N, RL = v.R[N - 1];
  int un[kMaxOrder];
  {
    unsigned t = blockIdx.x;
    for (int n = N - 2; n >= 0; --n) {
      un[n] = (int)(t % (unsigned)v.m[n]);
      t /= (unsigned)v.m[n];
    }
  }
  long long ur = 0, ucb = 0;
  for (int n = 1; n <= v.msplit && n < N - 1; ++n) ur = ur * v.m[n] + un[n];
  // the last mode is in the column group unless the split put it in the row group
  const bool last_in_row = v.msplit >= N - 1;
  for (int n = v.msplit + 1; n < N - 1; ++n) ucb = ucb * v.m[n] + un[n];
  const double* Su = S + (size_t)un[0] * v.Hsz;
  double* Bb = B + (size_t)blockIdx.x * RL * RL;
  for (int e = threadIdx.x; e < RL * RL; e += blockDim.x) {
    const int r = e / RL, c = e - r * RL;
    const int ul = upper_pair(min(r, c), max(r, c), RL);
    long long idx;
    if (last_in_row) idx = (ur * v.m[N - 1] + ul) * v.Ncol;
    else idx = ur * v.Ncol + ucb * v.m[N - 1] + ul;
    Bb[e] = __ldg(Su + idx);
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
  const VechSpec v = make_vech(spec);
  if (v.rowlen > kMaxRow) throw Error(4, "sketch_normal_eq: sum of ranks beyond mode 1 > 256");
  GramLayout l = layout(spec, work);
  const int I1 = spec.rows[0];
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
  const long long tiles_r = (v.Mrow + TB - 1) / TB, tiles_c = (v.Ncol + TB - 1) / TB;
  k_vech_bucket<<<dim3((unsigned)(tiles_r * tiles_c), I1), kTh,
                  (size_t)KC * v.rowlen * sizeof(double), st>>>(
      spec, v, idx, w, l.vals_sorted, l.bstart, l.blen, l.nbuckets, l.H);
  RTB_LAUNCH_CHECK();
  k_bucket_h<<<I1, 256, 0, st>>>(spec, x, idx, w, l.vals_sorted, l.bstart, l.blen, l.nbuckets,
                                 l.h);
  RTB_LAUNCH_CHECK();
  k_vech_contract<<<dim3((unsigned)((v.Hsz + TNC - 1) / TNC), (unsigned)ceil_div(v.m[0], TB)),
                    kTh, 0, st>>>(spec, v, l.H, l.bi1, l.nbuckets, l.S);
  RTB_LAUNCH_CHECK();
  // augmented rows: each adds (w^2 sqrt(lambda)) sqrt(lambda) to its diagonal,
  // w = sqrt((1/s) / (0.5/d)) (ref sketch_ridge.cpp:88, 18-36, 115-120)
  const double aug_term = gram_aug_term(spec);
  if (gram) {
    k_vech_expand<<<kNumSMs * 8, 256, 0, st>>>(spec, v, l.S, l.aug_count, aug_term, gram);
    RTB_LAUNCH_CHECK();
  }
  k_rhs<<<dim3(ceil_div(spec.dprime, 64), spec.ranks[0]), 256, 0, st>>>(spec, l.h, l.bi1,
                                                                        l.nbuckets, rhs);
  RTB_LAUNCH_CHECK();
}

void gram_expand_full(const GramSpec& spec, void* work, double* gram, cudaStream_t st) {
  const VechSpec v = make_vech(spec);
  GramLayout l = layout(spec, work);
  k_vech_expand<<<kNumSMs * 8, 256, 0, st>>>(spec, v, l.S, l.aug_count, gram_aug_term(spec), gram);
  RTB_LAUNCH_CHECK();
}

void gram_expand_blocks(const GramSpec& spec, void* work, double* blocks, cudaStream_t st) {
  const VechSpec v = make_vech(spec);
  GramLayout l = layout(spec, work);
  const long long nblk = gram_block_elems(spec) / ((long long)v.R[v.N - 1] * v.R[v.N - 1]);
  if (nblk > 0x7fffffffLL) throw Error(4, "gram_expand_blocks: too many blocks");
  k_vech_blocks<<<(unsigned)nblk, 256, 0, st>>>(spec, v, l.S, blocks);
  RTB_LAUNCH_CHECK();
}

}  // namespace rtb
