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
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <type_traits>

namespace rtb {

namespace {
constexpr int TB = 48;          // phase B/C output tile (6 x 8 rows)
constexpr int TNC = 64;         // phase C output tile columns
constexpr int KC = 32;          // samples (or buckets) per K chunk
#ifndef RTB_KCB
#define RTB_KCB 32
#define RTB_KCC 32
#endif
constexpr int KCB = RTB_KCB;     // k_vech_bucket2: draws per pipelined chunk
constexpr int KCC = RTB_KCC;     // k_vech_contract2: buckets per pipelined chunk
constexpr int LDB = TB + 4;     // padded smem rows (phase B operands)
constexpr int LDC = TNC + 4;    // padded smem rows (phase C H chunk)
constexpr int kTh = 192;        // 6 warps, one 8-row m-tile each
constexpr int kMaxRow = 256;    // max concatenated factor-row length (modes >= 2)
constexpr int kRhsSplit = 16;   // bucket groups of the two-level rhs reduction
constexpr int kBT = 18;         // whole-bucket kernel: up to 18 x 18 tiles of 8 x 8
constexpr int kBWarps = 18;     // ... 18 warps, warp w owns row tile w (second tile unused)
constexpr int LDZ = kBT * 8 + 4;
static_assert(kBWarps * 32 == 4 * kBT * 8, "generation maps 4 threads per column");

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
  double* dw2;    // [s] w^2 of the k-th data draw in bucket order
  double* dwx;    // [s] w^2 x
  int* dmode;     // [N][s] mode indices
  double* rhs_part;  // [kRhsSplit][d]
  double* drow;   // [s][rowlen] concatenated factor rows of modes >= 2, bucket order
  double* vt2;    // [I2][tab_width(m2)] vech Khatri-Rao table of A_2 (+ raw rows when R <= 16)
  double* vt3;    // [I3][tab_width(m3)]
  int* border;    // [I1] compacted buckets, longest first (k_bucket_order)
  int* bcounter;  // [1] next bucket of the persistent k_vech_bucket3
  double* vt1;    // [I1][160] mode-1 table per compacted bucket (k_vech_table1)
};

// vech table row length of mode n: 160 (136 vech padded to 144 + the raw row, k_vech_bucket5)
// for m_n <= 144; above that (R_n > 16, k_vech_bucket6) m_n rounded up to whole 144-wide tiles
int tab_width(int m) { return m <= 144 ? 160 : (m + 143) / 144 * 144; }

constexpr int kC3Ldt = 160, kC3Raw = 144;
constexpr int kC3Rows = 136;  // S rows per CTA (17 consumer warps x 8)
// Table geometry: m_1 <= 136 (C2): width 160, raw row at 144 (one staged window holds both).
// Larger m_1 (C5: 528): the Gram CTAs take row blocks of 136, each staging the 160-wide window
// at 136 rb; the raw row sits after all of them, at raw = 136 nrb + 24, in its own window.
struct C3Geom {
  int nrb, tw, raw;
};
C3Geom c3_geom(int m1) {
  C3Geom gm;
  gm.nrb = (m1 + kC3Rows - 1) / kC3Rows;
  if (gm.nrb <= 1) {
    gm.nrb = 1;
    gm.tw = kC3Ldt;
    gm.raw = kC3Raw;
  } else {
    gm.raw = gm.nrb * kC3Rows + 24;
    gm.tw = gm.raw + kC3Ldt;
  }
  return gm;
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
  t(spec.s * 8);                               // dw2: w^2 per sorted data draw
  t(spec.s * 8);                               // dwx: w^2 x per sorted data draw
  t(spec.s * 4 * (size_t)spec.order);          // dmode[n][k]
  t((size_t)kRhsSplit * spec.d * 8);           // rhs partials
  t(spec.s * (size_t)v.rowlen * 8);            // drow: factor rows (modes >= 2) per draw
  t((size_t)(spec.order >= 2 ? spec.rows[1] : 1) * tab_width(spec.order >= 2 ? v.m[1] : 1) * 8);  // vt2
  t((size_t)(spec.order >= 3 ? spec.rows[2] : 1) * tab_width(spec.order >= 3 ? v.m[2] : 1) * 8);  // vt3
  t((size_t)I1 * 4);                           // border
  t(16);                                       // bcounter
  t((size_t)I1 * c3_geom(v.m[0]).tw * 8);      // vt1 (k_vech_table1)
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
      case 14: l.dw2 = (double*)q; break;
      case 15: l.dwx = (double*)q; break;
      case 16: l.dmode = (int*)q; break;
      case 17: l.rhs_part = (double*)q; break;
      case 18: l.drow = (double*)q; break;
      case 19: l.vt2 = (double*)q; break;
      case 20: l.vt3 = (double*)q; break;
      case 21: l.border = (int*)q; break;
      case 22: l.bcounter = (int*)q; break;
      case 23: l.vt1 = (double*)q; break;
    }
  });
  return l;
}

GramSpec merged_spec(const GramSpec& s4) {
  GramSpec g{};
  g.order = 3;
  g.rows[0] = s4.rows[0] * s4.rows[1];
  g.rows[1] = s4.rows[2];
  g.rows[2] = s4.rows[3];
  g.ranks[0] = 1;
  g.ranks[1] = s4.ranks[2];
  g.ranks[2] = s4.ranks[3];
  g.factors[0] = nullptr;
  g.factors[1] = s4.factors[2];
  g.factors[2] = s4.factors[3];
  g.total_rows = s4.total_rows;
  g.d = s4.d;  // augmented draws index the order-4 d
  g.dprime = s4.ranks[2] * s4.ranks[3];
  g.lambda = s4.lambda;
  g.s = s4.s;
  // sharded along mode 1: the merged mode's rows (i1, i2) of this shard are contiguous
  g.i1_lo = s4.i1_hi > 0 ? s4.i1_lo * s4.rows[1] : 0;
  g.i1_hi = s4.i1_hi > 0 ? s4.i1_hi * s4.rows[1] : 0;
  return g;
}

bool merged4_ok(const GramSpec& spec) {
  if (spec.order != 4) return false;
  if ((long long)spec.rows[0] * spec.rows[1] > (1LL << 30)) return false;
  if (spec.ranks[2] > 16 || spec.ranks[3] > 16) return false;
  // worth it when the draws outnumber the (i1, i2) pairs
  return (double)spec.s > 2.0 * (double)spec.rows[0] * spec.rows[1];
}

struct M4Extra {
  double *Hd, *hd, *ka1, *ka2, *T, *Tr;
  void* w3;
  size_t w3_bytes, total;
};

M4Extra m4_extra(const GramSpec& s4, void* base) {
  const GramSpec g = merged_spec(s4);
  const VechSpec v3 = make_vech(g);
  M4Extra e{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t b) {
    void* r = p ? p + off : nullptr;
    off += (b + 255) & ~size_t(255);
    return r;
  };
  const long long P = (long long)g.rows[0];
  const int m1 = s4.ranks[0] * (s4.ranks[0] + 1) / 2, m2 = s4.ranks[1] * (s4.ranks[1] + 1) / 2;
  e.w3_bytes = gram_work_bytes(g);
  e.w3 = take(e.w3_bytes);
  e.Hd = (double*)take((size_t)P * v3.Hsz * 8);
  e.hd = (double*)take((size_t)P * g.dprime * 8);
  e.ka1 = (double*)take((size_t)s4.rows[0] * m1 * 8);
  e.ka2 = (double*)take((size_t)s4.rows[1] * m2 * 8);
  e.T = (double*)take((size_t)s4.rows[0] * m2 * v3.Hsz * 8);
  e.Tr = (double*)take((size_t)s4.rows[0] * s4.ranks[1] * g.dprime * 8);
  e.total = off;
  return e;
}

size_t m4_extra_bytes(const GramSpec& spec) { return m4_extra(spec, nullptr).total; }

}  // namespace

size_t gram_work_bytes(const GramSpec& spec) {
  return carve(spec, [](size_t, size_t) {}) + (merged4_ok(spec) ? m4_extra_bytes(spec) : 0);
}

double* gram_compact(const GramSpec& spec, void* work, size_t* count) {
  const VechSpec v = make_vech(spec);
  if (count) *count = (size_t)v.m[0] * v.Hsz;
  return layout(spec, work).S;
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
    if (spec.i1_hi > 0 && ((int)i1 < spec.i1_lo || (int)i1 >= spec.i1_hi)) {
      keys[t] = (unsigned)I1;  // another shard's draw: sorts with the augmented ones
      return;
    }
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

// (A') draw records in bucket order: one parallel gather of x and one decode of
// the flat index per data draw, so the bucket kernels stream contiguous arrays.
__global__ void k_gather_draws(GramSpec spec, const double* __restrict__ x,
                               const unsigned long long* __restrict__ idx,
                               const double* __restrict__ w, const unsigned* __restrict__ order,
                               const unsigned* __restrict__ keys_sorted, double* __restrict__ dw2,
                               double* __restrict__ dwx, int* __restrict__ dmode) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (long long)spec.s) return;
  if (keys_sorted[k] >= (unsigned)spec.rows[0]) return;  // augmented draws sort last
  const unsigned tt = order[k];
  unsigned long long flat = idx[tt];
  const double xv = __ldg(x + flat);
  for (int n = spec.order - 1; n >= 0; --n) {
    const unsigned long long rn = (unsigned long long)spec.rows[n];
    dmode[(size_t)n * spec.s + k] = (int)(flat % rn);
    flat /= rn;
  }
  const double wt = w[tt];
  const double w2 = wt * wt;
  dw2[k] = w2;
  dwx[k] = w2 * xv;
}

// drow[k][q] = a_n(i_n(k))[q - roff[n]] for modes n >= 2 (coalesced writes).
__global__ void k_gather_rows(GramSpec spec, VechSpec v, const unsigned* __restrict__ keys_sorted,
                              const int* __restrict__ dmode, double* __restrict__ drow) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int RL = v.rowlen;
  if (e >= (long long)spec.s * RL) return;
  const long long k = e / RL;
  const int q = (int)(e - k * RL);
  if (keys_sorted[k] >= (unsigned)spec.rows[0]) return;
  int n = 1;
  while (n + 1 < v.N && q >= v.roff[n + 1]) ++n;
  if (n >= v.N) return;
  const int in = dmode[(size_t)n * spec.s + k];
  drow[e] = __ldg(spec.factors[n] + (size_t)in * v.R[n] + (q - v.roff[n]));
}

// (B') one CTA per bucket computes the whole H_b (Mrow x Ncol <= 144 x 144) so
// the operand generation is done once per bucket and amortised over up to
// 18 x 18 DMMA tiles per K step. 9 warps; warp w owns row tiles w and w + 9; NTT
// column tiles are computed unconditionally (operands are zero-padded), so the
// DMMA stream has no branches. With HPT > 0 the same CTA also accumulates the
// rhs ingredient h_b[p'] = sum_t w_t^2 x_t prod_{n>=1} a_n(i_n)[p_n] from the
// staged factor rows (HPT outputs per thread).
// cp.async one chunk of draw records (KCB draws: factor rows, w^2, w^2 x) into buffer buf.
template <int HPT>
__device__ __forceinline__ void stage_bucket_chunk(const double* __restrict__ drow,
                                                   const double* __restrict__ dw2,
                                                   const double* __restrict__ dwx, double* frow,
                                                   double* w2s, double* wxs, int start, int len,
                                                   int k0, int buf, int RL, int RLp) {
  const int kn = min(KCB, len - k0);
  double* fr = frow + buf * KCB * RLp;
  for (int e = threadIdx.x; e < KCB * RL; e += blockDim.x) {
    const int k = e / RL, q = e - k * RL;
    const bool ok = k < kn;
    cp_async8(fr + k * RLp + q, ok ? drow + (size_t)(start + k0 + k) * RL + q : drow, ok);
  }
  if (threadIdx.x < KCB) {
    const bool ok = (int)threadIdx.x < kn;
    cp_async8(w2s + buf * KCB + threadIdx.x, ok ? dw2 + start + k0 + threadIdx.x : dw2, ok);
    if (HPT > 0) cp_async8(wxs + buf * KCB + threadIdx.x, ok ? dwx + start + k0 + threadIdx.x : dwx, ok);
  }
}

template <int NTT, int HPT, int NR, int NC>
__global__ void __launch_bounds__(kBWarps * 32, 1) k_vech_bucket2(
    GramSpec spec, VechSpec v, const double* __restrict__ dw2, const double* __restrict__ dwx,
    const double* __restrict__ drow, const int* __restrict__ bstart, const int* __restrict__ blen,
    const int* __restrict__ nbuckets, double* __restrict__ H, double* __restrict__ h) {
  extern __shared__ __align__(16) double smb[];
  const int RL = v.rowlen;
  const int RLp = (RL + 1) & ~1;
  // software pipeline, one barrier per chunk: while some warps still run the DMMAs of
  // chunk k, others already generate the operands of chunk k+1 into the other buffer
  // and the draw records of chunk k+2 land in the third frow buffer.
  double* zr = smb;                   // [2][KCB][LDZ]
  double* zc = zr + 2 * KCB * LDZ;     // [2][KCB][LDZ]
  double* frow = zc + 2 * KCB * LDZ;   // [3][KCB][RLp]
  double* w2s = frow + 3 * KCB * RLp;  // [3][KCB]
  double* wxs = w2s + 3 * KCB;         // [3][KCB]
  const int b = blockIdx.x;
  if (b >= *nbuckets) return;
  const int N = v.N;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int MT = (int)((v.Mrow + 7) / 8);
  // generation: thread -> fixed column c, rows k = k0r + 4 j (576 threads = 4 x 144)
  const int c = tid % (kBT * 8), k0r = tid / (kBT * 8);
  // (p, q) factor-row offsets of this thread's column in the row / column groups
  int ro[2 * (NR > 0 ? NR : 1)], co[2 * (NC > 0 ? NC : 1)];
  {
    long long u = c < v.Mrow ? c : 0;
#pragma unroll
    for (int j = NR - 1; j >= 0; --j) {  // row group = modes 1..NR (last fastest)
      const int n = 1 + j;
      const int un = (int)(u % v.m[n]);
      u /= v.m[n];
      int pa, pb;
      pair_of(un, v.R[n], pa, pb);
      ro[2 * j] = v.roff[n] + pa;
      ro[2 * j + 1] = v.roff[n] + pb;
    }
    u = c < v.Ncol ? c : 0;
#pragma unroll
    for (int j = NC - 1; j >= 0; --j) {  // column group = modes NR+1..NR+NC
      const int n = 1 + NR + j;
      const int un = (int)(u % v.m[n]);
      u /= v.m[n];
      int pa, pb;
      pair_of(un, v.R[n], pa, pb);
      co[2 * j] = v.roff[n] + pa;
      co[2 * j + 1] = v.roff[n] + pb;
    }
  }
  const bool rok = c < v.Mrow, cok = c < v.Ncol;
  // HPT == 1 (3-way, R_2, R_3 <= 16): the spare warp kBWarps-1 (row tiles <= 17)
  // accumulates h_b[p2][p3] = sum_t (w^2 x a_2)[p2] a_3[p3] with 4 DMMA tiles.
  const bool hwarp = HPT > 0 && warp == kBWarps - 1;
  double hacc[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
  const int start = bstart[b], len = blen[b];
  double acc[NTT][2];
#pragma unroll
  for (int j = 0; j < NTT; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int rt0 = warp;
  const int nch = (len + KCB - 1) / KCB;
  // generate chunk kk (its frow buffer kk % 3 has landed) into z buffer kk & 1
  auto generate = [&](int kk) {
    const int fb = kk % 3, zb = kk & 1;
    const double* fr = frow + fb * KCB * RLp;
    const double* w2c = w2s + fb * KCB;
    double* zrb = zr + zb * KCB * LDZ;
    double* zcb = zc + zb * KCB * LDZ;
#pragma unroll 4
    for (int j = 0; j < KCB / 4; ++j) {
      const int k = k0r + 4 * j;
      const double* f = fr + k * RLp;
      double zrv = 0.0, zcv = 0.0;
      if (rok) {
        zrv = w2c[k];
#pragma unroll
        for (int q = 0; q < NR; ++q) zrv *= f[ro[2 * q]] * f[ro[2 * q + 1]];
      }
      if (cok) {
        zcv = 1.0;
#pragma unroll
        for (int q = 0; q < NC; ++q) zcv *= f[co[2 * q]] * f[co[2 * q + 1]];
      }
      zrb[k * LDZ + c] = zrv;
      zcb[k * LDZ + c] = zcv;
    }
  };
  if (nch > 0) stage_bucket_chunk<HPT>(drow, dw2, dwx, frow, w2s, wxs, start, len, 0, 0, RL, RLp);
  cp_async_commit();
  if (nch > 1) stage_bucket_chunk<HPT>(drow, dw2, dwx, frow, w2s, wxs, start, len, KCB, 1, RL, RLp);
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();
  if (nch > 0) generate(0);
  __syncthreads();
  for (int kk = 0; kk < nch; ++kk) {
    // records of chunk kk+2 into frow buffer (kk+2) % 3 (last read by generate(kk-1))
    if (kk + 2 < nch)
      stage_bucket_chunk<HPT>(drow, dw2, dwx, frow, w2s, wxs, start, len, (kk + 2) * KCB,
                              (kk + 2) % 3, RL, RLp);
    cp_async_commit();
    const int zb = kk & 1;
    if (rt0 < MT) {
      const double* zrb = zr + zb * KCB * LDZ;
      const double* zcb = zc + zb * KCB * LDZ;
#pragma unroll
      for (int ks = 0; ks < KCB / 4; ++ks) {
        const double* zrk = zrb + (ks * 4 + t4) * LDZ;
        const double* zck = zcb + (ks * 4 + t4) * LDZ;
        const double a0 = zrk[rt0 * 8 + g];
#pragma unroll
        for (int nt = 0; nt < NTT; ++nt) dmma_8x8x4(acc[nt][0], acc[nt][1], a0, zck[nt * 8 + g]);
      }
    }
    if (hwarp) {
      const int fb = kk % 3;
      const double* fr = frow + fb * KCB * RLp;
      const double* wxc = wxs + fb * KCB;
      const int R2 = v.R[1], R3 = v.R[2], o2 = v.roff[1], o3 = v.roff[2];
#pragma unroll
      for (int ks = 0; ks < KCB / 4; ++ks) {
        const int k = ks * 4 + t4;
        const double* f = fr + k * RLp;
        const double wk = wxc[k];
        double af[2], bf[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          af[i] = (i * 8 + g < R2) ? wk * f[o2 + i * 8 + g] : 0.0;
          bf[i] = (i * 8 + g < R3) ? f[o3 + i * 8 + g] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma_8x8x4(hacc[i][j][0], hacc[i][j][1], af[i], bf[j]);
      }
    }
    if (kk + 1 < nch) {
      cp_async_wait<1>();   // chunk kk+1's records (this thread's copies) have landed
      __syncthreads();      // ... everyone's; and z buffer (kk+1)&1 is free (MMA kk-1 done)
      generate(kk + 1);
    }
    __syncthreads();        // z buffer (kk+1)&1 complete; MMA kk done before it is reused
  }
  cp_async_wait<0>();
  double* Hb = H + (size_t)b * v.Hsz;
  {
    const long long r = (long long)rt0 * 8 + g;
    if (rt0 < MT && r < v.Mrow) {
#pragma unroll
      for (int nt = 0; nt < NTT; ++nt) {
        const long long cc = (long long)nt * 8 + 2 * t4;
        if (cc < v.Ncol) Hb[r * v.Ncol + cc] = acc[nt][0];
        if (cc + 1 < v.Ncol) Hb[r * v.Ncol + cc + 1] = acc[nt][1];
      }
    }
  }
  if (hwarp) {
    const int R2 = v.R[1], R3 = v.R[2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int p2 = i * 8 + g, p3 = j * 8 + 2 * t4;
        if (p2 < R2 && p3 < R3) h[(size_t)b * spec.dprime + p2 * R3 + p3] = hacc[i][j][0];
        if (p2 < R2 && p3 + 1 < R3) h[(size_t)b * spec.dprime + p2 * R3 + p3 + 1] = hacc[i][j][1];
      }
  }
}

size_t vech_bucket2_smem(const VechSpec& v) {
  const size_t rlp = (size_t)((v.rowlen + 1) & ~1);
  return (size_t)(4 * KCB * LDZ + 3 * KCB * rlp + 6 * KCB) * 8 + 16;
}

// Buckets ranked longest first (ties by index): the persistent bucket kernel takes them in
// this order (longest-processing-time-first list scheduling over the SMs).
__global__ void __launch_bounds__(1024) k_bucket_order(const int* __restrict__ blen,
                                                       const int* __restrict__ nbuckets,
                                                       int* __restrict__ order, int* counter) {
  const int nb = *nbuckets;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const int lb = blen[b];
    int rank = 0;
    for (int j = 0; j < nb; ++j) {
      const int lj = blen[j];
      rank += (lj > lb) || (lj == lb && j < b);
    }
    order[rank] = b;
  }
  if (threadIdx.x == 0) *counter = 0;
}

// vech Khatri-Rao tables of the modes 2 and 3 (one per core update, L2-resident):
// vt[i][u] = A[i, p] A[i, q] for the vech pair u = (p <= q), zero up to column 144, then the
// raw row A[i, :] (the h_b operand), zero to ld: one bulk copy stages both per draw.
__global__ void k_vech_table(const double* __restrict__ A, int I, int R, int ld,
                             double* __restrict__ vt) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)I * ld) return;
  const long long i = e / ld;
  const int u = (int)(e - i * ld);
  double v = 0.0;
  if (u < R * (R + 1) / 2) {
    int pa, pb;
    pair_of(u, R, pa, pb);
    v = A[i * R + pa] * A[i * R + pb];
  } else if (u >= 144 && u < 144 + R) {
    v = A[i * R + (u - 144)];  // the raw factor row (h_b operand) after the padded vech part
  }
  vt[e] = v;
}

// (B'') 3-way H_b (+ h_b), persistent, two CTAs per SM. A work item is one half of a
// bucket's H_b (vech rows [72 h, 72 h + 72), all 144 padded columns); items are taken longest
// bucket first from an atomic counter (no partial last wave). The operands are NOT generated
// per draw: H_b = sum_t w_t^2 V2[i2_t]^T V3[i3_t] with V2, V3 the vech Khatri-Rao tables of
// A_2, A_3 (k_vech_table, L2-resident), so a chunk of 16 draws is a cp.async gather of table
// rows into a 3-stage ring (plus the raw factor rows for h_b) and the DMMA loop reads them
// directly, w^2 folded into the A fragment. 9 warps own 3 x 6 DMMA tiles each (0.5 fragment
// loads per DMMA); on the half-0 items warps 0-3 also accumulate one 8 x 8 tile each of
// h_b[p2][p3] = sum w^2 x a_2[p2] a_3[p3]. The K loop stops at the chunk's last draw
// (rounded to 4). A half's result does not depend on which CTA computes it.
// Warp-specialised: one producer warp runs ahead through this CTA's items (fetched from the
// atomic counter) and chunks, staging each chunk of kB5K draws into a kB5St-deep ring -- the
// draw scalars and zero padding by plain stores, the table rows (and raw factor rows for
// h_b) by TMA bulk copies completing on the stage's `full` mbarrier, the chunk's
// (bucket, position) in a metadata slot -- and 18 consumer warps (3 x 6 DMMA tiles each)
// wait on `full`, accumulate, write H_b after a bucket's last chunk and release the stage on
// its `empty` mbarrier. No CTA-wide barrier in the steady state.
constexpr int kB5Mma = 18;               // consumer warps
constexpr int kB5K = 24;                 // draws per stage
constexpr int kB5St = 3;                 // ring stages
constexpr int kB5Rows = 144;             // whole bucket per item
constexpr int kB5Halves = 1;
constexpr int kB5CtaPerSm = 1;
constexpr int kB5Threads = (kB5Mma + 1) * 32;
constexpr int kB5Tab = 160;              // table row: vech (136, padded to 144) + raw row (16)
constexpr int kB5Ld = kB5Tab + 4;        // staged row stride: conflict-free fragment loads
__global__ void __launch_bounds__(kB5Threads, kB5CtaPerSm) k_vech_bucket5(
    GramSpec spec, VechSpec v, const double* __restrict__ V2, const double* __restrict__ V3,
    const int* __restrict__ dmode, const double* __restrict__ dw2,
    const double* __restrict__ dwx, const int* __restrict__ bstart,
    const int* __restrict__ blen, const int* __restrict__ nbuckets,
    const int* __restrict__ order, int* counter, double* __restrict__ H, double* __restrict__ h) {
  extern __shared__ __align__(16) double smb[];
  double* zr = smb;                                  // [St][K][Ld] V2 rows (+ raw a_2 rows)
  double* zc = zr + kB5St * kB5K * kB5Ld;            // [St][K][Ld] V3 rows (+ raw a_3 rows)
  double* w2s = zc + kB5St * kB5K * kB5Ld;           // [St][K]
  double* wxs = w2s + kB5St * kB5K;                  // [St][K]
  __shared__ __align__(8) unsigned long long full[kB5St], empty[kB5St];
  __shared__ int meta[kB5St][4];  // bucket (-1: no more work), half, draws in chunk, last chunk
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int R2 = v.R[1], R3 = v.R[2];
  if (tid == 0) {
    for (int i = 0; i < kB5St; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kB5Mma);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kB5Mma) {
    // ---------------- producer ----------------
    const int nb = *nbuckets;
    const long long S = (long long)spec.s;
    unsigned q = 0;  // chunks staged so far
    auto next_stage = [&]() {
      const int sb = (int)(q % kB5St);
      if (q >= kB5St) mbar_wait(&empty[sb], ((q / kB5St) - 1) & 1);
      return sb;
    };
    // the next item (atomic ticket -> bucket -> its range) is fetched one item ahead, so the
    // chain of dependent global loads overlaps the staging of the current item's chunks
    auto fetch = [&](int& it, int& fb, int& fstart, int& flen) {
      int t = 0;
      if (lane == 0) t = atomicAdd(counter, 1);
      it = __shfl_sync(0xffffffffu, t, 0);
      fb = -1;
      fstart = flen = 0;
      if (it < kB5Halves * nb) {
        fb = order[it / kB5Halves];
        fstart = bstart[fb];
        flen = blen[fb];
      }
    };
    int nitem, nbk, nstart, nlen;
    fetch(nitem, nbk, nstart, nlen);
    for (;;) {
      const int item = nitem, b = nbk, start = nstart, len = nlen;
      if (item >= kB5Halves * nb) break;
      fetch(nitem, nbk, nstart, nlen);
      const int half = item % kB5Halves;
      const bool hrows = half == 0;
      const int nch = (len + kB5K - 1) / kB5K;
      for (int ch = 0; ch < nch; ++ch, ++q) {
        const int sb = next_stage();
        const int k0 = ch * kB5K, kn = min(kB5K, len - k0);
        double* zrs = zr + sb * kB5K * kB5Ld;
        double* zcs = zc + sb * kB5K * kB5Ld;
        int i2 = 0, i3 = 0;
        const bool ok = lane < kn;
        if (lane < kB5K) {
          if (ok) {
            const long long dk = start + k0 + lane;
            i2 = dmode[S + dk];
            i3 = dmode[2 * S + dk];
            w2s[sb * kB5K + lane] = dw2[dk];
            wxs[sb * kB5K + lane] = dwx[dk];
          } else if (lane < ((kn + 3) & ~3)) {  // padding draws of the last k-step
            w2s[sb * kB5K + lane] = 0.0;
            wxs[sb * kB5K + lane] = 0.0;
            for (int c = 0; c < kB5Tab; ++c) zrs[lane * kB5Ld + c] = zcs[lane * kB5Ld + c] = 0.0;
          }
        }
        if (lane == 0) {
          meta[sb][0] = b;
          meta[sb][1] = half;
          meta[sb][2] = kn;
          meta[sb][3] = ch == nch - 1;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&full[sb], 2u * kB5Tab * 8u * (unsigned)kn);
        __syncwarp();
        if (ok) {
          bulk_g2s(zrs + lane * kB5Ld, V2 + (long long)i2 * kB5Tab, kB5Tab * 8, &full[sb]);
          bulk_g2s(zcs + lane * kB5Ld, V3 + (long long)i3 * kB5Tab, kB5Tab * 8, &full[sb]);
        }
      }
    }
    // end of work: one sentinel stage
    const int sb = next_stage();
    if (lane == 0) {
      meta[sb][0] = -1;
      mbar_arrive(&full[sb]);
    }
    return;
  }
  // ---------------- consumers ----------------
  const int g = lane >> 2, t4 = lane & 3;
  const int rg = warp / 3, cg = warp % 3;
  const int hi = warp >> 1, hj = warp & 1;
  double acc[3][6][2];
  double hc0 = 0.0, hc1 = 0.0;
  bool fresh = true;
  for (unsigned q = 0;; ++q) {
    const int sb = (int)(q % kB5St);
    mbar_wait(&full[sb], (q / kB5St) & 1);
    const int b = meta[sb][0];
    if (b < 0) break;
    const int half = meta[sb][1], kn = meta[sb][2], last = meta[sb][3];
    if (fresh) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      hc0 = hc1 = 0.0;
      fresh = false;
    }
    const bool hw = half == 0 && warp < 4;
    const int ksn = (kn + 3) >> 2;
    {
      const double* zrb = zr + sb * kB5K * kB5Ld + rg * 24 + g;
      const double* zcb = zc + sb * kB5K * kB5Ld + cg * 48 + g;
      const double* w2c = w2s + sb * kB5K;
      for (int ks = 0; ks < ksn; ++ks) {
        const int k = ks * 4 + t4;
        const double wk = w2c[k];
        double av[3], bv[6];
#pragma unroll
        for (int i = 0; i < 3; ++i) av[i] = wk * zrb[k * kB5Ld + i * 8];
#pragma unroll
        for (int j = 0; j < 6; ++j) bv[j] = zcb[k * kB5Ld + j * 8];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 6; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
      }
    }
    if (hw) {
      const double* f2c = zr + sb * kB5K * kB5Ld + 144 + hi * 8 + g;
      const double* f3c = zc + sb * kB5K * kB5Ld + 144 + hj * 8 + g;
      const double* wxc = wxs + sb * kB5K;
      for (int ks = 0; ks < ksn; ++ks) {
        const int k = ks * 4 + t4;
        dmma_8x8x4(hc0, hc1, wxc[k] * f2c[k * kB5Ld], f3c[k * kB5Ld]);  // rows past R are 0
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sb]);  // this warp is done with the stage
    if (last) {
      double* Hb = H + (size_t)b * v.Hsz;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const long long row = (long long)half * kB5Rows + rg * 24 + i * 8 + g;
        if (row >= v.Mrow) continue;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const long long cc = (long long)cg * 48 + j * 8 + 2 * t4;
          if (cc < v.Ncol) Hb[row * v.Ncol + cc] = acc[i][j][0];
          if (cc + 1 < v.Ncol) Hb[row * v.Ncol + cc + 1] = acc[i][j][1];
        }
      }
      if (hw) {
        const int p2 = hi * 8 + g, p3 = hj * 8 + 2 * t4;
        if (p2 < R2 && p3 < R3) h[(size_t)b * spec.dprime + p2 * R3 + p3] = hc0;
        if (p2 < R2 && p3 + 1 < R3) h[(size_t)b * spec.dprime + p2 * R3 + p3 + 1] = hc1;
      }
      fresh = true;
    }
  }
}

size_t vech_bucket5_smem() { return (size_t)kB5St * kB5K * (2 * kB5Ld + 2) * 8 + 16; }

// (B''') 3-way H_b for large ranks (m_2 or m_3 above 144 vech pairs; C5: R = 32, m = 528):
// the H_b tile of k_vech_bucket5 (144 x 144, 18 consumer warps x 3 x 6 DMMA tiles, one producer
// warp, TMA bulk copies into a full/empty mbarrier ring) becomes a work item (bucket, row tile,
// column tile): per draw the producer copies the 144-wide slices [144 rt, 144 rt + 144) of the
// V2 table row and [144 ct, ...) of the V3 table row (tables of width tab_width(m), zero past
// m, L2-resident: C5 19 + 9 MB). Items run longest bucket first from an atomic counter. Warps
// whose 24 rows or 48 columns lie wholly in the zero padding of an edge tile skip their DMMAs,
// so the padded 576^2 tile grid costs (almost) only the 528^2 useful work on the shared FP64
// pipe. h_b comes from k_bucket_h2.
constexpr int kB6Ld = 144 + 4;            // staged slice stride (conflict-free fragment loads)
__global__ void __launch_bounds__(kB5Threads, 1) k_vech_bucket6(
    GramSpec spec, VechSpec v, int tw2, int tw3, const double* __restrict__ V2,
    const double* __restrict__ V3, const int* __restrict__ dmode, const double* __restrict__ dw2,
    const int* __restrict__ bstart, const int* __restrict__ blen,
    const int* __restrict__ nbuckets, const int* __restrict__ order, int* counter,
    double* __restrict__ H) {
  extern __shared__ __align__(16) double smb[];
  double* zr = smb;                                  // [St][K][Ld] V2 row slices
  double* zc = zr + kB5St * kB5K * kB6Ld;            // [St][K][Ld] V3 row slices
  double* w2s = zc + kB5St * kB5K * kB6Ld;           // [St][K]
  __shared__ __align__(8) unsigned long long full[kB5St], empty[kB5St];
  __shared__ int meta[kB5St][5];  // bucket (-1: no more work), row tile, col tile, draws, last
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T2 = tw2 / 144, T3 = tw3 / 144, TT = T2 * T3;
  if (tid == 0) {
    for (int i = 0; i < kB5St; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kB5Mma);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kB5Mma) {
    // ---------------- producer ----------------
    const int nb = *nbuckets;
    const long long S = (long long)spec.s;
    unsigned q = 0;
    auto next_stage = [&]() {
      const int sb = (int)(q % kB5St);
      if (q >= kB5St) mbar_wait(&empty[sb], ((q / kB5St) - 1) & 1);
      return sb;
    };
    auto fetch = [&](int& it, int& fb, int& fstart, int& flen) {
      int t = 0;
      if (lane == 0) t = atomicAdd(counter, 1);
      it = __shfl_sync(0xffffffffu, t, 0);
      fb = -1;
      fstart = flen = 0;
      if (it < TT * nb) {
        fb = order[it / TT];
        fstart = bstart[fb];
        flen = blen[fb];
      }
    };
    int nitem, nbk, nstart, nlen;
    fetch(nitem, nbk, nstart, nlen);
    for (;;) {
      const int item = nitem, b = nbk, start = nstart, len = nlen;
      if (item >= TT * nb) break;
      fetch(nitem, nbk, nstart, nlen);
      const int tile = item % TT, rt = tile / T3, ct = tile - rt * T3;
      const int nch = (len + kB5K - 1) / kB5K;
      for (int ch = 0; ch < nch; ++ch, ++q) {
        const int sb = next_stage();
        const int k0 = ch * kB5K, kn = min(kB5K, len - k0);
        double* zrs = zr + sb * kB5K * kB6Ld;
        double* zcs = zc + sb * kB5K * kB6Ld;
        int i2 = 0, i3 = 0;
        const bool ok = lane < kn;
        if (lane < kB5K) {
          if (ok) {
            const long long dk = start + k0 + lane;
            i2 = dmode[S + dk];
            i3 = dmode[2 * S + dk];
            w2s[sb * kB5K + lane] = dw2[dk];
          } else if (lane < ((kn + 3) & ~3)) {  // padding draws of the last k-step
            w2s[sb * kB5K + lane] = 0.0;
            for (int c = 0; c < 144; ++c) zrs[lane * kB6Ld + c] = zcs[lane * kB6Ld + c] = 0.0;
          }
        }
        if (lane == 0) {
          meta[sb][0] = b;
          meta[sb][1] = rt;
          meta[sb][2] = ct;
          meta[sb][3] = kn;
          meta[sb][4] = ch == nch - 1;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&full[sb], 2u * 144u * 8u * (unsigned)kn);
        __syncwarp();
        if (ok) {
          bulk_g2s(zrs + lane * kB6Ld, V2 + (long long)i2 * tw2 + rt * 144, 144 * 8, &full[sb]);
          bulk_g2s(zcs + lane * kB6Ld, V3 + (long long)i3 * tw3 + ct * 144, 144 * 8, &full[sb]);
        }
      }
    }
    const int sb = next_stage();
    if (lane == 0) {
      meta[sb][0] = -1;
      mbar_arrive(&full[sb]);
    }
    return;
  }
  // ---------------- consumers ----------------
  const int g = lane >> 2, t4 = lane & 3;
  const int rg = warp / 3, cg = warp % 3;
  double acc[3][6][2];
  bool fresh = true;
  for (unsigned q = 0;; ++q) {
    const int sb = (int)(q % kB5St);
    mbar_wait(&full[sb], (q / kB5St) & 1);
    const int b = meta[sb][0];
    if (b < 0) break;
    const int rt = meta[sb][1], ct = meta[sb][2], kn = meta[sb][3], last = meta[sb][4];
    if (fresh) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      fresh = false;
    }
    const long long row0 = (long long)rt * 144 + rg * 24, col0 = (long long)ct * 144 + cg * 48;
    const bool live = row0 < v.Mrow && col0 < v.Ncol;  // warp-uniform
    if (live) {
      const int ksn = (kn + 3) >> 2;
      const double* zrb = zr + sb * kB5K * kB6Ld + rg * 24 + g;
      const double* zcb = zc + sb * kB5K * kB6Ld + cg * 48 + g;
      const double* w2c = w2s + sb * kB5K;
      for (int ks = 0; ks < ksn; ++ks) {
        const int k = ks * 4 + t4;
        const double wk = w2c[k];
        double av[3], bv[6];
#pragma unroll
        for (int i = 0; i < 3; ++i) av[i] = wk * zrb[k * kB6Ld + i * 8];
#pragma unroll
        for (int j = 0; j < 6; ++j) bv[j] = zcb[k * kB6Ld + j * 8];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 6; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sb]);
    if (last) {
      if (live) {
        double* Hb = H + (size_t)b * v.Hsz;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const long long row = row0 + i * 8 + g;
          if (row >= v.Mrow) continue;
#pragma unroll
          for (int j = 0; j < 6; ++j) {
            const long long cc = col0 + j * 8 + 2 * t4;
            if (cc < v.Ncol) Hb[row * v.Ncol + cc] = acc[i][j][0];
            if (cc + 1 < v.Ncol) Hb[row * v.Ncol + cc + 1] = acc[i][j][1];
          }
        }
      }
      fresh = true;
    }
  }
}

size_t vech_bucket6_smem() { return (size_t)kB5St * kB5K * (2 * kB6Ld + 1) * 8 + 16; }

// h_b[p'] = sum_{t in b} w_t^2 x_t prod_{n>=1} a_n(i_n)[p_n] from the draw records.
__global__ void __launch_bounds__(256) k_bucket_h2(GramSpec spec, const double* __restrict__ dwx,
                                                   const int* __restrict__ dmode,
                                                   const int* __restrict__ bstart,
                                                   const int* __restrict__ blen,
                                                   const int* __restrict__ nbuckets,
                                                   double* __restrict__ h) {
  const int b = blockIdx.x;
  if (b >= *nbuckets) return;
  const int N = spec.order, dp = spec.dprime;
  const int start = bstart[b], len = blen[b];
  for (int p = threadIdx.x; p < dp; p += blockDim.x) {
    int pn[kMaxOrder];
    {
      int rem = p;
      for (int n = N - 1; n >= 1; --n) {
        pn[n] = rem % spec.ranks[n];
        rem /= spec.ranks[n];
      }
    }
    double acc = 0.0;
    for (int k = 0; k < len; ++k) {
      double z = __ldg(dwx + start + k);
      for (int n = 1; n < N; ++n)
        z *= __ldg(spec.factors[n] + (size_t)__ldg(dmode + (size_t)n * spec.s + start + k) *
                                         spec.ranks[n] + pn[n]);
      acc += z;
    }
    h[(size_t)b * dp + p] = acc;
  }
}

// h_b for order 3 with the draws' raw factor rows staged in shared memory, 64 draws per
// chunk (C5: ~980 draws x 1024 outputs per bucket; k_bucket_h2's per-output chains of
// dependent gathers took 2.7 ms there): h_b[p2, p3] = sum_k (w^2 x)_k a_2(i2_k)[p2] a_3(i3_k)[p3].
constexpr int kH4K = 64;
__global__ void __launch_bounds__(256) k_bucket_h4(GramSpec spec, const double* __restrict__ dwx,
                                                   const int* __restrict__ dmode,
                                                   const int* __restrict__ bstart,
                                                   const int* __restrict__ blen,
                                                   const int* __restrict__ nbuckets,
                                                   double* __restrict__ h) {
  __shared__ double f2[kH4K][33], f3[kH4K][33], wx[kH4K];
  const int b = blockIdx.x;
  if (b >= *nbuckets) return;
  const int R2 = spec.ranks[1], R3 = spec.ranks[2], dp = spec.dprime;
  const int start = bstart[b], len = blen[b];
  const double* A2 = spec.factors[1];
  const double* A3 = spec.factors[2];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int p2[4], p3[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int pp = threadIdx.x + 256 * j;
    p2[j] = pp < dp ? pp / R3 : 0;
    p3[j] = pp < dp ? pp - (pp / R3) * R3 : 0;
  }
  for (int k0 = 0; k0 < len; k0 += kH4K) {
    const int kn = min(kH4K, len - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kn * 32; e += 256) {
      const int k = e >> 5, c = e & 31;
      const long long dk = (long long)start + k0 + k;
      const int i2 = __ldg(dmode + spec.s + dk), i3 = __ldg(dmode + 2 * spec.s + dk);
      f2[k][c] = c < R2 ? __ldg(A2 + (size_t)i2 * R2 + c) : 0.0;
      f3[k][c] = c < R3 ? __ldg(A3 + (size_t)i3 * R3 + c) : 0.0;
      if (c == 0) wx[k] = __ldg(dwx + dk);
    }
    __syncthreads();
    for (int k = 0; k < kn; ++k) {
      const double w = wx[k];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = fma(w * f2[k][p2[j]], f3[k][p3[j]], acc[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int pp = threadIdx.x + 256 * j;
    if (pp < dp) h[(size_t)b * dp + pp] = acc[j];
  }
}

// h_b from the contiguous draw records (drow rows are shared by the whole CTA -> L1).
__global__ void __launch_bounds__(256) k_bucket_h3(GramSpec spec, VechSpec v,
                                                   const double* __restrict__ dwx,
                                                   const double* __restrict__ drow,
                                                   const int* __restrict__ bstart,
                                                   const int* __restrict__ blen,
                                                   const int* __restrict__ nbuckets,
                                                   double* __restrict__ h) {
  const int b = blockIdx.x;
  if (b >= *nbuckets) return;
  const int N = spec.order, dp = spec.dprime, RL = v.rowlen;
  const int start = bstart[b], len = blen[b];
  for (int p = threadIdx.x; p < dp; p += blockDim.x) {
    int hq[kMaxOrder];
    int rem = p;
#pragma unroll
    for (int n = kMaxOrder - 1; n >= 1; --n) {
      hq[n] = 0;
      if (n < N) {
        hq[n] = v.roff[n] + rem % v.R[n];
        rem /= v.R[n];
      }
    }
    double acc = 0.0;
#pragma unroll 4
    for (int k = 0; k < len; ++k) {
      const double* f = drow + (size_t)(start + k) * RL;
      double z = __ldg(dwx + start + k);
#pragma unroll
      for (int n = 1; n < kMaxOrder; ++n)
        if (n < N) z *= __ldg(f + hq[n]);
      acc += z;
    }
    h[(size_t)b * dp + p] = acc;
  }
}

// rhs, two levels: partial[g][p1 * d' + p'] = sum_{b in group g} A1[i1_b, p1] h[b, p'],
// then rhs = sum_g partial[g] (fixed order).
__global__ void __launch_bounds__(256) k_rhs_part(GramSpec spec, const double* __restrict__ h,
                                                  const int* __restrict__ bi1,
                                                  const int* __restrict__ nbuckets,
                                                  double* __restrict__ part) {
  const int R1 = spec.ranks[0], dp = spec.dprime;
  const int grp = blockIdx.y;
  const int nb = *nbuckets;
  const int per = (nb + kRhsSplit - 1) / kRhsSplit;
  const int b0 = grp * per, b1 = min(nb, b0 + per);
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)spec.d) return;
  const int p1 = (int)(e / dp), pp = (int)(e - (long long)p1 * dp);
  double s = 0.0;
  for (int b = b0; b < b1; ++b)
    s = fma(__ldg(spec.factors[0] + (size_t)__ldg(bi1 + b) * R1 + p1),
            __ldg(h + (size_t)b * dp + pp), s);
  part[(size_t)grp * spec.d + e] = s;
}

__global__ void k_rhs_sum(int d, const double* __restrict__ part, double* __restrict__ rhs) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d) return;
  double s = 0.0;
  for (int g = 0; g < kRhsSplit; ++g) s += part[(size_t)g * d + e];
  rhs[e] = s;
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

// (C') S = V1^T H with the full M = m_1 (<= 144) per CTA, so every H column panel is
// read once (the 48-row tiling of k_vech_contract reads it three times). 18 warps,
// warp w -> row tile w x 64 columns; K = buckets in chunks of 32: H chunks by
// cp.async, V1 chunks (vech(a1 a1^T) of the chunk's buckets; thread -> fixed pair
// column) generated while other warps run the previous chunk's DMMAs.
constexpr int TNC2 = 64;
constexpr int LDH2 = TNC2 + 4;
__global__ void __launch_bounds__(kBWarps * 32, 1) k_vech_contract2(GramSpec spec, VechSpec v,
                                                                  const double* __restrict__ H,
                                                                  const int* __restrict__ bi1,
                                                                  const int* __restrict__ nbuckets,
                                                                  double* __restrict__ S) {
  extern __shared__ __align__(16) double smc[];
  double* hs = smc;                    // [2][KCC][LDH2]
  double* vs = hs + 2 * KCC * LDH2;     // [2][KCC][LDZ]
  const int R0 = v.R[0], m0 = v.m[0];
  const int nb = *nbuckets;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const long long n0 = (long long)blockIdx.x * TNC2;
  const int MT = (m0 + 7) / 8;
  const int u = tid % (kBT * 8), k0r = tid / (kBT * 8);  // fixed pair column, rows k0r + 4j
  int pa = 0, pb = 0;
  const bool uok = u < m0;
  if (uok) pair_of(u, R0, pa, pb);
  const double* A0 = spec.factors[0];
  const bool vec = (v.Hsz & 1) == 0;
  auto load_h = [&](int kc, int buf) {
    double* dst = hs + buf * KCC * LDH2;
    for (int e = tid; e < KCC * (TNC2 / 2); e += blockDim.x) {
      const int k = e / (TNC2 / 2), c = (e % (TNC2 / 2)) * 2;
      const bool ok = (kc + k < nb) && (n0 + c < v.Hsz);
      const double* src = ok ? H + (size_t)(kc + k) * v.Hsz + n0 + c : H;
      if (vec) {
        cp_async16(dst + k * LDH2 + c, src, ok);
      } else {
        dst[k * LDH2 + c] = ok ? src[0] : 0.0;
        dst[k * LDH2 + c + 1] = (ok && n0 + c + 1 < v.Hsz) ? src[1] : 0.0;
      }
    }
  };
  auto gen_v = [&](int kc, int buf) {
    double* dst = vs + buf * KCC * LDZ;
#pragma unroll 4
    for (int j = 0; j < KCC / 4; ++j) {
      const int k = k0r + 4 * j;
      double val = 0.0;
      if (uok && kc + k < nb) {
        const double* a = A0 + (size_t)__ldg(bi1 + kc + k) * R0;
        val = __ldg(a + pa) * __ldg(a + pb);
      }
      dst[k * LDZ + u] = val;
    }
  };
  double acc[8][2];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  const int nch = (nb + KCC - 1) / KCC;
  if (nch > 0) load_h(0, 0);
  cp_async_commit();
  if (nch > 0) gen_v(0, 0);
  cp_async_wait<0>();
  __syncthreads();
  for (int kk = 0; kk < nch; ++kk) {
    const int cur = kk & 1;
    if (kk + 1 < nch) load_h((kk + 1) * KCC, cur ^ 1);
    cp_async_commit();
    if (warp < MT) {
      const double* hb = hs + cur * KCC * LDH2;
      const double* vb = vs + cur * KCC * LDZ;
#pragma unroll
      for (int ks = 0; ks < KCC / 4; ++ks) {
        const double af = vb[(ks * 4 + t4) * LDZ + warp * 8 + g];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
          dmma_8x8x4(acc[nt][0], acc[nt][1], af, hb[(ks * 4 + t4) * LDH2 + nt * 8 + g]);
      }
    }
    if (kk + 1 < nch) gen_v((kk + 1) * KCC, cur ^ 1);
    cp_async_wait<0>();
    __syncthreads();
  }
  const int uu = warp * 8 + g;
  if (warp < MT && uu < m0) {
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const long long c = n0 + nt * 8 + 2 * t4;
      if (c < v.Hsz) S[(size_t)uu * v.Hsz + c] = acc[nt][0];
      if (c + 1 < v.Hsz) S[(size_t)uu * v.Hsz + c + 1] = acc[nt][1];
    }
  }
}

// Mode-1 table of every compacted bucket's i_1 (rows b < nbuckets, ld kC3Ldt): vech(a_1 a_1^T)
// in columns [0, m_1) (zero to 144), the raw row a_1 in [144, 144 + R_1) (zero after) -- the A
// operands of k_vech_contract3's Gram and rhs tiles, built once per core update.
__global__ void k_vech_table1(const double* __restrict__ A, int R, const int* __restrict__ bi1,
                              const int* __restrict__ nbuckets, double* __restrict__ out, int tw,
                              int raw) {
  const int b = blockIdx.x;
  if (b >= *nbuckets) return;
  const double* a = A + (size_t)__ldg(bi1 + b) * R;
  const int m = R * (R + 1) / 2;
  for (int u = threadIdx.x; u < tw; u += blockDim.x) {
    double val = 0.0;
    if (u < m) {
      int p, q;
      pair_of(u, R, p, q);
      val = __ldg(a + p) * __ldg(a + q);
    } else if (u >= raw && u < raw + R) {
      val = __ldg(a + u - raw);
    }
    out[(size_t)b * tw + u] = val;
  }
}

// (C'') + (E), warp-specialised: S = V1^T H and rhs = A1_b^T h in one launch. A Gram CTA
// owns all m_1 (<= 136) rows x 128 columns of S (one wave at C2: 145 CTAs); an rhs CTA owns
// the R_1 (<= 16) rows x 128 columns of rhs (R_1 x d'), the same loop with the raw-row columns
// of the table as A and h as B. K = buckets in chunks of 32: a producer warp stages each
// chunk -- 32 row segments of H (or h) and 32 table rows -- by TMA bulk copies into a
// 3-deep ring (full / empty mbarriers); consumer warps own one 8-row tile x 16 column tiles
// each (17 fragment loads per 16 DMMAs). No generation, no CTA-wide barrier in the K loop.
// With `blocks` (order 3) the epilogue also writes S in the PCG's last-mode block layout
// (k_vech_blocks' output: B[u_1][u_2][p][q] = S[u_1][u_2 m_3 + vech(p, q)]).
constexpr int kC3N = 128, kC3K = 32, kC3St = 3;
constexpr int kC3Ldh = kC3N + 4, kC3Ldv = kC3Ldt + 4;  // conflict-free fragment loads
constexpr int kC3Mma = 17;
constexpr int kC3Threads = (kC3Mma + 1) * 32;
size_t vech_contract3_smem() { return (size_t)kC3St * kC3K * (kC3Ldh + kC3Ldv) * 8; }
__global__ void __launch_bounds__(kC3Threads, 1) k_vech_contract3(
    VechSpec v, const double* __restrict__ H, const double* __restrict__ V1,
    const int* __restrict__ nbuckets, double* __restrict__ S, const double* __restrict__ h,
    int dprime, double* __restrict__ rhs, double* __restrict__ blocks, C3Geom gm) {
  extern __shared__ __align__(16) double smc3[];
  double* hs = smc3;                          // [St][K][Ldh]
  double* vs = hs + kC3St * kC3K * kC3Ldh;    // [St][K][Ldv]
  __shared__ __align__(8) unsigned long long full[kC3St], empty[kC3St];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gram_ctas = (int)((v.Hsz + kC3N - 1) / kC3N) * gm.nrb;
  const bool is_rhs = (int)blockIdx.x >= gram_ctas;
  // Gram CTA: column tile ct, row block rb (consecutive CTAs share the column tile of H)
  const int ct = is_rhs ? (int)blockIdx.x - gram_ctas : (int)blockIdx.x / gm.nrb;
  const int rb = is_rhs ? 0 : (int)blockIdx.x - ct * gm.nrb;
  const int row0 = rb * kC3Rows;
  const int rows = is_rhs ? v.R[0] : min(kC3Rows, v.m[0] - row0), MT = (rows + 7) / 8;
  // staged window of the table row, and the A columns within it
  const int woff = is_rhs ? (gm.nrb == 1 ? 0 : gm.raw) : row0;
  const int acol = is_rhs ? (gm.nrb == 1 ? kC3Raw : 0) : 0;
  const long long ld = is_rhs ? dprime : v.Hsz;
  const double* B = is_rhs ? h : H;
  const long long n0 = (long long)ct * kC3N;
  const int ncols = (int)(ld - n0 < kC3N ? ld - n0 : kC3N);
  const int nb = *nbuckets;
  const int nch = (nb + kC3K - 1) / kC3K;
  if (tid == 0) {
    for (int i = 0; i < kC3St; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], MT);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kC3Mma) {
    // ---------------- producer ----------------
    const unsigned hbytes = (unsigned)ncols * 8u;
    for (int ch = 0; ch < nch; ++ch) {
      const int sb = ch % kC3St;
      if (ch >= kC3St) mbar_wait(&empty[sb], ((ch / kC3St) - 1) & 1);
      const int k = ch * kC3K + lane;
      double* hrow = hs + (sb * kC3K + lane) * kC3Ldh;
      double* vrow = vs + (sb * kC3K + lane) * kC3Ldv;
      const bool ok = k < nb;
      if (!ok) {  // past the last bucket: zero rows (finite products with the zero V rows)
        for (int c = 0; c < kC3N; ++c) hrow[c] = 0.0;
        for (int c = 0; c < kC3Ldt; ++c) vrow[c] = 0.0;
      }
      const int kn = min(kC3K, nb - ch * kC3K);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[sb], (hbytes + kC3Ldt * 8u) * (unsigned)kn);
      __syncwarp();
      if (ok) {
        bulk_g2s(hrow, B + (size_t)k * ld + n0, hbytes, &full[sb]);
        bulk_g2s(vrow, V1 + (size_t)k * gm.tw + woff, kC3Ldt * 8u, &full[sb]);
      }
    }
    return;
  }
  if (warp >= MT) return;
  // ---------------- consumers ----------------
  const int g = lane >> 2, t4 = lane & 3;
  double acc[16][2];
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    const int sb = ch % kC3St;
    mbar_wait(&full[sb], (ch / kC3St) & 1);
    const double* hb = hs + sb * kC3K * kC3Ldh + g;
    const double* vb = vs + sb * kC3K * kC3Ldv + acol + warp * 8 + g;
    const int ksn = (min(kC3K, nb - ch * kC3K) + 3) >> 2;
    for (int ks = 0; ks < ksn; ++ks) {
      const int k = ks * 4 + t4;
      const double af = vb[k * kC3Ldv];
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) dmma_8x8x4(acc[nt][0], acc[nt][1], af, hb[k * kC3Ldh + nt * 8]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sb]);
  }
  const int uu = warp * 8 + g;
  if (is_rhs) {
    if (uu >= rows) return;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const int c = nt * 8 + 2 * t4;
      if (c < ncols) rhs[(size_t)uu * dprime + n0 + c] = acc[nt][0];
      if (c + 1 < ncols) rhs[(size_t)uu * dprime + n0 + c + 1] = acc[nt][1];
    }
    return;
  }
  // epilogue through shared memory (the ring is free: every chunk was consumed): the tile
  // (rows x 128) is staged, then S rows and the PCG blocks are written coalesced
  asm volatile("bar.sync 1, %0;" ::"r"(MT * 32) : "memory");
  double* T = smc3;  // [rows][kC3Ldh]
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    T[uu * kC3Ldh + nt * 8 + 2 * t4] = acc[nt][0];
    T[uu * kC3Ldh + nt * 8 + 2 * t4 + 1] = acc[nt][1];
  }
  asm volatile("bar.sync 1, %0;" ::"r"(MT * 32) : "memory");
  const int nth = MT * 32;
  for (int i = tid; i < rows * ncols; i += nth) {
    const int r = i / ncols, c = i - r * ncols;
    S[(size_t)(row0 + r) * v.Hsz + n0 + c] = T[r * kC3Ldh + c];
  }
  if (!blocks) return;
  // column c of the tile is U = n0 + c = (u_2, vech(p, q)): entries (p, q) and (q, p) of block
  // (u_1, u_2); the map is built once per CTA, then every thread writes tile entries
  const int m3 = (int)v.Ncol, R3 = v.R[2], RR = R3 * R3;
  __shared__ int cmap[3][kC3N];
  asm volatile("bar.sync 1, %0;" ::"r"(MT * 32) : "memory");
  for (int c = tid; c < ncols; c += nth) {
    const long long U = n0 + c;
    const int u2 = (int)(U / m3);
    int p, q;
    pair_of((int)(U - (long long)u2 * m3), R3, p, q);
    cmap[0][c] = u2 * RR;
    cmap[1][c] = p * R3 + q;
    cmap[2][c] = q * R3 + p;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(MT * 32) : "memory");
  for (int i = tid; i < rows * kC3N; i += nth) {
    const int r = i / kC3N, c = i % kC3N;
    if (c >= ncols) continue;
    const double val = T[r * kC3Ldh + c];
    double* bb = blocks + (size_t)(row0 + r) * v.m[1] * RR + cmap[0][c];
    bb[cmap[1][c]] = val;
    bb[cmap[2][c]] = val;
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
                              double* __restrict__ B, unsigned boff = 0) {
  // one CTA per block (u_1..u_{N-1}); threads over the R_N x R_N entries; boff: the first
  // block of a slice range (the output starts there)
  const int N = v.N, RL = v.R[N - 1];
  int un[kMaxOrder];
  {
    unsigned t = blockIdx.x + boff;
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

namespace {

// (A)-(B) and the rhs ingredient: sort the draws by i1, gather their records, H_b and h_b
// per nonempty bucket (compacted: bucket b holds i1 = bi1[b]).
void keys_reset(const GramSpec& spec, const GramLayout& l, unsigned long long* data_draws_dev,
                cudaStream_t st) {
  RTB_CUDA(cudaMemsetAsync(l.counts, 0, (size_t)spec.rows[0] * 4, st));
  RTB_CUDA(cudaMemsetAsync(l.aug_count, 0, (size_t)spec.d * 4, st));
  RTB_CUDA(cudaMemsetAsync(data_draws_dev, 0, 8, st));
}

// stable sort of the draws by key (i1), the compacted bucket table, and (with `order`) the
// buckets longest first for the persistent bucket kernels
void sort_keys(const GramSpec& spec, const GramLayout& l, bool order, cudaStream_t st) {
  const int I1 = spec.rows[0];
  size_t cb = l.cub_bytes;
  RTB_CUDA(cub::DeviceRadixSort::SortPairs(l.cub_tmp, cb, l.keys, l.keys_sorted, l.vals,
                                           l.vals_sorted, (int)spec.s, 0, key_bits(I1), st));
  k_bucket_scan<<<1, 1024, 0, st>>>(I1, l.counts, l.bstart, l.blen, l.bi1, l.nbuckets);
  RTB_LAUNCH_CHECK();
  if (order) {
    k_bucket_order<<<1, 1024, 0, st>>>(l.blen, l.nbuckets, l.border, l.bcounter);
    RTB_LAUNCH_CHECK();
  }
}

void bucket_stage(const GramSpec& spec, const VechSpec& v, const GramLayout& l, const double* x,
                  const unsigned long long* idx, const double* w,
                  unsigned long long* data_draws_dev, cudaStream_t st, bool keys_ready = false) {
  const int I1 = spec.rows[0];
  const unsigned sb = (unsigned)ceil_div<unsigned long long>(spec.s, 256ULL);
  if (!keys_ready) {
    keys_reset(spec, l, data_draws_dev, st);
    k_sketch_keys<<<sb, 256, 0, st>>>(spec, idx, l.keys, l.vals, l.counts, l.aug_count,
                                      data_draws_dev);
    RTB_LAUNCH_CHECK();
    sort_keys(spec, l, false, st);
  }
  // draw records in bucket order (one gather of x per draw)
  k_gather_draws<<<sb, 256, 0, st>>>(spec, x, idx, w, l.vals_sorted, l.keys_sorted, l.dw2, l.dwx,
                                     l.dmode);
  RTB_LAUNCH_CHECK();
  // Every bucket slot up to I1 is launched; blocks beyond *nbuckets exit.
  const int NTn = (int)((v.Ncol + 7) / 8);
  const int nr = v.msplit, nc = v.N - 1 - v.msplit;
  const bool whole = (v.Mrow + 7) / 8 <= kBT && NTn <= kBT && v.N >= 2 &&
                     ((nr == 1 && nc <= 2) || (nr == 2 && nc == 1)) &&
                     vech_bucket2_smem(v) <= 227 * 1024;
  // h_b by the bucket kernel's spare warp in the 3-way case (R_2, R_3 <= 16)
  const bool fused_h = whole && nr == 1 && nc == 1 && v.R[1] <= 16 && v.R[2] <= 16 &&
                       (v.Mrow + 7) / 8 < kBWarps;
  static const bool b5_off_g = std::getenv("RTB_NO_BUCKET5") != nullptr;
  static const bool b6_off_g = std::getenv("RTB_NO_BUCKET6") != nullptr;
  // the 144 x 144-tile bucket kernel pays off for R_2 = R_3 = 16 (136 vech pairs) and
  // buckets long enough to fill its 24-draw stages (C2: ~195 draws per bucket)
  const bool b5 = fused_h && !b5_off_g && v.N == 3 && v.R[1] <= 16 && v.R[2] <= 16 &&
                  v.Mrow > 120 && v.Ncol > 120 && (double)spec.s >= 48.0 * I1;
  if (whole) {
    if (!b5) {
      k_gather_rows<<<(unsigned)ceil_div<unsigned long long>(spec.s * v.rowlen, 256ULL), 256, 0,
                      st>>>(spec, v, l.keys_sorted, l.dmode, l.drow);
      RTB_LAUNCH_CHECK();
    }
    const size_t smb = vech_bucket2_smem(v);
    const int smax = 227 * 1024;
    auto launch = [&](auto kern) {
      set_max_smem(kern, smax);
      kern<<<I1, kBWarps * 32, smb, st>>>(spec, v, l.dw2, l.dwx, l.drow, l.bstart, l.blen,
                                          l.nbuckets, l.H, l.h);
      RTB_LAUNCH_CHECK();
    };
    // (NR, NC) = (1, 1) for 3-way; (1, 0) for 2-way; (1, 2) / (2, 1) for 4-way
    auto by_nt = [&](auto hpt, auto nrt, auto nct) {
      constexpr int H_ = decltype(hpt)::value, R_ = decltype(nrt)::value, C_ = decltype(nct)::value;
      if (NTn <= 4) launch(k_vech_bucket2<4, H_, R_, C_>);
      else if (NTn <= 8) launch(k_vech_bucket2<8, H_, R_, C_>);
      else if (NTn <= 12) launch(k_vech_bucket2<12, H_, R_, C_>);
      else if (NTn == 17) {
        launch(k_vech_bucket2<17, H_, R_, C_>);  // R = 16: 136 = 17 x 8
        count_variant("k_vech_bucket2<17>");
      }
      else launch(k_vech_bucket2<18, H_, R_, C_>);
    };
    using I0 = std::integral_constant<int, 0>;
    using I1c = std::integral_constant<int, 1>;
    using I2c = std::integral_constant<int, 2>;
    auto by_groups = [&](auto hpt) {
      if (nr == 1 && nc == 1) by_nt(hpt, I1c{}, I1c{});
      else if (nr == 1 && nc == 0) by_nt(hpt, I1c{}, I0{});
      else if (nr == 1 && nc == 2) by_nt(hpt, I1c{}, I2c{});
      else by_nt(hpt, I2c{}, I1c{});
    };
    if (b5) {
      // vech tables of A_2, A_3, then the persistent table-gather bucket kernel
      k_vech_table<<<(unsigned)ceil_div<long long>((long long)spec.rows[1] * kB5Tab, 256), 256, 0,
                     st>>>(spec.factors[1], spec.rows[1], v.R[1], kB5Tab, l.vt2);
      RTB_LAUNCH_CHECK();
      k_vech_table<<<(unsigned)ceil_div<long long>((long long)spec.rows[2] * kB5Tab, 256), 256, 0,
                     st>>>(spec.factors[2], spec.rows[2], v.R[2], kB5Tab, l.vt3);
      RTB_LAUNCH_CHECK();
      if (!keys_ready) {
        k_bucket_order<<<1, 1024, 0, st>>>(l.blen, l.nbuckets, l.border, l.bcounter);
        RTB_LAUNCH_CHECK();
      }
      const size_t smb5 = vech_bucket5_smem();
      set_max_smem(k_vech_bucket5, (int)smb5);
      int dev = 0, sms = 0;
      RTB_CUDA(cudaGetDevice(&dev));
      RTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      static const int b5_grid = std::getenv("RTB_B5_GRID") ? std::atoi(std::getenv("RTB_B5_GRID")) : 0;
      k_vech_bucket5<<<b5_grid > 0 ? b5_grid : std::min(kB5Halves * I1, kB5CtaPerSm * sms),
                       kB5Threads, smb5, st>>>(
          spec, v, l.vt2, l.vt3, l.dmode, l.dw2, l.dwx, l.bstart, l.blen, l.nbuckets, l.border,
          l.bcounter, l.H, l.h);
      RTB_LAUNCH_CHECK();
      count_variant("k_vech_bucket5");
    } else if (fused_h) {
      by_nt(I1c{}, I1c{}, I1c{});
    } else {
      by_groups(I0{});
    }
  } else if (v.N == 3 && nr == 1 && nc == 1 && v.R[1] <= 32 && v.R[2] <= 32 && !b6_off_g) {
    // large ranks (C5): table-gather tiles of 144 x 144
    const int tw2 = tab_width(v.m[1]) == 160 ? 144 : tab_width(v.m[1]);
    const int tw3 = tab_width(v.m[2]) == 160 ? 144 : tab_width(v.m[2]);
    k_vech_table<<<(unsigned)ceil_div<long long>((long long)spec.rows[1] * tw2, 256), 256, 0, st>>>(
        spec.factors[1], spec.rows[1], v.R[1], tw2, l.vt2);
    RTB_LAUNCH_CHECK();
    k_vech_table<<<(unsigned)ceil_div<long long>((long long)spec.rows[2] * tw3, 256), 256, 0, st>>>(
        spec.factors[2], spec.rows[2], v.R[2], tw3, l.vt3);
    RTB_LAUNCH_CHECK();
    if (!keys_ready) {
      k_bucket_order<<<1, 1024, 0, st>>>(l.blen, l.nbuckets, l.border, l.bcounter);
      RTB_LAUNCH_CHECK();
    }
    const size_t smb6 = vech_bucket6_smem();
    set_max_smem(k_vech_bucket6, (int)smb6);
    int dev = 0, sms = 0;
    RTB_CUDA(cudaGetDevice(&dev));
    RTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long long items = (long long)(tw2 / 144) * (tw3 / 144) * I1;
    k_vech_bucket6<<<(unsigned)std::min<long long>(items, sms), kB5Threads, smb6, st>>>(
        spec, v, tw2, tw3, l.vt2, l.vt3, l.dmode, l.dw2, l.bstart, l.blen, l.nbuckets, l.border,
        l.bcounter, l.H);
    RTB_LAUNCH_CHECK();
    count_variant("k_vech_bucket6");
  } else {
    const long long tiles_r = (v.Mrow + TB - 1) / TB, tiles_c = (v.Ncol + TB - 1) / TB;
    k_vech_bucket<<<dim3((unsigned)(tiles_r * tiles_c), I1), kTh,
                    (size_t)KC * v.rowlen * sizeof(double), st>>>(
        spec, v, idx, w, l.vals_sorted, l.bstart, l.blen, l.nbuckets, l.H);
    RTB_LAUNCH_CHECK();
  }
  if (whole && !fused_h) {
    k_bucket_h3<<<I1, 256, 0, st>>>(spec, v, l.dwx, l.drow, l.bstart, l.blen, l.nbuckets, l.h);
    RTB_LAUNCH_CHECK();
  } else if (!fused_h && v.N == 3 && v.R[1] <= 32 && v.R[2] <= 32 && spec.dprime <= 1024) {
    k_bucket_h4<<<I1, 256, 0, st>>>(spec, l.dwx, l.dmode, l.bstart, l.blen, l.nbuckets, l.h);
    RTB_LAUNCH_CHECK();
  } else if (!fused_h) {
    k_bucket_h2<<<I1, 256, 0, st>>>(spec, l.dwx, l.dmode, l.bstart, l.blen, l.nbuckets, l.h);
    RTB_LAUNCH_CHECK();
  }
}

// ---- order 4, bucketing by (i1, i2) ----
// The order-4 vech Gram S[u1][u2][u3][u4] (vech pairs per mode) bucketed by i1 alone costs
// s_data m2 m3 m4 multiply-adds in (B) (C3: 4.2e10). Bucketing by the pair (i1, i2) instead
// -- the order-3 pipeline run on the merged view (I1 I2) x I3 x I4, whose flat draw indices are
// the same numbers -- gives H_{(i1,i2)}[u3][u4] at s_data m3 m4 (C3: 7.6e8) plus two GEMMs
// over vech Khatri-Rao rows:
//   T_{i1}[u2][U] = sum_{i2} v2(i2)[u2] H_{(i1,i2)}[U]        (batched over i1)
//   S[u1][u2 U]   = sum_{i1} v1(i1)[u1] T_{i1}[u2 U]
// and likewise rhs = sum_{i1} a1(i1) (x) sum_{i2} a2(i2) (x) h_{(i1,i2)} (C3: 6.5e9 MACs in
// all, 6.7x fewer).
// dense per-(i1, i2) copies of the compacted H_b and h_b (zero rows for empty pairs)
__global__ void k_scatter_buckets(const double* __restrict__ H, const double* __restrict__ h,
                                  const int* __restrict__ bi1, const int* __restrict__ nbuckets,
                                  long long hsz, int hp, double* __restrict__ Hd,
                                  double* __restrict__ hd) {
  const int b = blockIdx.x;
  if (b >= *nbuckets) return;
  const long long dst = bi1[b];
  for (long long e = threadIdx.x; e < hsz; e += blockDim.x) Hd[dst * hsz + e] = H[(long long)b * hsz + e];
  for (int e = threadIdx.x; e < hp; e += blockDim.x) hd[dst * hp + e] = h[(long long)b * hp + e];
}

// vech Khatri-Rao rows: kr[i][u] = A[i,a] A[i,b], u = vech pair (a <= b)
__global__ void k_vech_kr(const double* __restrict__ A, int I, int R, double* __restrict__ kr) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int m = R * (R + 1) / 2;
  if (e >= (long long)I * m) return;
  const long long i = e / m;
  int a, b;
  pair_of((int)(e % m), R, a, b);
  kr[e] = A[i * R + a] * A[i * R + b];
}

void sketch_normal_eq_m4(const GramSpec& spec, const double* x, const unsigned long long* idx,
                         const double* w, void* work, double* gram, double* rhs,
                         unsigned long long* data_draws_dev, cudaStream_t st) {
  const VechSpec v4 = make_vech(spec);
  GramLayout l4 = layout(spec, work);
  const size_t base4 = carve(spec, [](size_t, size_t) {});
  M4Extra e = m4_extra(spec, static_cast<char*>(work) + base4);
  const GramSpec g = merged_spec(spec);
  const VechSpec v3 = make_vech(g);
  GramLayout l3 = layout(g, e.w3);
  bucket_stage(g, v3, l3, x, idx, w, data_draws_dev, st);
  const int I1 = spec.rows[0], I2 = spec.rows[1], R1 = spec.ranks[0], R2 = spec.ranks[1];
  const long long P = (long long)I1 * I2;
  RTB_CUDA(cudaMemsetAsync(e.Hd, 0, (size_t)P * v3.Hsz * 8, st));
  RTB_CUDA(cudaMemsetAsync(e.hd, 0, (size_t)P * g.dprime * 8, st));
  k_scatter_buckets<<<(unsigned)P, 256, 0, st>>>(l3.H, l3.h, l3.bi1, l3.nbuckets, v3.Hsz, g.dprime,
                                                 e.Hd, e.hd);
  RTB_LAUNCH_CHECK();
  const int m1 = v4.m[0], m2 = v4.m[1];
  k_vech_kr<<<ceil_div(I1 * m1, 256), 256, 0, st>>>(spec.factors[0], I1, R1, e.ka1);
  RTB_LAUNCH_CHECK();
  k_vech_kr<<<ceil_div(I2 * m2, 256), 256, 0, st>>>(spec.factors[1], I2, R2, e.ka2);
  RTB_LAUNCH_CHECK();
  const long long U = v3.Hsz;  // m3 m4
  // sharded along mode 1: only this shard's i1 rows hold draws, so the contractions run over
  // them alone and S / rhs are this shard's partial sums (the engine all-reduces them)
  const int i1lo = spec.i1_hi > 0 ? spec.i1_lo : 0, i1hi = spec.i1_hi > 0 ? spec.i1_hi : I1;
  const int nl = i1hi - i1lo;
  const double* Hd = e.Hd + (size_t)i1lo * I2 * U;
  const double* hd = e.hd + (size_t)i1lo * I2 * g.dprime;
  // T_{i1} (m2 x U) = KA2^T Hd_{i1}
  gemm_tn(e.ka2, m2, Hd, U, m2, U, I2, e.T, U, st, nl, 0, (long long)I2 * U, (long long)m2 * U);
  // S (m1 x m2 U) = KA1^T T, straight into the order-4 layout's compact Gram
  gemm_tn(e.ka1 + (size_t)i1lo * m1, m1, e.T, (long long)m2 * U, m1, (long long)m2 * U, nl, l4.S,
          (long long)m2 * U, st);
  // rhs: Tr_{i1} (R2 x R3 R4) = A2^T hd_{i1}; rhs (R1 x R2 R3 R4) = A1^T Tr
  const long long hp = g.dprime;
  gemm_tn(spec.factors[1], R2, hd, hp, R2, hp, I2, e.Tr, hp, st, nl, 0, (long long)I2 * hp,
          (long long)R2 * hp);
  gemm_tn(spec.factors[0] + (size_t)i1lo * R1, R1, e.Tr, (long long)R2 * hp, R1,
          (long long)R2 * hp, nl, rhs, (long long)R2 * hp, st);
  RTB_CUDA(cudaMemcpyAsync(l4.aug_count, l3.aug_count, (size_t)spec.d * 4,
                           cudaMemcpyDeviceToDevice, st));
  if (gram) {
    k_vech_expand<<<kNumSMs * 8, 256, 0, st>>>(spec, v4, l4.S, l4.aug_count, gram_aug_term(spec),
                                              gram);
    RTB_LAUNCH_CHECK();
  }
}

}  // namespace

GramKeyBufs gram_key_buffers(const GramSpec& spec, void* work) {
  const GramLayout l = layout(spec, work);
  return GramKeyBufs{l.keys, l.vals, l.counts, l.aug_count};
}

void gram_keys_reset(const GramSpec& spec, void* work, unsigned long long* data_draws_dev,
                     cudaStream_t st) {
  keys_reset(spec, layout(spec, work), data_draws_dev, st);
}

void gram_sort_keys(const GramSpec& spec, void* work, cudaStream_t st) {
  if (spec.order != 3) throw Error(4, "gram_sort_keys: order 3 only");
  sort_keys(spec, layout(spec, work), true, st);
}

bool sketch_normal_eq(const GramSpec& spec, const double* x, const unsigned long long* idx,
                      const double* w, void* work, size_t work_bytes, double* gram, double* rhs,
                      unsigned long long* data_draws_dev, cudaStream_t st, double* blocks,
                      bool keys_ready) {
  if (work_bytes < gram_work_bytes(spec)) throw Error(4, "sketch_normal_eq: workspace too small");
  const VechSpec v = make_vech(spec);
  if (v.rowlen > kMaxRow) throw Error(4, "sketch_normal_eq: sum of ranks beyond mode 1 > 256");
  if (keys_ready && spec.order != 3) throw Error(4, "sketch_normal_eq: keys ahead for order 3 only");
  if (merged4_ok(spec)) {
    sketch_normal_eq_m4(spec, x, idx, w, work, gram, rhs, data_draws_dev, st);
    return false;
  }
  GramLayout l = layout(spec, work);
  bucket_stage(spec, v, l, x, idx, w, data_draws_dev, st, keys_ready);
  if (const char* dump = std::getenv("RTB_DUMP_H")) {  // debugging aid: H and bucket table
    std::vector<double> hh((size_t)spec.rows[0] * v.Hsz);
    std::vector<int> meta(3 * (size_t)spec.rows[0] + 1);
    RTB_CUDA(cudaMemcpyAsync(hh.data(), l.H, hh.size() * 8, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaMemcpyAsync(meta.data(), l.bi1, (size_t)spec.rows[0] * 4, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaMemcpyAsync(meta.data() + spec.rows[0], l.blen, (size_t)spec.rows[0] * 4, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaMemcpyAsync(meta.data() + 3 * (size_t)spec.rows[0], l.nbuckets, 4, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaStreamSynchronize(st));
    FILE* f = std::fopen(dump, "wb");
    if (f) {
      std::fwrite(hh.data(), 8, hh.size(), f);
      std::fwrite(meta.data(), 4, meta.size(), f);
      std::fclose(f);
    }
  }
  const int I1 = spec.rows[0];
  static const bool no_c3 = std::getenv("RTB_NO_CONTRACT3") != nullptr;
  bool rhs_done = false, blocks_done = false;
  static const bool no_c3big = std::getenv("RTB_NO_CONTRACT3_BIG") != nullptr;  // experiments
  if (!no_c3 && (v.m[0] <= 8 * kC3Mma || (!no_c3big && v.R[0] <= 32)) && (v.Hsz & 1) == 0 &&
      v.Hsz >= 16 * kC3N) {
    const C3Geom gm = c3_geom(v.m[0]);
    k_vech_table1<<<I1, 256, 0, st>>>(spec.factors[0], v.R[0], l.bi1, l.nbuckets, l.vt1, gm.tw,
                                      gm.raw);
    RTB_LAUNCH_CHECK();
    const size_t smc = vech_contract3_smem();
    set_max_smem(k_vech_contract3, (int)smc);
    // rhs tiles in the same launch when a_1 fits the table's raw-row window
    static const bool no_rhs = std::getenv("RTB_C3_NORHS") != nullptr;  // experiments
    static const bool no_blk = std::getenv("RTB_C3_NOBLK") != nullptr;
    const int rawcap = gm.nrb == 1 ? kC3Ldt - kC3Raw : kC3Rows;
    const bool fuse_rhs = !no_rhs && v.R[0] <= rawcap && (spec.dprime & 1) == 0;
    const unsigned gram_ctas = (unsigned)((v.Hsz + kC3N - 1) / kC3N) * gm.nrb;
    const unsigned rhs_ctas = fuse_rhs ? (unsigned)ceil_div(spec.dprime, kC3N) : 0u;
    double* bl = (blocks && v.N == 3 && !no_blk) ? blocks : nullptr;
    k_vech_contract3<<<gram_ctas + rhs_ctas, kC3Threads, smc, st>>>(
        v, l.H, l.vt1, l.nbuckets, l.S, l.h, spec.dprime, fuse_rhs ? rhs : nullptr, bl, gm);
    if (gm.nrb > 1) count_variant("k_vech_contract3_rows");
    count_variant("k_vech_contract3");
    rhs_done = fuse_rhs;
    blocks_done = bl != nullptr;
  } else if ((v.m[0] + 7) / 8 <= kBWarps) {
    const size_t smc = (size_t)(2 * KCC * LDH2 + 2 * KCC * LDZ) * 8;
    set_max_smem(k_vech_contract2, (int)smc);
    k_vech_contract2<<<(unsigned)((v.Hsz + TNC2 - 1) / TNC2), kBWarps * 32, smc, st>>>(
        spec, v, l.H, l.bi1, l.nbuckets, l.S);
    count_variant("k_vech_contract2");
  } else {
    k_vech_contract<<<dim3((unsigned)((v.Hsz + TNC - 1) / TNC), (unsigned)ceil_div(v.m[0], TB)),
                      kTh, 0, st>>>(spec, v, l.H, l.bi1, l.nbuckets, l.S);
  }
  RTB_LAUNCH_CHECK();
  const double aug_term = gram_aug_term(spec);
  if (gram) {
    k_vech_expand<<<kNumSMs * 8, 256, 0, st>>>(spec, v, l.S, l.aug_count, aug_term, gram);
    RTB_LAUNCH_CHECK();
  }
  if (!rhs_done) {
    k_rhs_part<<<dim3(ceil_div(spec.d, 256), kRhsSplit), 256, 0, st>>>(spec, l.h, l.bi1,
                                                                        l.nbuckets, l.rhs_part);
    RTB_LAUNCH_CHECK();
    k_rhs_sum<<<ceil_div(spec.d, 256), 256, 0, st>>>(spec.d, l.rhs_part, rhs);
    RTB_LAUNCH_CHECK();
  }
  return blocks_done;
}

void gram_expand_full(const GramSpec& spec, void* work, double* gram, cudaStream_t st) {
  const VechSpec v = make_vech(spec);
  GramLayout l = layout(spec, work);
  k_vech_expand<<<kNumSMs * 8, 256, 0, st>>>(spec, v, l.S, l.aug_count, gram_aug_term(spec), gram);
  RTB_LAUNCH_CHECK();
}

void gram_expand_blocks_range(const GramSpec& spec, void* work, double* blocks, int u_lo, int u_hi,
                              cudaStream_t st) {
  const VechSpec v = make_vech(spec);
  GramLayout l = layout(spec, work);
  const long long mmid = gram_block_elems(spec) / ((long long)v.R[v.N - 1] * v.R[v.N - 1]) / v.m[0];
  const long long nblk = (long long)(u_hi - u_lo) * mmid;
  if (nblk <= 0) return;
  if (nblk > 0x7fffffffLL) throw Error(4, "gram_expand_blocks: too many blocks");
  k_vech_blocks<<<(unsigned)nblk, 256, 0, st>>>(spec, v, l.S, blocks, (unsigned)(u_lo * mmid));
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
