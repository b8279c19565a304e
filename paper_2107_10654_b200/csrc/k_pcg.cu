// k_pcg.cu -- the sketched core solve as Kronecker-preconditioned conjugate gradients.
//
// Reference: solve_sketched_ridge solves G x = b with a Jacobi-SVD pseudoinverse
// (ref sketch_ridge.cpp:130-139). G = K^T W K + lambda * diag(c) is SPD whenever
// lambda > 0 and every augmented row was drawn (c_j > 0), and it is a (1 +- eps)
// spectral approximation of the unsketched K^T K + lambda I (the point of ridge
// leverage-score sampling). For the Kronecker design K = A_1 (x) ... (x) A_N that
// matrix is cheap to invert exactly:
//     M = (x)_n A_n^T A_n + lambda I = V diag(lambda + prod_n mu_n) V^T,  V = (x)_n V_n
// (V_n, mu_n = eigenpairs of the R_n x R_n factor Gram), so M^-1 r costs 2 N
// mode products on a d-vector. Preconditioned by M, CG sees eigenvalues in
// [1 - eps, 1 + eps] and converges in a few tens of iterations.
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
// every CTA redundantly and bit-identically updates the FULL r, applies M^-1,
// forms the dot products and the next p in shared memory. The result is accepted
// only if the true residual ||b - G x|| <= check_tol ||b|| (one extra matvec);
// otherwise status != 0 and the caller falls back to the Cholesky path.
#include "common.cuh"
#include "kernels.h"

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
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1u);
    while (ld_acquire_u32(counter) < target) __nanosleep(20);
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

// out[o, j, k] = sum_i W[i * R + j] X[o, i, k] on a d-vector in shared memory
// (W = V for X x_n V^T, W = V^T for X x_n V). One thread per fiber (o, k): the R
// inputs are read once, W reads are warp-uniform (J > 1) or contiguous (J = 1).
__device__ __forceinline__ void mode_product(const double* X, double* out, const double* W, int d,
                                             int R, int J) {
  if (J == 1) {  // contiguous fibers: one output per thread, W reads contiguous in j
    for (int e = threadIdx.x; e < d; e += kThreads) {
      const int o = e / R, j = e - o * R;
      const double* x = X + o * R;
      double acc = 0.0;
#pragma unroll 4
      for (int i = 0; i < R; ++i) acc = fma(W[i * R + j], x[i], acc);
      out[e] = acc;
    }
    return;
  }
  const int fibers = d / R;
  for (int f = threadIdx.x; f < fibers; f += kThreads) {
    const int o = f / J, k = f - o * J;
    const int base = o * R * J + k;
    for (int j0 = 0; j0 < R; j0 += 8) {
      double acc[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] = 0.0;
      for (int i = 0; i < R; ++i) {
        const double xi = X[base + i * J];
        const double* w = W + i * R + j0;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (j0 + t < R) acc[t] = fma(w[t], xi, acc[t]);
      }
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (j0 + t < R) out[base + (j0 + t) * J] = acc[t];
    }
  }
}

// z = M^-1 r using scratch a, b; returns the buffer holding z (a or b).
__device__ double* precondition(const PcgShared& sh, const double* r, double* a, double* b,
                                const double* Vs, const double* VTs, const int* voff,
                                const double* dinv) {
  const double* src = r;
  double* dst = a;
  for (int n = 0; n < sh.order; ++n) {
    mode_product(src, dst, Vs + voff[n], sh.d, sh.R[n], sh.J[n]);
    __syncthreads();
    src = dst;
    dst = (dst == a) ? b : a;
  }
  double* t = const_cast<double*>(src);
  for (int e = threadIdx.x; e < sh.d; e += kThreads) t[e] *= dinv[e];
  __syncthreads();
  for (int n = 0; n < sh.order; ++n) {
    mode_product(src, dst, VTs + voff[n], sh.d, sh.R[n], sh.J[n]);
    __syncthreads();
    src = dst;
    dst = (dst == a) ? b : a;
  }
  return const_cast<double*>(src);
}

struct PcgArgs {
  const double* B;        // last-mode blocks of the data Gram
  const double* b;
  double* x;
  double* q;              // [d]
  double* part;           // [m1][2][d']
  double* rpart;          // [grid] residual partials
  unsigned* counter;
  int* status;            // [0] status, [1] iterations
  const double* evals;
  const double* evecs;
  int eig_stride;
  const int* aug_count;
  double aug_term;
  double lambda;
  int max_iter;
  double tol;
  double check_tol;
};

// (A) slice partials: for slice u1 = v(a, b), side 0 = q[a, :] from p[b, :],
// side 1 = q[b, :] from p[a, :] (absent when a == b).
__device__ void slice_partials(const PcgArgs& A, const PcgShared& sh, const double* p) {
  const int last = sh.last, mid = sh.mid, dp = sh.dprime;
  const int nout = 2 * dp;
  for (int u1 = blockIdx.x; u1 < sh.m1; u1 += gridDim.x) {
    int a, b;
    pair_of(u1, sh.R[0], a, b);
    const double* Bs = A.B + (size_t)u1 * sh.mmid * last * last;
    for (int o = threadIdx.x; o < nout; o += kThreads) {
      const int r = o % last;
      const int t = o / last;
      const int side = t & 1, im = t >> 1;
      if (side == 1 && a == b) continue;
      const double* pv = p + (size_t)(side == 0 ? b : a) * dp;
      // middle-mode digits of im (mixed radix R_1..R_{N-2}, last fastest)
      int idig[kMaxOrder];
      {
        int rem = im;
        for (int n = sh.order - 2; n >= 1; --n) {
          idig[n] = rem % sh.R[n];
          rem /= sh.R[n];
        }
      }
      int jdig[kMaxOrder];
      for (int n = 1; n <= sh.order - 2; ++n) jdig[n] = 0;
      double sum = 0.0;
      for (int jm = 0; jm < mid; ++jm) {
        int umid = 0;
        for (int n = 1; n <= sh.order - 2; ++n) {
          const int x = idig[n], y = jdig[n];
          umid = umid * sh.m[n] + upper_pair(min(x, y), max(x, y), sh.R[n]);
        }
        const double* row = Bs + ((size_t)umid * last + r) * last;
        const double* ps = pv + (size_t)jm * last;
        if ((last & 1) == 0) {
          for (int c = 0; c < last; c += 2) {
            const double2 g = __ldg(reinterpret_cast<const double2*>(row + c));
            const double2 pp = *reinterpret_cast<const double2*>(ps + c);
            sum = fma(g.x, pp.x, sum);
            sum = fma(g.y, pp.y, sum);
          }
        } else {
          for (int c = 0; c < last; ++c) sum = fma(__ldg(row + c), ps[c], sum);
        }
        for (int n = sh.order - 2; n >= 1; --n) {  // odometer over the middle modes
          if (++jdig[n] < sh.R[n]) break;
          jdig[n] = 0;
        }
      }
      A.part[((size_t)u1 * 2 + side) * dp + (size_t)im * last + r] = sum;
    }
  }
}

// (B) own rows: q[e] = sum_{j1} partial + augmented diagonal * p[e].
__device__ void reduce_rows(const PcgArgs& A, const PcgShared& sh, const double* p, int row0,
                            int nrows, double* qout) {
  const int dp = sh.dprime, R1 = sh.R[0];
  for (int e = row0 + threadIdx.x; e < row0 + nrows; e += kThreads) {
    const int i1 = e / dp, rest = e - i1 * dp;
    double s = 0.0;
    for (int j1 = 0; j1 < R1; ++j1) {
      const int u1 = upper_pair(min(i1, j1), max(i1, j1), R1);
      const int side = i1 <= j1 ? 0 : 1;
      s += __ldcg(A.part + ((size_t)u1 * 2 + side) * dp + rest);
    }
    const int c = __ldg(A.aug_count + e);
    if (c > 0) s = fma((double)c * A.aug_term, p[e], s);
    qout[e] = s;
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_pcg(const PcgArgs A, const PcgShared shc) {
  extern __shared__ __align__(16) double sm[];
  const PcgShared sh = shc;
  const int d = sh.d;
  int voff[kMaxOrder];
  int vtot = 0;
  for (int n = 0; n < sh.order; ++n) {
    voff[n] = vtot;
    vtot += sh.R[n] * sh.R[n];
  }
  const int dv = (d + 1) & ~1;
  double* Vs = sm;
  double* VTs = Vs + ((vtot + 1) & ~1);
  double* dinv = VTs + ((vtot + 1) & ~1);
  double* r = dinv + dv;
  double* p = r + dv;
  double* s0 = p + dv;
  double* s1 = s0 + dv;
  double* red = s1 + dv;

  // applicability: every augmented column drawn (then G >= lambda * min c_j > 0)
  int missing = 0;
  for (int e = threadIdx.x; e < d; e += kThreads) missing |= __ldg(A.aug_count + e) == 0;
  if (__syncthreads_or(missing) || !(A.lambda > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.status[0] = 3;
      A.status[1] = 0;
    }
    return;
  }

  for (int n = 0; n < sh.order; ++n) {
    const int R = sh.R[n];
    for (int e = threadIdx.x; e < R * R; e += kThreads) {
      const double v = A.evecs[(size_t)n * A.eig_stride + e];  // V[i][k], column k
      Vs[voff[n] + e] = v;
      VTs[voff[n] + (e % R) * R + e / R] = v;
    }
  }
  for (int e = threadIdx.x; e < d; e += kThreads) {
    double m = 1.0;
    int rem = e;
    for (int n = sh.order - 1; n >= 0; --n) {
      const int j = rem % sh.R[n];
      rem /= sh.R[n];
      m *= fmax(A.evals[(size_t)n * A.eig_stride + j], 0.0);
    }
    dinv[e] = 1.0 / (m + A.lambda);
    r[e] = A.b[e];
  }
  __syncthreads();

  const int row0 = min(d, (int)blockIdx.x * sh.rows_per_cta);
  const int nrows = min(d, row0 + sh.rows_per_cta) - row0;
  unsigned sync_target = 0;

  double bb = 0.0;
  for (int e = threadIdx.x; e < d; e += kThreads) bb = fma(r[e], r[e], bb);
  bb = block_sum_det(bb, red);
  for (int e = row0 + threadIdx.x; e < row0 + nrows; e += kThreads) A.x[e] = 0.0;
  if (bb == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.status[0] = 0;
      A.status[1] = 0;
    }
    return;
  }
  double* z = precondition(sh, r, s0, s1, Vs, VTs, voff, dinv);
  double rho = 0.0;
  for (int e = threadIdx.x; e < d; e += kThreads) {
    p[e] = z[e];
    rho = fma(r[e], z[e], rho);
  }
  rho = block_sum_det(rho, red);

  const double stop = A.tol * A.tol * bb;
  int it = 0;
  int fail = 0;
  for (; it < A.max_iter; ++it) {
    slice_partials(A, sh, p);
    sync_target += gridDim.x;
    grid_barrier(A.counter, sync_target);
    reduce_rows(A, sh, p, row0, nrows, A.q);
    sync_target += gridDim.x;
    grid_barrier(A.counter, sync_target);
    // every CTA: alpha from the full p.q, full r update, own x rows
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
    double rr = 0.0;
    for (int e = threadIdx.x; e < d; e += kThreads) {
      const double re = fma(-alpha, s0[e], r[e]);
      r[e] = re;
      rr = fma(re, re, rr);
    }
    for (int e = row0 + threadIdx.x; e < row0 + nrows; e += kThreads)
      A.x[e] = fma(alpha, p[e], A.x[e]);
    rr = block_sum_det(rr, red);
    if (rr <= stop) {
      ++it;
      break;
    }
    z = precondition(sh, r, s0, s1, Vs, VTs, voff, dinv);
    double rho2 = 0.0;
    for (int e = threadIdx.x; e < d; e += kThreads) rho2 = fma(r[e], z[e], rho2);
    rho2 = block_sum_det(rho2, red);
    const double beta = rho2 / rho;
    rho = rho2;
    for (int e = threadIdx.x; e < d; e += kThreads) p[e] = fma(beta, p[e], z[e]);
    __syncthreads();
  }
  // true residual ||b - G x||: gather x, one matvec, reduce over CTAs
  sync_target += gridDim.x;
  grid_barrier(A.counter, sync_target);
  for (int e = threadIdx.x; e < d; e += kThreads) p[e] = __ldcg(A.x + e);
  __syncthreads();
  slice_partials(A, sh, p);
  sync_target += gridDim.x;
  grid_barrier(A.counter, sync_target);
  reduce_rows(A, sh, p, row0, nrows, A.q);
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
    if (!st && !(tot <= A.check_tol * A.check_tol * bb)) st = 1;
    A.status[0] = st;
    A.status[1] = it;
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

size_t pcg_smem(int d, int order, const int* ranks) {
  int vtot = 0;
  for (int n = 0; n < order; ++n) vtot += ranks[n] * ranks[n];
  const size_t dv = (size_t)((d + 1) & ~1);
  return 8 * (2 * (size_t)((vtot + 1) & ~1) + 5 * dv + 32);
}

}  // namespace

size_t pcg_work_bytes(int d, int r1) {
  const size_t m1 = (size_t)r1 * (r1 + 1) / 2;
  const size_t dp = (size_t)d / r1;
  return ((size_t)d + m1 * 2 * dp + 1024) * 8 + 256;
}

bool pcg_supported(int d, int order, const int* ranks) {
  return d >= 1 && order >= 2 && order <= kMaxOrder && pcg_smem(d, order, ranks) <= 220 * 1024;
}

void pcg_solve(const PcgSpec& spec, const double* blocks, const double* b, double* x, void* work,
               int* status_dev, cudaStream_t st) {
  const int d = spec.d;
  const int grid = num_sms();
  if (!pcg_supported(d, spec.order, spec.ranks)) throw Error(4, "pcg_solve: unsupported shape");
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
  if (inner != d) throw Error(1, "pcg_solve: prod(ranks) != d");
  sh.dprime = d / sh.R[0];
  sh.last = sh.R[spec.order - 1];
  sh.mid = sh.dprime / sh.last;
  sh.mmid = 1;
  for (int n = 1; n < spec.order - 1; ++n) sh.mmid *= sh.m[n];
  sh.m1 = sh.m[0];
  const size_t smem = pcg_smem(d, spec.order, spec.ranks);

  char* w = static_cast<char*>(work);
  PcgArgs a{};
  a.B = blocks;
  a.b = b;
  a.x = x;
  a.q = reinterpret_cast<double*>(w);
  a.part = a.q + d;
  a.rpart = a.part + (size_t)sh.m1 * 2 * sh.dprime;
  a.counter = reinterpret_cast<unsigned*>(a.rpart + 1024);
  a.status = status_dev;
  a.evals = spec.evals;
  a.evecs = spec.evecs;
  a.eig_stride = spec.eig_stride;
  a.aug_count = spec.aug_count;
  a.aug_term = spec.aug_term;
  a.lambda = spec.lambda;
  a.max_iter = spec.max_iter;
  a.tol = spec.tol;
  a.check_tol = spec.check_tol;
  RTB_CUDA(cudaMemsetAsync(a.counter, 0, 64, st));
  static bool attr_set = false;
  if (!attr_set) {
    RTB_CUDA(cudaFuncSetAttribute(k_pcg, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr_set = true;
  }
  void* args[] = {(void*)&a, (void*)&sh};
  RTB_CUDA(cudaLaunchCooperativeKernel((void*)k_pcg, dim3(grid), dim3(kThreads), args, smem, st));
  RTB_LAUNCH_CHECK();
}

}  // namespace rtb
