// k_chol.cu -- on-device Cholesky solve of the sketched normal equations.
//
// The reference solves G x = rhs with a one-sided Jacobi SVD pseudoinverse
// (ref sketch_ridge.cpp:130-139, svd.cpp:21-111): O(sweeps d^3), 186.7 s at
// d = 1024 on one core. G is symmetric positive definite whenever every
// augmented row was drawn at least once (lambda > 0), so we factor G = L L^T.
//
// k_chol_dag is ONE persistent cooperative kernel executing the right-looking
// tile Cholesky as a task DAG over 64x64 tiles (T = ceil(d/64)):
//   P(k)      Cholesky of tile (k,k) (lazy-scaled, all 256 threads) + its
//             inverse Linv_kk (kept for the solves)
//   S(i,k)    L_ik = A_ik Linv_kk^T                        (FP64 DMMA.8x8x4)
//   U(k,i,j)  A_ij -= L_ik L_jk^T, k < j <= i              (FP64 DMMA.8x8x4)
// The right-hand side rides along as a bordered row of 1x64 tiles (i = T), so
// the forward substitution y = L^-1 b falls out of the same DAG. Every tile
// has a state counter (= updates applied); a task waits until its inputs'
// states are final and its target's state equals its panel k, so updates land
// in k order (bitwise deterministic). Tasks are queued with lookahead 1:
//   P(k), S(.,k), U(k-1,.,j>=k+1), U(k,.,k+1), P(k+1), ...
// so the panel chain P -> S -> U(next column) overlaps the previous panel's
// bulk update. All waits point backwards in the queue and all CTAs are
// co-resident (cooperative launch), so the scheme cannot deadlock.
// k_trsv_back then runs the backward substitution as a flag wavefront.
// A non-positive pivot is reported in *status (column + 1); the caller then
// falls back to the eigen/pinv path.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

namespace rtb {

namespace {
constexpr int NB = 64;
constexpr int LDT = NB + 4;  // DMMA operand tiles
constexpr int LDW = NB + 4;  // potrf work tile (also the second row-task buffer)
constexpr int kThreads = 256;
enum { TP = 0, TS = 1, TU = 2, TR = 3 };  // TR: row task U(k, i, j = from..)

struct CholWork {
  double* linv;   // [T][64*64]
  double* bw;     // [T*64] working copy of b (border row)
  double* y;      // [T*64]
  double* x;      // [T*64]
  int* state;     // [(T+1)(T+2)/2] tile (i,j) update counters, row T = border
  int* xflag;     // [T]
  const int4* tasks;  // (type, k, i, j)
  int* counter;   // [2]
  unsigned long long* trace;  // optional [ntasks][4]: grab, ready, end (ns), smid
  volatile int* progress;     // optional host-mapped debug markers
  int T, ntasks;
};

unsigned long long* g_trace = nullptr;  // set by chol_set_trace (profiling tools)
volatile int* g_progress = nullptr;

template <typename F>
size_t carve(int d, F&& take) {
  const int T = (d + NB - 1) / NB;
  size_t off = 0;
  auto t = [&](size_t b) {
    take(off);
    off += (b + 255) & ~size_t(255);
  };
  t((size_t)T * NB * NB * 8);
  t((size_t)T * NB * 8);
  t((size_t)T * NB * 8);
  t((size_t)T * NB * 8);
  t((size_t)((T + 1) * (T + 2) / 2) * 4);
  t((size_t)T * 4);
  t(64);
  return off;
}

CholWork layout(int d, void* base) {
  CholWork w{};
  char* p = static_cast<char*>(base);
  int k = 0;
  carve(d, [&](size_t off) {
    void* q = p + off;
    switch (k++) {
      case 0: w.linv = (double*)q; break;
      case 1: w.bw = (double*)q; break;
      case 2: w.y = (double*)q; break;
      case 3: w.x = (double*)q; break;
      case 4: w.state = (int*)q; break;
      case 5: w.xflag = (int*)q; break;
      case 6: w.counter = (int*)q; break;
    }
  });
  w.T = (d + NB - 1) / NB;
  return w;
}

// Task queue (see the header comment). Pf(k) = {S(k,k-1), U(k-1,k,k), potrf(k)}.
// Every task only waits on tasks queued before it.
std::vector<int4> build_tasks(int T) {
  std::vector<int4> q;
  auto P = [&](int) {};  // the panel chain Pf(k) runs on CTA 0, outside the queue
  auto S = [&](int k, int from) {  // S(i,k) for tile rows i >= from, plus the border row
    for (int i = from; i < T; ++i) q.push_back(make_int4(TS, k, i, k));
    q.push_back(make_int4(TS, k, T, k));
  };
  auto Ucol = [&](int k, int j, int from) {  // U(k, i, j) for i = from..T-1 and the border
    for (int i = from; i < T; ++i) q.push_back(make_int4(TU, k, i, j));
    q.push_back(make_int4(TU, k, T, j));
  };
  P(0);
  if (T > 1) P(1);
  S(0, 2);
  if (T > 1) Ucol(0, 1, 2);
  for (int k = 1; k < T; ++k) {
    if (k + 1 < T) {
      Ucol(k - 1, k + 1, k + 1);  // column k+1 from panel k-1 (incl. its diagonal)
      P(k + 1);
    }
    S(k, k + 2);
    if (k + 1 < T) Ucol(k, k + 1, k + 2);
    if (k + 2 < T) {  // bulk of panel k-1: one row task per tile row (longest first)
      for (int i = T - 1; i >= k + 2; --i) q.push_back(make_int4(TR, k - 1, i, k + 2));
      q.push_back(make_int4(TR, k - 1, T, k + 2));
    }
  }
  return q;
}

__device__ __forceinline__ int tile_id(int i, int j) { return i * (i + 1) / 2 + j; }

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// Spin until *f >= v (acquire loads: later reads see the producer's data).
// Watchdog: after ~2 s of device time the wait gives up, records (flag index,
// value, wanted) in dbg[0..2], sets *abort and returns, so a scheduling bug can
// never hang the GPU (the caller sees status -2).
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_ge(const int* f, int v, int* abort_flag = nullptr,
                                        int* dbg = nullptr, const int* base = nullptr) {
  if (ld_acquire(f) >= v) return;
  const long long t0 = clock64();
  while (ld_acquire(f) < v) {
    __nanosleep(20);
    if (abort_flag) {
      if (ld_acquire(abort_flag)) return;
      if (clock64() - t0 > 4000000000LL) {
        if (atomicCAS(abort_flag, 0, 1) == 0 && dbg) {
          dbg[0] = (int)(f - base);
          dbg[1] = ld_acquire(f);
          dbg[2] = v;
        }
        return;
      }
    }
  }
}

// Callers: all threads store, __syncthreads(), then thread 0 publishes; the
// gpu-scope fence after the CTA barrier orders the whole CTA's stores
// (cumulativity) before the flag.
__device__ __forceinline__ void publish(int* f, int v) {
  __threadfence();
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
}  // namespace

size_t chol_work_bytes(int d) { return carve(d, [](size_t) {}); }

void chol_set_trace(unsigned long long* trace) { g_trace = trace; }
void chol_set_progress(volatile int* p) { g_progress = p; }
void chol_debug(int d, void* work, int* out4) {
  CholWork w = layout(d, work);
  RTB_CUDA(cudaMemcpy(out4, w.counter + 1, 16, cudaMemcpyDeviceToHost));
}
int chol_task_count(int d) {
  const int T = (d + NB - 1) / NB;
  return (int)build_tasks(T).size() + T;  // queued tasks + the CTA-0 panel chain
}
void chol_task_table(int d, int* out4) {
  const int T = (d + NB - 1) / NB;
  std::vector<int4> q = build_tasks(T);
  for (int k = 0; k < T; ++k) q.push_back(make_int4(TP, k, k, k));
  for (size_t t = 0; t < q.size(); ++t) {
    out4[4 * t] = q[t].x;
    out4[4 * t + 1] = q[t].y;
    out4[4 * t + 2] = q[t].z;
    out4[4 * t + 3] = q[t].w;
  }
}

__global__ void k_chol_init(CholWork w, const double* b, int d) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  if (t < 8) w.counter[t] = 0;
  const int T = w.T;
  const int ns = (T + 1) * (T + 2) / 2;
  for (int e = t; e < ns; e += stride) w.state[e] = 0;
  for (int e = t; e < T; e += stride) w.xflag[e] = 0;
  for (int e = t; e < T * NB; e += stride) w.bw[e] = e < d ? b[e] : 0.0;
}

// acc (64x64 fragments of this thread) +-= ta * tb^T over one 64-wide k chunk
__device__ __forceinline__ void mma_tile(double (&acc)[2][4][2], const double (*ta)[LDT],
                                         const double (*tb)[LDT], int mbase, int nbase, int g,
                                         int t4, bool subtract) {
#pragma unroll
  for (int ks = 0; ks < NB / 4; ++ks) {
    double af[2], bf[4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const double v = ta[mbase + mt * 8 + g][ks * 4 + t4];
      af[mt] = subtract ? -v : v;
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = tb[nbase + nt * 8 + g][ks * 4 + t4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
  }
}

// rows [r0, r0+64) x cols [c0, c0+64) of a (ld = d) into a padded smem tile (zero fill)
__device__ __forceinline__ void load_tile(double (*dst)[LDT], const double* a, int d, int r0,
                                          int c0, bool vec) {
  for (int e = threadIdx.x; e < NB * (NB / 2); e += kThreads) {
    const int r = e / (NB / 2), c = (e % (NB / 2)) * 2;
    const int gr = r0 + r, gc = c0 + c;
    if (vec) {
      const bool ok = gr < d && gc < d;
      cp_async16(&dst[r][c], ok ? a + (size_t)gr * d + gc : a, ok);
    } else {
      dst[r][c] = (gr < d && gc < d) ? __ldcg(a + (size_t)gr * d + gc) : 0.0;
      dst[r][c + 1] = (gr < d && gc + 1 < d) ? __ldcg(a + (size_t)gr * d + gc + 1) : 0.0;
    }
  }
}

__device__ __forceinline__ void load_acc(double (&acc)[2][4][2], const double* a, int d, int i0,
                                         int j0, int mbase, int nbase, int g, int t4) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int r = i0 + mbase + mt * 8 + g, cc = j0 + nbase + nt * 8 + 2 * t4;
      acc[mt][nt][0] = (r < d && cc < d) ? __ldcg(a + (size_t)r * d + cc) : 0.0;
      acc[mt][nt][1] = (r < d && cc + 1 < d) ? __ldcg(a + (size_t)r * d + cc + 1) : 0.0;
    }
}

__device__ __forceinline__ void store_acc(const double (&acc)[2][4][2], double* a, int d, int i0,
                                          int j0, int mbase, int nbase, int g, int t4) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int r = i0 + mbase + mt * 8 + g, cc = j0 + nbase + nt * 8 + 2 * t4;
      if (r < d && cc < d) a[(size_t)r * d + cc] = acc[mt][nt][0];
      if (r < d && cc + 1 < d) a[(size_t)r * d + cc + 1] = acc[mt][nt][1];
    }
}

// Blocked Cholesky of the 64x64 tile W (tw, lower part, identity-padded) into
// L (ta, lower) and Linv (tb, lower; caller zeroed it). Four 16-wide steps:
// warp 0 factors and inverts the 16x16 diagonal block (rows in registers,
// columns broadcast through shared memory), then all warps do the panel TRSM
// and the trailing update on the FP64 tensor cores; finally the off-diagonal
// blocks of Linv by block forward substitution, also on DMMA.
__device__ long long* g_ftclk = nullptr;  // profiling probe: phase clocks of factor_tile
#define FTCLK(slot) \
  if (g_ftclk && threadIdx.x == 0) g_ftclk[slot] = clock64();

__device__ void factor_tile(double (*tw)[LDW], double (*ta)[LDT], double (*tb)[LDT], int k0,
                            int* status, double* sdiag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  constexpr unsigned FULL = 0xffffffffu;
  FTCLK(0);
#pragma unroll 1
  for (int c0 = 0; c0 < NB; c0 += 16) {
    if (warp == 0) {
      const int r = lane & 15;
      double row[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) row[q] = tw[c0 + r][c0 + q];
      bool bad = false;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const double piv = __shfl_sync(FULL, row[c], c);
        bad |= (lane == c) && !(piv > 0.0);
        const double rs = rsqrt(piv);
        row[c] = (r == c) ? piv * rs : ((r > c) ? row[c] * rs : row[c]);
        if (lane < 16 && r >= c) ta[c0 + r][c0 + c] = row[c];
        if (lane == c) sdiag[c0 + c] = rs;
        __syncwarp();
#pragma unroll
        for (int l = 1; l < 16; ++l) {
          if (l > c) {
            const double llc = ta[c0 + l][c0 + c];  // broadcast read of L[l][c]
            row[l] = (r >= l) ? row[l] - row[c] * llc : row[l];
          }
        }
      }
      if (bad) atomicCAS(status, 0, k0 + c0 + lane + 1);
      if (lane < 16) {
#pragma unroll
        for (int q = 1; q < 16; ++q)
          if (q > r) ta[c0 + r][c0 + q] = 0.0;
      }
      __syncwarp();
      if (g_ftclk && lane == 0) g_ftclk[16 + c0 / 16] = clock64();
      // inverse of the 16x16 block, column col = lane & 15
      const int col = r;
      double x[16];
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        double s0 = (rr == col) ? 1.0 : 0.0, s1 = 0.0;
#pragma unroll
        for (int l = 0; l < 15; ++l) {
          if (l < rr) {
            const double lv = ta[c0 + rr][c0 + l];
            if (l & 1) s1 -= lv * x[l];
            else s0 -= lv * x[l];
          }
        }
        x[rr] = (rr >= col) ? (s0 + s1) * sdiag[c0 + rr] : 0.0;
      }
      if (lane < 16) {
#pragma unroll
        for (int q = 0; q < 16; ++q) tb[c0 + q][c0 + col] = x[q];
      }
    }
    __syncthreads();
    FTCLK(1 + 3 * (c0 / 16));
    if (c0 + 16 < NB) {
      const int r0 = c0 + 16, R = NB - r0;
      // panel TRSM on DMMA: L[r0+m][c0+n] = sum_q W[r0+m][c0+q] Linv16[n][q]
      if (warp < R / 8) {
        const int m0 = warp * 8;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          double c0v = 0.0, c1v = 0.0;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            dmma_8x8x4(c0v, c1v, tw[r0 + m0 + g][c0 + ks * 4 + t4],
                       tb[c0 + nt * 8 + g][c0 + ks * 4 + t4]);
          ta[r0 + m0 + g][c0 + nt * 8 + 2 * t4] = c0v;
          ta[r0 + m0 + g][c0 + nt * 8 + 2 * t4 + 1] = c1v;
        }
      }
      __syncthreads();
      FTCLK(2 + 3 * (c0 / 16));
      // trailing update of the lower 8x8 tiles on DMMA: W -= L_p L_p^T
      const int mt_n = R / 8;
      const int ntiles = mt_n * (mt_n + 1) / 2;
      for (int tI = warp; tI < ntiles; tI += kThreads / 32) {
        int mi = 0, rem = tI;
        while (rem > mi) {
          rem -= mi + 1;
          ++mi;
        }
        const int ni = rem;
        double c0v = tw[r0 + mi * 8 + g][r0 + ni * 8 + 2 * t4];
        double c1v = tw[r0 + mi * 8 + g][r0 + ni * 8 + 2 * t4 + 1];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          dmma_8x8x4(c0v, c1v, -ta[r0 + mi * 8 + g][c0 + ks * 4 + t4],
                     ta[r0 + ni * 8 + g][c0 + ks * 4 + t4]);
        tw[r0 + mi * 8 + g][r0 + ni * 8 + 2 * t4] = c0v;
        tw[r0 + mi * 8 + g][r0 + ni * 8 + 2 * t4 + 1] = c1v;
      }
      __syncthreads();
      FTCLK(3 + 3 * (c0 / 16));
    }
  }
  // off-diagonal blocks of Linv on DMMA:
  //   T_J = sum_{K=J}^{I-1} L[I][K] Linv[K][J];  Linv[I][J] = -Linv[I][I] T_J
#pragma unroll 1
  for (int I = 1; I < 4; ++I) {
    for (int pidx = warp; pidx < I * 4; pidx += kThreads / 32) {
      const int J = pidx >> 2, mt = (pidx >> 1) & 1, nt = pidx & 1;
      double c0v = 0.0, c1v = 0.0;
      for (int K = J; K < I; ++K)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          dmma_8x8x4(c0v, c1v, ta[16 * I + mt * 8 + g][16 * K + ks * 4 + t4],
                     tb[16 * K + ks * 4 + t4][16 * J + nt * 8 + g]);
      tw[16 * I + mt * 8 + g][16 * J + nt * 8 + 2 * t4] = c0v;
      tw[16 * I + mt * 8 + g][16 * J + nt * 8 + 2 * t4 + 1] = c1v;
    }
    __syncthreads();
    for (int pidx = warp; pidx < I * 4; pidx += kThreads / 32) {
      const int J = pidx >> 2, mt = (pidx >> 1) & 1, nt = pidx & 1;
      double c0v = 0.0, c1v = 0.0;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        dmma_8x8x4(c0v, c1v, tb[16 * I + mt * 8 + g][16 * I + ks * 4 + t4],
                   tw[16 * I + ks * 4 + t4][16 * J + nt * 8 + g]);
      tb[16 * I + mt * 8 + g][16 * J + nt * 8 + 2 * t4] = -c0v;
      tb[16 * I + mt * 8 + g][16 * J + nt * 8 + 2 * t4 + 1] = -c1v;
    }
    __syncthreads();
  }
  FTCLK(13);
}

#define WAIT(f, v) wait_ge((f), (v), &w.counter[1], w.counter + 2, w.state)
__global__ void __launch_bounds__(kThreads, 1) k_chol_dag(double* a, int d, CholWork w,
                                                          int* status) {
  extern __shared__ __align__(16) double smem[];
  double(*ta)[LDT] = reinterpret_cast<double(*)[LDT]>(smem);
  double(*tb)[LDT] = reinterpret_cast<double(*)[LDT]>(smem + NB * LDT);
  double(*tw)[LDW] = reinterpret_cast<double(*)[LDW]>(smem + 2 * NB * LDT);
  __shared__ int s_task;
  __shared__ double s_diag[NB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int mbase = 16 * (warp >> 1), nbase = 32 * (warp & 1);
  const int T = w.T;
  const bool vec = (d % 2) == 0;

  int chain_k = 0;  // CTA 0: next panel of the Pf chain
  for (;;) {
    int task, type, k, i, j;
    if (blockIdx.x == 0) {
      if (chain_k >= T) break;
      task = w.ntasks + chain_k;  // trace slot after the queued tasks
      type = TP;
      k = i = j = chain_k++;
    } else {
      if (tid == 0) s_task = atomicAdd(&w.counter[0], 1);
      __syncthreads();
      task = s_task;
      __syncthreads();
      if (task >= w.ntasks) break;
      const int4 tk = w.tasks[task];
      type = tk.x;
      k = tk.y;
      i = tk.z;
      j = tk.w;
    }
    if (w.progress && tid == 0) {
      w.progress[0] = task + 1;
      w.progress[4 + (blockIdx.x & 255)] = task + 1;
    }
    if (w.trace && tid == 0) {
      w.trace[4 * task + 0] = gtime();
      w.trace[4 * task + 3] = smid();
    }
    const int k0 = k * NB, i0 = i * NB, j0 = j * NB;

    if (type == TR) {
      // ---- row task: A_ij -= L_ik L_jk^T for j = j..last, L_ik kept in smem,
      //      L_jk double-buffered (tb / tw) ----
      const int jlast = (i == T) ? T - 1 : i;
      if (i == T) {
        const int c = tid >> 2, q = tid & 3;
        if (tid == 0) {
          WAIT(&w.state[tile_id(T, k)], k + 1);  // y_k
          if (w.trace) w.trace[4 * task + 1] = gtime();
        }
        __syncthreads();
        for (int jj = j; jj <= jlast; ++jj) {
          if (tid == 0) {
            WAIT(&w.state[tile_id(jj, k)], k + 1);
            WAIT(&w.state[tile_id(T, jj)], k);
          }
          __syncthreads();
          double v = 0.0;
          const int row = jj * NB + c;
          if (row < d) {
            const double* L = a + (size_t)row * d + k0;
            for (int l = q * 16; l < q * 16 + 16; ++l) v += __ldcg(L + l) * __ldcg(w.y + k0 + l);
          }
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          if (q == 0) w.bw[jj * NB + c] = __ldcg(w.bw + jj * NB + c) - v;
          __syncthreads();
          if (tid == 0) publish(&w.state[tile_id(T, jj)], k + 1);
        }
      } else {
        double(*buf[2])[LDT] = {tb, reinterpret_cast<double(*)[LDT]>(&tw[0][0])};
        double(*cbuf[2])[LDT] = {reinterpret_cast<double(*)[LDT]>(smem + 3 * NB * LDT),
                                 reinterpret_cast<double(*)[LDT]>(smem + 4 * NB * LDT)};
        if (tid == 0) {
          WAIT(&w.state[tile_id(i, k)], k + 1);
          WAIT(&w.state[tile_id(j, k)], k + 1);
          WAIT(&w.state[tile_id(i, j)], k);
          if (w.trace) w.trace[4 * task + 1] = gtime();
        }
        __syncthreads();
        load_tile(ta, a, d, i0, k0, vec);
        load_tile(buf[0], a, d, j0, k0, vec);
        load_tile(cbuf[0], a, d, i0, j0, vec);
        cp_async_commit();
        for (int jj = j; jj <= jlast; ++jj) {
          const int cur = (jj - j) & 1;
          if (jj + 1 <= jlast) {  // prefetch tile jj+1 (its inputs are usually ready)
            if (tid == 0) {
              WAIT(&w.state[tile_id(jj + 1, k)], k + 1);
              WAIT(&w.state[tile_id(i, jj + 1)], k);
            }
            __syncthreads();
            load_tile(buf[cur ^ 1], a, d, (jj + 1) * NB, k0, vec);
            load_tile(cbuf[cur ^ 1], a, d, i0, (jj + 1) * NB, vec);
          }
          cp_async_commit();
          cp_async_wait<1>();
          __syncthreads();
          double acc[2][4][2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              const double2 v = *reinterpret_cast<const double2*>(
                  &cbuf[cur][mbase + mt * 8 + g][nbase + nt * 8 + 2 * t4]);
              acc[mt][nt][0] = v.x;
              acc[mt][nt][1] = v.y;
            }
          mma_tile(acc, ta, jj == i ? ta : buf[cur], mbase, nbase, g, t4, true);
          // publish the previous tile (its stores preceded the last barrier)
          if (jj > j && tid == kThreads - 32) publish(&w.state[tile_id(i, jj - 1)], k + 1);
          store_acc(acc, a, d, i0, jj * NB, mbase, nbase, g, t4);
          __syncthreads();
        }
        if (tid == kThreads - 32) publish(&w.state[tile_id(i, jlast)], k + 1);
        cp_async_wait<0>();
      }
      if (tid == 0 && w.trace) w.trace[4 * task + 2] = gtime();
      __syncthreads();
      continue;
    }

    if (type == TU) {
      // ---- A_ij -= L_ik L_jk^T (border: b_j -= L_jk y_k) ----
      if (tid == 0) {
        WAIT(&w.state[tile_id(j, k)], k + 1);
        WAIT(&w.state[tile_id(i, k)], k + 1);
        WAIT(&w.state[tile_id(i, j)], k);
        if (w.trace) w.trace[4 * task + 1] = gtime();
      }
      __syncthreads();
      if (i == T) {
        const int c = tid >> 2, q = tid & 3;
        double v = 0.0;
        if (j0 + c < d) {
          const double* L = a + (size_t)(j0 + c) * d + k0;
          for (int l = q * 16; l < q * 16 + 16; ++l) v += __ldcg(L + l) * __ldcg(w.y + k0 + l);
        }
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (q == 0) w.bw[j0 + c] = __ldcg(w.bw + j0 + c) - v;
      } else {
        load_tile(ta, a, d, i0, k0, vec);
        if (i != j) load_tile(tb, a, d, j0, k0, vec);
        cp_async_commit();
        double acc[2][4][2];
        load_acc(acc, a, d, i0, j0, mbase, nbase, g, t4);
        cp_async_wait<0>();
        __syncthreads();
        mma_tile(acc, ta, i == j ? ta : tb, mbase, nbase, g, t4, true);
        store_acc(acc, a, d, i0, j0, mbase, nbase, g, t4);
      }
      __syncthreads();
      if (tid == 0) {
        publish(&w.state[tile_id(i, j)], k + 1);
        if (w.trace) w.trace[4 * task + 2] = gtime();
      }
      continue;
    }

    if (type == TS) {
      // ---- L_ik = A_ik Linv_kk^T (border: y_k = Linv_kk b_k) ----
      if (tid == 0) {
        WAIT(&w.state[tile_id(k, k)], k + 1);
        WAIT(&w.state[tile_id(i, k)], k);
        if (w.trace) w.trace[4 * task + 1] = gtime();
      }
      __syncthreads();
      const double* iv = w.linv + (size_t)k * NB * NB;
      if (i == T) {
        const int c = tid >> 2, q = tid & 3;
        double v = 0.0;
        for (int l = q * 16; l < q * 16 + 16; ++l) v += __ldcg(iv + c * NB + l) * __ldcg(w.bw + k0 + l);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (q == 0) w.y[k0 + c] = v;
      } else {
        for (int e = tid; e < NB * (NB / 2); e += kThreads) {
          const int r = e / (NB / 2), c = (e % (NB / 2)) * 2;
          cp_async16(&tb[r][c], iv + r * NB + c, true);
        }
        cp_async_commit();
        load_tile(ta, a, d, i0, k0, vec);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        double acc[2][4][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        mma_tile(acc, ta, tb, mbase, nbase, g, t4, false);
        store_acc(acc, a, d, i0, k0, mbase, nbase, g, t4);
      }
      __syncthreads();
      if (tid == 0) {
        publish(&w.state[tile_id(i, k)], k + 1);
        if (w.trace) w.trace[4 * task + 2] = gtime();
      }
      continue;
    }

    // ---- Pf(k): [S(k,k-1), U(k-1,k,k) fused] + Cholesky of tile (k,k) ----
    const int nb = min(NB, d - k0);
    if (k > 0) {
      const int p0 = (k - 1) * NB;
      if (tid == 0) {
        WAIT(&w.state[tile_id(k, k - 1)], k - 1);
        WAIT(&w.state[tile_id(k, k)], k - 1);
      }
      __syncthreads();
      load_tile(ta, a, d, k0, p0, vec);  // A_{k,k-1}
      cp_async_commit();
      double acc[2][4][2];
      load_acc(acc, a, d, k0, k0, mbase, nbase, g, t4);  // A_kk
      if (tid == 0) {
        WAIT(&w.state[tile_id(k - 1, k - 1)], k);  // Linv_{k-1}
        if (w.trace) w.trace[4 * task + 1] = gtime();
      }
      __syncthreads();
      {
        const double* iv = w.linv + (size_t)(k - 1) * NB * NB;
        for (int e = tid; e < NB * (NB / 2); e += kThreads) {
          const int r = e / (NB / 2), c = (e % (NB / 2)) * 2;
          cp_async16(&tb[r][c], iv + r * NB + c, true);
        }
        cp_async_commit();
      }
      cp_async_wait<0>();
      __syncthreads();
      double lk[2][4][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) lk[mt][nt][0] = lk[mt][nt][1] = 0.0;
      mma_tile(lk, ta, tb, mbase, nbase, g, t4, false);  // L_{k,k-1} = A Linv^T
      store_acc(lk, a, d, k0, p0, mbase, nbase, g, t4);
      __syncthreads();
      if (tid == 0) publish(&w.state[tile_id(k, k - 1)], k);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int r = mbase + mt * 8 + g, cc = nbase + nt * 8 + 2 * t4;
          ta[r][cc] = lk[mt][nt][0];
          ta[r][cc + 1] = lk[mt][nt][1];
        }
      __syncthreads();
      mma_tile(acc, ta, ta, mbase, nbase, g, t4, true);  // A_kk -= L L^T
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int r = mbase + mt * 8 + g, cc = nbase + nt * 8 + 2 * t4;
          tw[r][cc] = acc[mt][nt][0];
          tw[r][cc + 1] = acc[mt][nt][1];
        }
      __syncthreads();
    } else {
      if (tid == 0 && w.trace) w.trace[4 * task + 1] = gtime();
      for (int e = tid; e < NB * NB; e += kThreads) {
        const int r = e / NB, c = e % NB;
        tw[r][c] = (r < nb && c <= r) ? __ldcg(a + (size_t)(k0 + r) * d + k0 + c) : 0.0;
      }
      __syncthreads();
    }
    // identity padding beyond the matrix edge (partial last tile)
    for (int e = tid; e < NB * NB; e += kThreads) {
      const int r = e / NB, c = e % NB;
      if (r >= nb || c >= nb) tw[r][c] = (r == c) ? 1.0 : 0.0;
      tb[r][c] = 0.0;
    }
    __syncthreads();
    if (w.progress && tid == 0) w.progress[2] = 1000 + k;
    factor_tile(tw, ta, tb, k0, status, s_diag);
    if (w.progress && tid == 0) w.progress[2] = 2000 + k;
    double* ivw = w.linv + (size_t)k * NB * NB;
    for (int e = tid; e < NB * NB; e += kThreads) {
      const int r = e / NB, c = e % NB;
      ivw[e] = c <= r ? tb[r][c] : 0.0;
      if (r < nb && c <= r) a[(size_t)(k0 + r) * d + k0 + c] = ta[r][c];
    }
    __syncthreads();
    if (tid == 0) {
      publish(&w.state[tile_id(k, k)], k + 1);
      if (w.trace) w.trace[4 * task + 2] = gtime();
    }
  }
}

#undef WAIT

__global__ void k_chol_check(CholWork w, int* status) {
  if (w.progress && threadIdx.x == 0) w.progress[1] = 7;
  if (threadIdx.x == 0 && w.counter[1]) atomicCAS(status, 0, -2);  // watchdog fired
}

// Backward substitution L^T x = y as a wavefront: block c (64 unknowns) is
// owned by CTA (T-1-c) mod grid, blocks processed in descending order. The CTA
// streams L_kc (k > c) through a double-buffered smem tile -- those loads do not
// depend on x -- and subtracts L_kc^T x_k as each x_k is published; then
// x_c = Linv_cc^T (y_c - sum).
__global__ void __launch_bounds__(kThreads) k_trsv_back(const double* a, int d, CholWork w,
                                                        double* x_out, const int* status) {
  if (*status) return;
  extern __shared__ __align__(16) double bsm[];
  double(*lt[2])[LDT] = {reinterpret_cast<double(*)[LDT]>(bsm),
                         reinterpret_cast<double(*)[LDT]>(bsm + NB * LDT)};
  double(*iv)[LDT] = reinterpret_cast<double(*)[LDT]>(bsm + 2 * NB * LDT);
  __shared__ double v[NB];
  __shared__ double xk[NB];
  __shared__ double part[4][NB];
  const int tid = threadIdx.x;
  const int T = w.T;
  const bool vec = (d % 2) == 0;
  const int l = tid & (NB - 1), q = tid >> 6;  // 64 columns x 4 row groups
  for (int c = T - 1 - (int)blockIdx.x; c >= 0; c -= gridDim.x) {
    const int c0 = c * NB;
    {  // Linv_cc
      const double* src = w.linv + (size_t)c * NB * NB;
      for (int e = tid; e < NB * (NB / 2); e += kThreads) {
        const int r = e / (NB / 2), cc = (e % (NB / 2)) * 2;
        cp_async16(&iv[r][cc], src + r * NB + cc, true);
      }
    }
    if (T - 1 > c) load_tile(lt[0], a, d, (T - 1) * NB, c0, vec);
    cp_async_commit();
    double s = 0.0;
    for (int k = T - 1; k > c; --k) {
      const int cur = (T - 1 - k) & 1;
      if (k - 1 > c) load_tile(lt[cur ^ 1], a, d, (k - 1) * NB, c0, vec);
      cp_async_commit();
      if (tid == 0) wait_ge(&w.xflag[k], 1, &w.counter[1], w.counter + 2, w.xflag);
      __syncthreads();
      if (tid < NB) xk[tid] = __ldcg(w.x + k * NB + tid);
      cp_async_wait<1>();
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 16; ++r) s += lt[cur][q * 16 + r][l] * xk[q * 16 + r];
      __syncthreads();
    }
    cp_async_wait<0>();
    part[q][l] = s;
    __syncthreads();
    if (tid < NB)
      v[tid] = (c0 + tid < d ? __ldcg(w.y + c0 + tid) : 0.0) -
               ((part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]));
    __syncthreads();
    // x[l] = sum_{r >= l} Linv[r][l] v[r]
    double xs = 0.0;
#pragma unroll
    for (int r = 0; r < 16; ++r) xs += iv[q * 16 + r][l] * v[q * 16 + r];
    part[q][l] = xs;
    __syncthreads();
    if (tid < NB) {
      const double xv = (part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]);
      w.x[c0 + tid] = xv;
      if (c0 + tid < d) x_out[c0 + tid] = xv;
    }
    __syncthreads();
    if (tid == 0) publish(&w.xflag[c], 1);
  }
}

void chol_solve(double* a, int d, double* b, int* status_dev, void* work, cudaStream_t st) {
  CholWork w = layout(d, work);
  int dev = 0, sms = 0;
  RTB_CUDA(cudaGetDevice(&dev));
  RTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // task queue, built once per (device, T) and kept resident
  static std::mutex mu;
  static std::map<std::pair<int, int>, std::pair<int4*, int>> queues;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(dev, w.T);
    auto it = queues.find(key);
    if (it == queues.end()) {
      std::vector<int4> q = build_tasks(w.T);
      int4* dq = nullptr;
      RTB_CUDA(cudaMalloc(&dq, q.size() * sizeof(int4)));
      RTB_CUDA(cudaMemcpy(dq, q.data(), q.size() * sizeof(int4), cudaMemcpyHostToDevice));
      it = queues.emplace(key, std::make_pair(dq, (int)q.size())).first;
    }
    w.tasks = it->second.first;
    w.ntasks = it->second.second;
  }
  w.trace = g_trace;
  w.progress = g_progress;
  RTB_CUDA(cudaMemsetAsync(status_dev, 0, sizeof(int), st));
  k_chol_init<<<kNumSMs, 256, 0, st>>>(w, b, d);
  RTB_LAUNCH_CHECK();
  const int smem = 5 * NB * LDT * sizeof(double);  // ta, tb, tw, 2 row-task C buffers
  set_max_smem(k_chol_dag, smem);
  int per_sm = 0;
  RTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chol_dag, kThreads, smem));
  if (per_sm < 1) throw Error(4, "chol: kernel does not fit on an SM");
  // CTA 0 runs the panel chain; at least one more CTA drains the queue
  const int grid = std::max(2, std::min(sms * per_sm, w.ntasks + 1));
  {
    int* sc = status_dev;
    void* args[] = {(void*)&a, (void*)&d, (void*)&w, (void*)&sc};
    RTB_CUDA(cudaLaunchCooperativeKernel((void*)k_chol_dag, grid, kThreads, args, smem, st));
    RTB_LAUNCH_CHECK();
  }
  k_chol_check<<<1, 32, 0, st>>>(w, status_dev);
  RTB_LAUNCH_CHECK();
  {
    const int bsmem = 3 * NB * LDT * sizeof(double);
    set_max_smem(k_trsv_back, bsmem);
    int per2 = 0;
    RTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_trsv_back, kThreads, bsmem));
    const int g2 = std::min(w.T, sms * std::max(per2, 1));
    const double* ac = a;
    const int* sc = status_dev;
    void* args[] = {(void*)&ac, (void*)&d, (void*)&w, (void*)&b, (void*)&sc};
    RTB_CUDA(cudaLaunchCooperativeKernel((void*)k_trsv_back, g2, kThreads, args, bsmem, st));
    RTB_LAUNCH_CHECK();
  }
}

}  // namespace rtb
