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
constexpr int LDW = NB + 1;  // potrf work tile (odd stride)
constexpr int kThreads = 256;
enum { TP = 0, TS = 1, TU = 2 };

struct CholWork {
  double* linv;   // [T][64*64]
  double* bw;     // [T*64] working copy of b (border row)
  double* y;      // [T*64]
  double* x;      // [T*64]
  int* state;     // [(T+1)(T+2)/2] tile (i,j) update counters, row T = border
  int* xflag;     // [T]
  const int4* tasks;  // (type, k, i, j)
  int* counter;   // [2]
  int T, ntasks;
};

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

// Task queue with lookahead 1 (see the header comment).
std::vector<int4> build_tasks(int T) {
  std::vector<int4> q;
  auto P = [&](int k) { q.push_back(make_int4(TP, k, k, k)); };
  auto S = [&](int k) {
    for (int i = k + 1; i <= T; ++i) q.push_back(make_int4(TS, k, i, k));  // i == T: border
  };
  auto Ucol = [&](int k, int j) {  // U(k, i, j) for i = j..T (T: border)
    for (int i = j; i <= T; ++i) q.push_back(make_int4(TU, k, i, j));
  };
  for (int k = 0; k < T; ++k) {
    P(k);
    S(k);
    if (k >= 1)
      for (int j = k + 1; j < T; ++j) Ucol(k - 1, j);
    if (k + 1 < T) Ucol(k, k + 1);
  }
  return q;
}

__device__ __forceinline__ int tile_id(int i, int j) { return i * (i + 1) / 2 + j; }

__device__ __forceinline__ void wait_ge(const int* f, int v) {
  if (atomicAdd(const_cast<int*>(f), 0) >= v) return;
  while (atomicAdd(const_cast<int*>(f), 0) < v) __nanosleep(32);
}

__device__ __forceinline__ void publish(int* f, int v) {
  __threadfence();
  atomicExch(f, v);
}
}  // namespace

size_t chol_work_bytes(int d) { return carve(d, [](size_t) {}); }

__global__ void k_chol_init(CholWork w, const double* b, int d) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  if (t == 0) {
    w.counter[0] = 0;
    w.counter[1] = 0;
  }
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

__global__ void __launch_bounds__(kThreads, 2) k_chol_dag(double* a, int d, CholWork w,
                                                          int* status) {
  extern __shared__ __align__(16) double smem[];
  double(*ta)[LDT] = reinterpret_cast<double(*)[LDT]>(smem);
  double(*tb)[LDT] = reinterpret_cast<double(*)[LDT]>(smem + NB * LDT);
  double(*tw)[LDW] = reinterpret_cast<double(*)[LDW]>(smem + 2 * NB * LDT);
  __shared__ int s_task;
  __shared__ double s_rd[NB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int mbase = 16 * (warp >> 1), nbase = 32 * (warp & 1);
  const int T = w.T;
  const bool vec = (d % 2) == 0;

  for (;;) {
    if (tid == 0) s_task = atomicAdd(&w.counter[0], 1);
    __syncthreads();
    const int task = s_task;
    __syncthreads();
    if (task >= w.ntasks) break;
    const int4 tk = w.tasks[task];
    const int type = tk.x, k = tk.y, i = tk.z, j = tk.w;
    const int k0 = k * NB, i0 = i * NB, j0 = j * NB;

    if (type == TU) {
      // ---- A_ij -= L_ik L_jk^T (border: b_j -= L_jk y_k) ----
      if (tid == 0) {
        wait_ge(&w.state[tile_id(j, k)], k + 1);
        wait_ge(&w.state[tile_id(i, k)], k + 1);
        wait_ge(&w.state[tile_id(i, j)], k);
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
      if (tid == 0) publish(&w.state[tile_id(i, j)], k + 1);
      continue;
    }

    if (type == TS) {
      // ---- L_ik = A_ik Linv_kk^T (border: y_k = Linv_kk b_k) ----
      if (tid == 0) {
        wait_ge(&w.state[tile_id(k, k)], k + 1);
        wait_ge(&w.state[tile_id(i, k)], k);
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
      if (tid == 0) publish(&w.state[tile_id(i, k)], k + 1);
      continue;
    }

    // ---- P(k): Cholesky of tile (k,k) + inverse ----
    if (tid == 0) wait_ge(&w.state[tile_id(k, k)], k);
    __syncthreads();
    const int nb = min(NB, d - k0);
    for (int e = tid; e < NB * NB; e += kThreads) {
      const int r = e / NB, c = e % NB;
      tw[r][c] = (r < nb && c <= r) ? __ldcg(a + (size_t)(k0 + r) * d + k0 + c) : 0.0;
    }
    __syncthreads();
    // right-looking, lazily scaled: W[r][l] -= W[r][c] W[l][c] / W[c][c];
    // L[r][c] = W[r][c] / sqrt(W[c][c]) goes to ta. One barrier per column.
    const int tr = tid >> 4, tl = tid & 15;
    for (int c = 0; c < nb; ++c) {
      const double p = tw[c][c];
      if (!(p > 0.0)) {
        if (tid == 0) atomicCAS(status, 0, k0 + c + 1);
      }
      const double sd = sqrt(p);
      const double pinv = 1.0 / p;
      if (tid < nb - c) {
        const int r = c + tid;
        ta[r][c] = r == c ? sd : tw[r][c] / sd;
      }
      for (int r = c + 1 + tr; r < nb; r += 16) {
        const double wr = tw[r][c] * pinv;
        for (int l = c + 1 + tl; l <= r; l += 16) tw[r][l] -= wr * tw[l][c];
      }
      __syncthreads();
    }
    // inverse of L (ta, lower) into tb: column col by 4 lanes
    if (tid < NB) s_rd[tid] = tid < nb ? 1.0 / ta[tid][tid] : 0.0;
    __syncthreads();
    {
      const int col = tid >> 2, q = tid & 3;
      for (int r = 0; r < NB; ++r) {
        double s = 0.0;
        if (r < nb && col < nb && r > col)
          for (int l = col + q; l < r; l += 4) s += ta[r][l] * tb[l][col];
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        double xr = 0.0;
        if (r < nb && col < nb && r >= col) xr = ((r == col ? 1.0 : 0.0) - s) * s_rd[r];
        if (q == 0) tb[r][col] = xr;
        __syncwarp();
      }
    }
    __syncthreads();
    double* ivw = w.linv + (size_t)k * NB * NB;
    for (int e = tid; e < NB * NB; e += kThreads) {
      const int r = e / NB, c = e % NB;
      ivw[e] = tb[r][c];
      if (r < nb && c <= r) a[(size_t)(k0 + r) * d + k0 + c] = ta[r][c];
    }
    __syncthreads();
    if (tid == 0) publish(&w.state[tile_id(k, k)], k + 1);
  }
}

// Backward substitution L^T x = y as a wavefront: block c (64 unknowns) is
// owned by CTA (T-1-c) mod grid, blocks processed in descending order; it
// subtracts L_kc^T x_k for every k > c as soon as x_k is published.
__global__ void __launch_bounds__(kThreads) k_trsv_back(const double* a, int d, CholWork w,
                                                        double* x_out, const int* status) {
  if (*status) return;
  __shared__ double v[NB];
  __shared__ double part[4][NB];
  const int tid = threadIdx.x;
  const int T = w.T;
  const int l = tid & (NB - 1), q = tid >> 6;  // 64 columns x 4 row groups
  for (int c = T - 1 - (int)blockIdx.x; c >= 0; c -= gridDim.x) {
    const int c0 = c * NB;
    double s = 0.0;
    for (int k = T - 1; k > c; --k) {
      if (tid == 0) wait_ge(&w.xflag[k], 1);
      __syncthreads();
      const int k0 = k * NB;
      if (c0 + l < d) {
        for (int r = q * 16; r < q * 16 + 16; ++r) {
          if (k0 + r < d) s += __ldcg(a + (size_t)(k0 + r) * d + c0 + l) * __ldcg(w.x + k0 + r);
        }
      }
    }
    part[q][l] = s;
    __syncthreads();
    if (tid < NB)
      v[tid] = (c0 + tid < d ? __ldcg(w.y + c0 + tid) : 0.0) -
               ((part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]));
    __syncthreads();
    // x_c = Linv_cc^T v : x[l] = sum_{r >= l} Linv[r][l] v[r]
    const double* iv = w.linv + (size_t)c * NB * NB;
    double xs = 0.0;
    for (int r = q * 16; r < q * 16 + 16; ++r) xs += __ldcg(iv + r * NB + l) * v[r];
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
  RTB_CUDA(cudaMemsetAsync(status_dev, 0, sizeof(int), st));
  k_chol_init<<<kNumSMs, 256, 0, st>>>(w, b, d);
  RTB_LAUNCH_CHECK();
  const int smem = (2 * NB * LDT + NB * LDW) * sizeof(double);
  RTB_CUDA(cudaFuncSetAttribute(k_chol_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  RTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chol_dag, kThreads, smem));
  if (per_sm < 1) throw Error(4, "chol: kernel does not fit on an SM");
  const int grid = std::min(sms * per_sm, w.ntasks);
  {
    int* sc = status_dev;
    void* args[] = {(void*)&a, (void*)&d, (void*)&w, (void*)&sc};
    RTB_CUDA(cudaLaunchCooperativeKernel((void*)k_chol_dag, grid, kThreads, args, smem, st));
    RTB_LAUNCH_CHECK();
  }
  {
    int per2 = 0;
    RTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_trsv_back, kThreads, 0));
    const int g2 = std::min(w.T, sms * std::max(per2, 1));
    const double* ac = a;
    const int* sc = status_dev;
    void* args[] = {(void*)&ac, (void*)&d, (void*)&w, (void*)&b, (void*)&sc};
    RTB_CUDA(cudaLaunchCooperativeKernel((void*)k_trsv_back, g2, kThreads, args, 0, st));
    RTB_LAUNCH_CHECK();
  }
}

}  // namespace rtb
