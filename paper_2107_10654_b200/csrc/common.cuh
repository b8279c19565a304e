// common.cuh -- shared device helpers for the sm_100a kernels.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include <stdexcept>
#include <string>

namespace rtb {

// Host-side error type carrying an rtucker_status code.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define RTB_CUDA(call)                                                                \
  do {                                                                                \
    cudaError_t err_ = (call);                                                        \
    if (err_ != cudaSuccess)                                                          \
      throw ::rtb::Error(4, std::string("CUDA error: ") + cudaGetErrorString(err_) +  \
                                " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// Every launch site ends with RTB_LAUNCH_CHECK(): it checks the launch and
// counts it (rtucker_b200_launch_count exposes the total for bench.py).
std::atomic<unsigned long long>& launch_counter();

// Per-variant launch counters for the headline kernels (tests assert which kernel a
// configuration actually ran; rtucker_b200_variant_count).
void count_variant(const char* name);
unsigned long long variant_count(const char* name);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel): the
// attribute is per device, so the cache is keyed by the current device ordinal.
void set_max_smem_impl(const void* fn, int bytes);
template <typename F>
inline void set_max_smem(F* fn, int bytes) {
  set_max_smem_impl(reinterpret_cast<const void*>(fn), bytes);
}
#define RTB_LAUNCH_CHECK()          \
  do {                              \
    RTB_CUDA(cudaGetLastError());   \
    ++::rtb::launch_counter();      \
  } while (0)

constexpr int kNumSMs = 148;
constexpr int kMaxOrder = 8;

// vech index of the unordered pair (a <= b) among n items (row-major upper
// triangle) and its inverse; the Gram of Kronecker rows is indexed by these.
__host__ __device__ __forceinline__ int upper_pair(int a, int b, int n) {
  return a * n - a * (a - 1) / 2 + (b - a);
}
__host__ __device__ __forceinline__ void pair_of(int u, int n, int& a, int& b) {
  a = 0;
  while (u >= n - a) {
    u -= n - a;
    ++a;
  }
  b = a + u;
}

// ---- SplitMix64 (ref rng.hpp:12-62) in counter form: output k of a stream
// seeded with `seed` is mix(seed + (k+1)*gamma). ----
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t sm_at(uint64_t seed, uint64_t k) {
  return sm_mix(seed + (k + 1) * kGamma);
}
// next_double(): top 53 bits times 2^-53, exact (ref rng.hpp:24-26).
__device__ __forceinline__ double u64_to_unit(uint64_t u) {
  return __dmul_rn(static_cast<double>(u >> 11), 0x1.0p-53);
}

// ---- FP64 tensor-core MMA: D(8x8) += A(8x4) * B(4x8), one DMMA.8x8x4 ----
// Fragment ownership (lane l, g = l>>2, t = l&3):
//   A: a = A[g][t]   B: b = B[t][g]   C/D: c0 = C[g][2t], c1 = C[g][2t+1]
// (not volatile: the asm has outputs, so the compiler may schedule loads around it)
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// m16n8k16 f64 (CuTe SM90_16x8x16_F64F64F64F64_TN layouts), g = lane / 4, t = lane % 4:
//   a[v] = A[g + 8 (v & 1)][t + 4 (v >> 1)]   (v < 8, A is 16 x 16 row-major M x K)
//   b[v] = B[t + 4 v][g]                       (v < 4, B is 16 x 8, K x N)
//   c[v] = C[g + 8 (v >> 1)][2 t + (v & 1)]    (v < 4, C is 16 x 8)
__device__ __forceinline__ void dmma_16x8x16(double (&c)[4], const double (&a)[8],
                                             const double (&b)[4]) {
  asm("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// ---- cp.async (LDGSTS) with zero fill: copies `src_bytes` (0 or the full
// size) and zero-fills the rest of the destination. ----
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(gmem),
               "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// ---- TMA bulk copies (cp.async.bulk, 1-D, no tensor map) + mbarrier ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// make the inits (and prior generic smem writes) visible to the async proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, 16-byte aligned ends)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 2-D tensor-map TMA load (cp.async.bulk.tensor): box at (c0 innermost, c1) -> smem, completing
// on `bar`; `map` is the address of a __grid_constant__ CUtensorMap kernel parameter
__device__ __forceinline__ void tma_load_2d(void* dst, const void* map, int c0, int c1,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar))
      : "memory");
}
// this thread's prior cp.async copies arrive on `bar` when they complete (counts
// as one of the barrier's expected arrivals)
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <typename T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) {
  return (a + b - 1) / b;
}

// Deterministic block-wide sum (fixed tree order for a fixed blockDim).
template <int kThreads>
__device__ __forceinline__ double block_sum(double v, double* smem) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < kThreads / 32 ? smem[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0 (and all of warp 0)
}

}  // namespace rtb
