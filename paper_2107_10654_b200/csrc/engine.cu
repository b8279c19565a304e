// engine.cu -- device-resident sketched Tucker-ALS (ref tucker.cpp:192-276).
//
// One sweep, everything on the GPU, X read from HBM twice:
//   F_n, n < N : Y = T x_{m != n, N} A_m^T  (T = X x_N A_N^T, cached from the
//                previous loss pass), M = Y_(n) G_(n)^T, KK^T from the factor
//                Grams, A_n = M pinv(KK^T + lambda I)            (tucker.cpp:70-89)
//   F_N        : Y = X x_1 A_1^T x_2 ...  (one strided pass over X)
//   Core       : sketched (scores -> parallel draw decode -> Kronecker-factored
//                Gram/RHS -> Cholesky)                           (tucker.cpp:141-166)
//                or exact (factor SVD bases, 2 TTM chains)       (tucker.cpp:91-129)
//   Loss       : fused pass: residual of X against G x_n A_n rebuilt in
//                registers + next sweep's T                      (tucker.cpp:216-229)
#include "engine.h"

#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "kernels.h"

namespace rtb {

// ---------------------------------------------------------------------------
// streams and buffers

namespace {
thread_local cudaStream_t t_stream = nullptr;
std::mutex g_stream_mu;
std::map<int, cudaStream_t> g_default_streams;
}  // namespace

// per-device stream for parallel graph branches (Engine::fork); never destroyed
cudaStream_t side_stream(int k = 0) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, cudaStream_t> streams;
  int dev = 0;
  RTB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = streams.find({dev, k});
  if (it != streams.end()) return it->second;
  cudaStream_t s;
  RTB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  streams[{dev, k}] = s;
  return s;
}

cudaStream_t current_stream() {
  if (t_stream) return t_stream;
  int dev = 0;
  RTB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_stream_mu);
  auto it = g_default_streams.find(dev);
  if (it != g_default_streams.end()) return it->second;
  cudaStream_t s;
  RTB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // keep freed pool memory cached across runs (no cudaMalloc per call)
  cudaMemPool_t pool;
  RTB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = UINT64_MAX;
  RTB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  g_default_streams[dev] = s;
  return s;
}

void set_stream(cudaStream_t s) { t_stream = s; }

std::atomic<unsigned long long>& launch_counter() {
  static std::atomic<unsigned long long> n{0};
  return n;
}

namespace {
std::mutex g_variant_mu;
std::map<std::string, unsigned long long>& variants() {
  static std::map<std::string, unsigned long long> m;
  return m;
}
}  // namespace
void count_variant(const char* name) {
  std::lock_guard<std::mutex> lk(g_variant_mu);
  ++variants()[name];
}
unsigned long long variant_count(const char* name) {
  std::lock_guard<std::mutex> lk(g_variant_mu);
  auto it = variants().find(name);
  return it == variants().end() ? 0 : it->second;
}

void set_max_smem_impl(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  RTB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{dev, fn}];
  if (have >= bytes) return;
  RTB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

DevBuf::DevBuf(size_t b, cudaStream_t s) { ensure(b, s); }
DevBuf::~DevBuf() {
  if (p) cudaFreeAsync(p, st);
}
DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
  if (this != &o) {
    if (p) cudaFreeAsync(p, st);
    p = o.p;
    bytes = o.bytes;
    st = o.st;
    o.p = nullptr;
    o.bytes = 0;
  }
  return *this;
}
// The stream-ordered allocator's default pool gives freed memory back to the driver at every
// synchronisation (release threshold 0), so each new job (engine) paid for fresh mappings: a
// C1 job spent ~2 ms of its ~8 in allocation and free. Keep freed memory in the pool instead
// (once per device; memory is still reused by the next allocation, not leaked).
static void keep_pool_memory() {
  static std::mutex mu;
  static std::map<int, bool> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return;
  done[dev] = true;
  static const bool off = std::getenv("RTB_POOL_RELEASE") != nullptr;  // experiments
  if (off) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

// Small pinned host slots (the core verdict each engine reads behind its core step). One
// cudaHostAlloc per process instead of one per engine: pinning and unpinning cost ~1 ms each
// (cudaFreeHost also synchronises the device), which a C1 job of 10 sweeps noticed.
static std::mutex g_pin_mu;
static std::vector<int*> g_pin_free;
int* pinned_slot() {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (g_pin_free.empty()) {
    constexpr int kSlots = 64, kInts = 16;
    int* base = nullptr;
    RTB_CUDA(cudaHostAlloc((void**)&base, (size_t)kSlots * kInts * sizeof(int),
                           cudaHostAllocDefault));
    for (int k = kSlots - 1; k >= 0; --k) g_pin_free.push_back(base + k * kInts);
  }
  int* p = g_pin_free.back();
  g_pin_free.pop_back();
  return p;
}
void pinned_slot_free(int* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(p);
}

void DevBuf::ensure(size_t b, cudaStream_t s) {
  if (b <= bytes && p) return;
  keep_pool_memory();
  if (p) cudaFreeAsync(p, st);
  p = nullptr;
  st = s;
  bytes = b;
  if (b == 0) return;
  static const bool trace = std::getenv("RTB_ALLOC_TRACE") != nullptr;  // debugging aid
  if (trace && b >= (64u << 20)) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    std::fprintf(stderr, "[rtb alloc] %.3f GB (free %.3f GB)\n", b / 1e9, fr / 1e9);
  }
  RTB_CUDA(cudaMallocAsync(&p, b, s));
}

// ---------------------------------------------------------------------------
// small kernels

__global__ void k_uniform_init(double* out, long long n, unsigned long long seed,
                               long long offset) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = u64_to_unit(sm_at(seed, (uint64_t)(offset + i)));
}

// K K^T + lambda I of an order-3 factor update (ref tucker.cpp:70-89), one CTA per column r:
// Q_r = Gram_a S_r Gram_b with S_r the slice of G at index r of mode n (a < b the other modes),
// then kk[i][r] = <S_i, Q_r> + lambda [i == r]. One launch with R_n CTAs instead of the chain of
// two mode products, the contraction and the diagonal (4 launches) on the factor-update branch.
__global__ void __launch_bounds__(256) k_fu_kkt3(const double* __restrict__ core,
                                                 const double* __restrict__ grams, int stride,
                                                 int n, int R0, int R1, int R2, double lambda,
                                                 double* __restrict__ kk) {
  __shared__ double Ga[32 * 33], Gb[32 * 33], S[32 * 33], T[32 * 33];
  const int Rs[3] = {R0, R1, R2};
  const int a = n == 0 ? 1 : 0, b = n == 2 ? 1 : 2;
  const int Ra = Rs[a], Rb = Rs[b], Rn = Rs[n];
  const int r = blockIdx.x;
  // G index (i0, i1, i2) -> flat; the slice at mode-n index q: S[p][t] over (mode a, mode b)
  auto gidx = [&](int q, int p, int t) {
    int id[3];
    id[n] = q;
    id[a] = p;
    id[b] = t;
    return (id[0] * R1 + id[1]) * R2 + id[2];
  };
  for (int e = threadIdx.x; e < Ra * Ra; e += blockDim.x)
    Ga[(e / Ra) * 33 + e % Ra] = grams[(size_t)a * stride + e];
  for (int e = threadIdx.x; e < Rb * Rb; e += blockDim.x)
    Gb[(e / Rb) * 33 + e % Rb] = grams[(size_t)b * stride + e];
  for (int e = threadIdx.x; e < Ra * Rb; e += blockDim.x) {
    const int p = e / Rb, t = e - p * Rb;
    S[p * 33 + t] = core[gidx(r, p, t)];
  }
  __syncthreads();
  // T = S Gram_b
  for (int e = threadIdx.x; e < Ra * Rb; e += blockDim.x) {
    const int p = e / Rb, t = e - p * Rb;
    double acc = 0.0;
    for (int k = 0; k < Rb; ++k) acc = fma(S[p * 33 + k], Gb[k * 33 + t], acc);
    T[p * 33 + t] = acc;
  }
  __syncthreads();
  // Q = Gram_a T (into S)
  for (int e = threadIdx.x; e < Ra * Rb; e += blockDim.x) {
    const int p = e / Rb, t = e - p * Rb;
    double acc = 0.0;
    for (int k = 0; k < Ra; ++k) acc = fma(Ga[p * 33 + k], T[k * 33 + t], acc);
    S[p * 33 + t] = acc;
  }
  __syncthreads();
  // kk[i][r] = <G slice i, Q_r>: warp per i
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = warp; i < Rn; i += nw) {
    double acc = 0.0;
    for (int e = lane; e < Ra * Rb; e += 32) {
      const int p = e / Rb, t = e - p * Rb;
      acc = fma(__ldg(core + gidx(i, p, t)), S[p * 33 + t], acc);
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) kk[i * Rn + r] = acc + (i == r ? lambda : 0.0);
  }
}

__global__ void k_add_diag(double* a, int n, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[(size_t)i * n + i] += v;
}

// sum of squares of several arrays in a fixed order (one block)
struct NormSet {
  const double* p[9];
  long long n[9];
  int count;
};
__global__ void k_norms(NormSet ns, double* out) {
  __shared__ double red[32];
  double total = 0.0;
  for (int a = 0; a < ns.count; ++a) {
    double s = 0.0;
    for (long long i = threadIdx.x; i < ns.n[a]; i += blockDim.x) s += ns.p[a][i] * ns.p[a][i];
    s = block_sum<1024>(s, red);
    total += s;  // meaningful in thread 0
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = total;
}

// loss = residual + lambda * reg; rmse = sqrt(residual / size)  (tucker.cpp:216-229)
__global__ void k_finish_loss(const double* residual, const double* reg, double lambda,
                              double size, double* loss_out, double* rmse_out) {
  const double r = *residual;
  *loss_out = r + lambda * *reg;
  *rmse_out = sqrt(r / size);
}

// per-block partial sums of x^2 (||X||^2 for the fast loss)
__global__ void k_sumsq_partials(const double* __restrict__ x, long long n, double* partial) {
  __shared__ double red[32];
  double s = 0.0;
  const long long n2 = n >> 1;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(x2 + i);
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) s = fma(x[n - 1], x[n - 1], s);
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// Fast loss: sum (X - Xhat)^2 = ||X||^2 - 2 <Y, G> + <Q, G>, Y = X x_n A_n^T (all n),
// Q = G x_n (A_n^T A_n) (all n). Accepted when the residual is >= thr ||X||^2 (the
// cancellation then costs < ~1e-9 relative); otherwise *need = 1 and the direct
// pass queued behind it runs.
__global__ void k_fast_loss(const double* __restrict__ Y, const double* __restrict__ Q,
                            const double* __restrict__ G, long long d,
                            const double* __restrict__ xx, const double* __restrict__ reg,
                            double lambda, double size, double thr, double* loss_out,
                            double* rmse_out, int* need) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (long long i = threadIdx.x; i < d; i += blockDim.x) {
    a = fma(Y[i], G[i], a);
    b = fma(Q[i], G[i], b);
  }
  a = block_sum<1024>(a, red);
  __syncthreads();
  b = block_sum<1024>(b, red);
  if (threadIdx.x == 0) {
    const double x2 = *xx;
    const double r = (x2 - 2.0 * a) + b;
    if (r >= thr * x2 && isfinite(r)) {
      *loss_out = r + lambda * *reg;
      *rmse_out = sqrt(r / size);
      *need = 0;
    } else {
      *need = 1;
    }
  }
}

__global__ void k_finish_loss_guarded(const double* residual, const double* reg, double lambda,
                                      double size, double* loss_out, double* rmse_out,
                                      const int* need) {
  if (*need == 0) return;
  const double r = *residual;
  *loss_out = r + lambda * *reg;
  *rmse_out = sqrt(r / size);
}

__global__ void k_resid_partials(const double* x, const double* xh, long long n, double* partial) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double d = x[i] - xh[i];
    s += d * d;
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// U = A V diag(1/sigma) over the first `rank` eigenpairs (exact core bases)
__global__ void k_factor_u(const double* A, int I, int R, const double* V, const double* mu,
                           const int* rank, double* U) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int r = *rank;
  if (e >= (long long)I * r) return;
  const int i = (int)(e / r), k = (int)(e % r);
  double s = 0.0;
  for (int j = 0; j < R; ++j) s += A[(size_t)i * R + j] * V[j * R + k];
  U[e] = s / sqrt(mu[k]);
}

// rank from eigenvalues of a Gram with the Gram-form cutoff used by k_leverage_rows
__global__ void k_gram_rank(const double* evals, int stride, const int* rows, const int* cols,
                            int order, int* ranks) {
  const int m = threadIdx.x;
  if (m >= order) return;
  const double* mu = evals + (size_t)m * stride;
  const int I = rows[m], R = cols[m];
  const double cut = (double)(I > R ? I : R) * DBL_EPSILON * mu[0];
  int r = 0;
  while (r < R && mu[r] > cut && mu[r] > 0.0) ++r;
  ranks[m] = r;
}

// w[t] *= s_t / (s_t^2 + lambda), s_t = prod_n sigma_n[t_n] (tucker.cpp:116-124)
struct ScaleSpec {
  int order;
  int dims[8];
  const double* mu[8];
};
__global__ void k_core_scale(double* w, long long n, ScaleSpec sp, double lambda) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  long long rem = e;
  double sigma = 1.0;
  for (int m = sp.order - 1; m >= 0; --m) {
    const int t = (int)(rem % sp.dims[m]);
    rem /= sp.dims[m];
    sigma *= sqrt(sp.mu[m][t]);
  }
  w[e] *= sigma / (sigma * sigma + lambda);
}

__global__ void k_transpose_small(const double* V, int R, int r, double* out /* R x r */) {
  // out[i][k] = V[i][k] for k < r (V is R x R, column k = eigvec k)
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R * r) return;
  const int i = e / r, k = e % r;
  out[e] = V[i * R + k];
}

__global__ void k_any_zero_rank(const int* ranks, int order, int* flag) {
  if (threadIdx.x == 0) {
    int z = 0;
    for (int m = 0; m < order; ++m) z |= ranks[m] == 0;
    *flag = z;
  }
}

__global__ void k_check_finite(const double* v, long long n, int* bad) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !isfinite(v[i])) atomicExch(bad, 1);
}

// Per-sweep seeds from device counters, so a captured sweep draws new ones every launch:
// seeds[0] = sketch_rng.next_u64() for sweep k (ref tucker.cpp:254-255), seeds[1 + n] =
// factor_rng.next_u64() for the n-th sketched factor update (perf mode, orc_als_fs).
__global__ void k_sweep_seeds(unsigned long long* seeds, unsigned long long* ctr,
                              unsigned long long sketch_rng, unsigned long long factor_rng,
                              int nf) {
  if (threadIdx.x != 0) return;
  const unsigned long long k = ctr[0], f = ctr[1];
  seeds[0] = sm_at(sketch_rng, k);
  for (int n = 0; n < nf; ++n) seeds[1 + n] = sm_at(factor_rng, f + n);
  ctr[0] = k + 1;
  ctr[1] = f + nf;
}

// Verdict of a PCG core solve for the host: post = {PCG status, iterations, zero-factor
// flag, core not finite}; the warm-start flag of the next solve = accepted and finite.
__global__ void k_core_post(const double* __restrict__ core, long long d, const int* pcg_status,
                            const int* zero_flag, int* warm, int* post) {
  int bad = 0;
  for (long long i = threadIdx.x; i < d; i += blockDim.x) bad |= !isfinite(core[i]);
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    const int ok = pcg_status[0] == 0 && *zero_flag == 0;
    post[0] = pcg_status[0];
    post[1] = pcg_status[1];
    post[2] = *zero_flag;
    post[3] = bad;
    *warm = ok && !bad;
  }
}

__global__ void k_set_int(int* p, int v) { *p = v; }

// Grid-stride finiteness scan (exponent field all ones = Inf/NaN), 2 doubles per load.
__global__ void k_all_finite(const double* v, long long n, int* bad) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  int hit = 0;
  const long long n2 = n >> 1;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 a = __ldcs(v2 + i);
    hit |= !isfinite(a.x) | !isfinite(a.y);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) hit |= !isfinite(v[n - 1]);
  if (__syncthreads_or(hit) && threadIdx.x == 0) atomicExch(bad, 1);
}

// ---------------------------------------------------------------------------
// profiling (optional per-kernel-family device time)

struct Profiler {
  bool on = false;
  cudaStream_t st = nullptr;
  struct Ev {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Ev> evs;
  std::map<std::string, KernelTiming> acc;
  void begin(const char* name, cudaEvent_t* a) {
    if (!on) return;
    RTB_CUDA(cudaEventCreate(a));
    RTB_CUDA(cudaEventRecord(*a, st));
    (void)name;
  }
  void end(const char* name, cudaEvent_t a) {
    if (!on) return;
    cudaEvent_t b;
    RTB_CUDA(cudaEventCreate(&b));
    RTB_CUDA(cudaEventRecord(b, st));
    evs.push_back({name, a, b});
  }
  void collect() {
    for (auto& e : evs) {
      float ms = 0.f;
      RTB_CUDA(cudaEventSynchronize(e.b));
      RTB_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
      auto& k = acc[e.name];
      k.name = e.name;
      k.total += ms * 1e-3;
      k.launches += 1;
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    evs.clear();
  }
  ~Profiler() {
    for (auto& e : evs) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
  }
};

struct Scope {
  Profiler& p;
  const char* n;
  cudaEvent_t a{};
  Scope(Profiler& pr, const char* name) : p(pr), n(name) { p.begin(n, &a); }
  ~Scope() {
    try {
      p.end(n, a);
    } catch (...) {
    }
  }
};

// ---------------------------------------------------------------------------
// Engine

static uint64_t prod(const std::vector<uint64_t>& v, size_t from = 0, size_t to = SIZE_MAX) {
  uint64_t p = 1;
  for (size_t i = from; i < v.size() && i < to; ++i) p *= v[i];
  return p;
}

bool cuda_device_present() {
  static const bool present = [] {
    int n = 0;
    const bool ok = cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
    cudaGetLastError();
    return ok;
  }();
  return present;
}

void upload_checked(double* dst, const double* src, uint64_t n, cudaStream_t st,
                    const char* what) {
  RTB_CUDA(cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyHostToDevice, st));
  DevBuf flag;
  flag.ensure(4, st);
  RTB_CUDA(cudaMemsetAsync(flag.p, 0, 4, st));
  int sms = 148;
  int dev = 0;
  RTB_CUDA(cudaGetDevice(&dev));
  RTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const long long blocks = std::max<long long>(1, std::min<long long>(sms * 4LL, ceil_div<long long>((long long)n / 2 + 1, 256)));
  if (n) {
    k_all_finite<<<(unsigned)blocks, 256, 0, st>>>(dst, (long long)n, flag.as<int>());
    RTB_LAUNCH_CHECK();
  }
  int bad = 0;
  RTB_CUDA(cudaMemcpyAsync(&bad, flag.p, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (bad) throw Error(1, std::string(what) + ": non-finite entry");
}

uint64_t sample_count_formula(double beta_prime, uint64_t d, double epsilon, double delta) {
  // ref sketch_ridge.cpp:40-50
  if (beta_prime <= 0.0 || epsilon <= 0.0 || epsilon >= 1.0 || delta <= 0.0 || delta >= 1.0 ||
      d == 0)
    throw Error(1, "sample_count: parameters out of range");
  const double dd = (double)d;
  const double log_term = 420.0 * std::log(4.0 * dd / delta);
  const double tail_term = 1.0 / (delta * epsilon);
  return (uint64_t)std::ceil(4.0 * dd / beta_prime * std::max(log_term, tail_term));
}

// Generating the P rows inside the loss pass (no P in HBM) measured slower than
// materialising P (the per-row-block generation stalls the residual warps): off.
constexpr bool kGenerateP = false;

class Engine {
 public:
  Engine(const double* x, const std::vector<uint64_t>& shape, const std::vector<uint64_t>& ranks,
         const AlsOptions& opt)
      : x_(x), shape_(shape), ranks_(ranks), opt_(opt), N_((int)shape.size()) {
    st_ = current_stream();
    prof_.on = opt.profile;
    prof_.st = st_;
    total_ = prod(shape_);
    d_ = prod(ranks_);
    // Multi-GPU: this process holds rows [lo_, lo_ + nloc_) of mode 1 (the even split
    // r * I_1 / P); X passes, the mode-1 factor rows and the Gram's data draws are
    // local, partial sums meet in opt_.allreduce.
    if (opt_.shard_count > 1) {
      const uint64_t I1 = shape_[0], P = opt_.shard_count, r = opt_.shard_rank;
      lo_ = (long long)(r * I1 / P);
      nloc_ = (long long)((r + 1) * I1 / P) - lo_;
    } else {
      lo_ = 0;
      nloc_ = (long long)shape_[0];
    }
    lshape_ = shape_;
    lshape_[0] = (uint64_t)nloc_;
    ltotal_ = prod(lshape_);
    rmax_ = 0;
    for (auto r : ranks_) rmax_ = std::max<int>(rmax_, (int)r);
    eig_stride_ = std::max(rmax_ * rmax_, 1);
    allocate();
  }

  // ---- model init (ref tucker.cpp:168-190) and initial loss ----
  void init_model() {
    if (opt_.init_core) {
      RTB_CUDA(cudaMemcpyAsync(core_.p, opt_.init_core, d_ * 8, cudaMemcpyHostToDevice, st_));
      RTB_CUDA(cudaMemcpyAsync(fac_.p, opt_.init_factors, fac_elems_ * 8, cudaMemcpyHostToDevice,
                               st_));
    } else {
      k_uniform_init<<<ceil_div<long long>(d_, 256), 256, 0, st_>>>(core_.as<double>(), d_,
                                                                     opt_.seed, 0);
      RTB_LAUNCH_CHECK();
      k_uniform_init<<<ceil_div<long long>(fac_elems_, 256), 256, 0, st_>>>(
          fac_.as<double>(), fac_elems_, opt_.seed, (long long)d_);
      RTB_LAUNCH_CHECK();
    }
    for (int n = 0; n < N_; ++n) factor_gram(n);
    sketch_rng_ = opt_.seed;
    // SplitMix64(seed).split(): next_u64 ^ 0x5851f42d4c957f2d (ref rng.hpp:56, tucker.cpp:206)
    sketch_rng_ = sm_at(opt_.seed, 0) ^ 0x5851f42d4c957f2dULL;
    sketch_k_ = 0;
    // perf mode: factor sketch seeds from a second split of the same generator
    // (orc_als_fs), one next_u64 per (sweep, mode)
    factor_rng_ = sm_at(opt_.seed, 1) ^ 0x5851f42d4c957f2dULL;
    factor_k_ = 0;
    RTB_CUDA(cudaMemsetAsync(ctr_dev_.p, 0, 16, st_));
    RTB_CUDA(cudaMemsetAsync(warm_dev_.p, 0, 4, st_));
    scores_valid_ = false;
    t_valid_ = false;
  }

  double* hist_loss(size_t i) { return hist_.as<double>() + 2 * i; }

  void record_loss(size_t slot) {
    // loss pass writes loss/rmse into history slot `slot`
    loss_pass(hist_loss(slot), hist_loss(slot) + 1);
  }

  // ---- one sweep ----
  // Enqueues sweep `iter` without a host round trip: the per-sweep seeds come from device
  // counters (k_sweep_seeds), the core solve's verdict goes to pinned host memory behind
  // the step event core_done (resolve_core() reads it while the GPU runs the loss pass),
  // and from the second sweep on the whole sweep is one CUDA graph launch when the path
  // allows it (sketched core with the PCG solve, no profiling, no sharding).
  void sweep(uint32_t iter) {
    const int rows = opt_.record_history ? N_ + 1 : 1;
    ensure_hist(hist_rows_.size() + rows);
    const size_t first = hist_rows_.size();
    if (opt_.record_history)
      for (int n = 0; n < N_; ++n) hist_rows_.push_back({iter, "F" + std::to_string(n + 1)});
    hist_rows_.push_back({iter, "Core"});
    core_row_ = hist_rows_.size() - 1;
    if (graph_ok() && sweeps_enqueued_ >= 1 && !gexec_) capture_sweep();
    if (gexec_) {
      RTB_CUDA(cudaGraphLaunch(gexec_, st_));
      launch_counter() += graph_kernels_;
      ++graph_launches_;
      RTB_CUDA(cudaMemcpyAsync(hist_loss(first), loss_rows_.p, (size_t)rows * 16,
                               cudaMemcpyDeviceToDevice, st_));
    } else {
      sweep_body(hist_loss(first));
    }
    core_pending_ = opt_.sketched && deferred_core_;
    ++sweeps_enqueued_;
    iterations_ = iter;
    if (!core_pending_) {  // exact core / non-CG solve: the stream was synchronised inside
      RTB_CUDA(cudaEventSynchronize(step_ev_[2 * N_ + 1]));
      collect_steps();
    }
  }

  // the kernels of one sweep; loss rows (loss, rmse) go to rows[0..]
  void sweep_body(double* rows) {
    k_sweep_seeds<<<1, 32, 0, st_>>>(seed_dev_.as<unsigned long long>(),
                                     ctr_dev_.as<unsigned long long>(), sketch_rng_, factor_rng_,
                                     (opt_.factor_samples > 0 && N_ >= 2) ? N_ : 0);
    RTB_LAUNCH_CHECK();
    decoded_ahead_ = false;
    keys_ahead_ = keys_ready_ = false;
    if (opt_.sketched) decode_ahead(seed_dev_.as<unsigned long long>());
    int r = 0;
    for (int n = 0; n < N_; ++n) {
      rec(step_ev_[2 * n]);
      if (opt_.factor_samples > 0 && N_ >= 2)
        update_factor_sketched(n, 0, seed_dev_.as<unsigned long long>() + 1 + n);
      else
        update_factor(n);
      if (n == 0) keys_ahead();
      rec(step_ev_[2 * n + 1]);
      if (opt_.record_history) {
        loss_pass(rows + 2 * r, rows + 2 * r + 1);
        ++r;
      }
    }
    rec(step_ev_[2 * N_]);
    deferred_core_ = false;
    if (opt_.sketched) {
      // per-sweep sketch seed = sketch_seed_rng.next_u64() (ref tucker.cpp:254-255), read
      // from seed_dev_[0] on the device
      update_core_sketched(0, seed_dev_.as<unsigned long long>(), true);
    } else {
      update_core_exact();
    }
    rec(step_ev_[2 * N_ + 1]);  // = core_done: the core verdict is in post_host_ after it
    loss_pass(rows + 2 * r, rows + 2 * r + 1);
  }

  void rec(cudaEvent_t e) {
    if (capturing_) RTB_CUDA(cudaEventRecordWithFlags(e, st_, cudaEventRecordExternal));
    else RTB_CUDA(cudaEventRecord(e, st_));
  }

  bool graph_ok() const {
    static const bool off = std::getenv("RTB_NO_GRAPH") != nullptr;
    // capturing and instantiating a sweep costs about one small sweep (C1: ~0.5 ms) and saves
    // ~15% of each later one: a short run (< 16 sweeps) on a small tensor (< 2^24 entries,
    // launch-latency bound) stays eager
    return !off && !opt_.no_graph && !graph_failed_ && opt_.sketched && !opt_.profile && !sharded() &&
           pcg_path_ && !opt_.fast_loss && (opt_.max_iterations >= 16 || total_ >= (1ull << 24));
  }

  // Stream-captures one steady-state sweep into gexec_ (loss rows into loss_rows_). Any
  // failure leaves the engine on the eager path.
  void capture_sweep() {
    const unsigned long long before = launch_counter();
    cudaGraph_t g = nullptr;
    RTB_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed));
    capturing_ = true;
    try {
      sweep_body(loss_rows_.as<double>());
    } catch (...) {
      capturing_ = false;
      cudaStreamEndCapture(st_, &g);
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      graph_failed_ = true;
      launch_counter() -= launch_counter() - before;
      return;
    }
    capturing_ = false;
    cudaError_t e = cudaStreamEndCapture(st_, &g);
    if (e == cudaSuccess && deferred_core_)
      e = cudaGraphInstantiateWithFlags(&gexec_, g, 0);
    if (g) cudaGraphDestroy(g);
    graph_kernels_ = launch_counter() - before;
    launch_counter() -= graph_kernels_;  // counted per graph launch instead
    if (e != cudaSuccess || !deferred_core_) {
      cudaGetLastError();
      gexec_ = nullptr;
      graph_failed_ = true;
    }
  }

  void drop_graph() {
    if (gexec_) cudaGraphExecDestroy(gexec_);
    gexec_ = nullptr;
  }

  // Lookbehind check of the sweep just enqueued: waits for its core_done event (the GPU
  // meanwhile runs that sweep's loss pass, and the host then enqueues the next sweep
  // behind it), reads the core solve's verdict, and runs the fallback solve plus a fresh
  // loss pass for that sweep if the PCG answer was not accepted.
  void resolve_core() {
    if (!core_pending_) return;
    core_pending_ = false;
    RTB_CUDA(cudaEventSynchronize(step_ev_[2 * N_ + 1]));
    collect_steps();
    if (finish_core_solve()) {
      drop_graph();  // the fallback may have (re)allocated workspaces
      record_loss(core_row_);
    }
  }

  double last_loss_host() {
    double v[2];
    RTB_CUDA(cudaMemcpyAsync(v, hist_loss(hist_rows_.size() - 1), 16, cudaMemcpyDeviceToHost,
                             st_));
    RTB_CUDA(cudaStreamSynchronize(st_));
    return v[0];
  }

  void initial_loss() {
    loss_pass(init_loss_.as<double>(), init_loss_.as<double>() + 1);
  }
  double initial_loss_host() {
    double v[2];
    RTB_CUDA(cudaMemcpyAsync(v, init_loss_.p, 16, cudaMemcpyDeviceToHost, st_));
    RTB_CUDA(cudaStreamSynchronize(st_));
    return v[0];
  }

  void output(AlsOutput& out) {
    resolve_core();
    RTB_CUDA(cudaStreamSynchronize(st_));
    out.shape = shape_;
    out.ranks = ranks_;
    out.lambda = opt_.lambda;
    out.core.resize(d_);
    out.factors.resize(fac_elems_);
    RTB_CUDA(cudaMemcpy(out.core.data(), core_.p, d_ * 8, cudaMemcpyDeviceToHost));
    RTB_CUDA(cudaMemcpy(out.factors.data(), fac_.p, fac_elems_ * 8, cudaMemcpyDeviceToHost));
    std::vector<double> h(2 * hist_rows_.size());
    if (!h.empty())
      RTB_CUDA(cudaMemcpy(h.data(), hist_.p, h.size() * 8, cudaMemcpyDeviceToHost));
    out.history.clear();
    for (size_t i = 0; i < hist_rows_.size(); ++i)
      out.history.push_back({hist_rows_[i].iter, hist_rows_[i].step, h[2 * i], h[2 * i + 1]});
    out.timings.assign(N_ + 1, StepTiming{});
    for (int n = 0; n < N_; ++n) out.timings[n].step = "F" + std::to_string(n + 1);
    out.timings[N_].step = "Core";
    for (int k = 0; k <= N_; ++k) {
      out.timings[k].total = step_total_[k];
      out.timings[k].count = step_count_[k];
    }
    prof_.collect();
    out.kernels.clear();
    for (auto& kv : prof_.acc) out.kernels.push_back(kv.second);
    out.iterations = iterations_;
    if (!out.history.empty()) {
      out.final_loss = out.history.back().loss;
      out.final_rmse = out.history.back().rmse;
    }
    out.converged = converged_;
    out.last_sample_count = last_s_;
    RTB_CUDA(cudaMemcpy(&out.last_data_draws, data_draws_.p, 8, cudaMemcpyDeviceToHost));
    out.last_rank_deficient = last_rank_deficient_;
    out.last_solver_path = last_solver_path_;
    out.last_pcg_iterations = last_pcg_iters_;
    out.sweep_seconds = sweep_seconds_;
    out.graph_launches = graph_launches_;
  }

  ~Engine() {
    if (gexec_) cudaGraphExecDestroy(gexec_);
    for (auto e : step_ev_)
      if (e) cudaEventDestroy(e);
    pinned_slot_free(post_host_);
    if (fork_ev_) cudaEventDestroy(fork_ev_);
    if (join_ev_) cudaEventDestroy(join_ev_);
    if (dfork_ev_) cudaEventDestroy(dfork_ev_);
    if (kfork_ev_) cudaEventDestroy(kfork_ev_);
    if (djoin_ev_) cudaEventDestroy(djoin_ev_);
  }

  // Adds the elapsed times of the last sweep's step events (the stream has passed them).
  void collect_steps() {
    for (int k = 0; k <= N_; ++k) {
      float ms = 0.f;
      RTB_CUDA(cudaEventElapsedTime(&ms, step_ev_[2 * k], step_ev_[2 * k + 1]));
      step_total_[k] += ms * 1e-3;
      step_count_[k] += 1;
    }
  }

  // exposed for the single-op entry points
  void set_model(const double* core_h, const double* fac_h) {
    RTB_CUDA(cudaMemcpyAsync(core_.p, core_h, d_ * 8, cudaMemcpyHostToDevice, st_));
    RTB_CUDA(cudaMemcpyAsync(fac_.p, fac_h, fac_elems_ * 8, cudaMemcpyHostToDevice, st_));
    for (int n = 0; n < N_; ++n) factor_gram(n);
    t_valid_ = false;
  }
  void get_core(double* h) {
    RTB_CUDA(cudaMemcpyAsync(h, core_.p, d_ * 8, cudaMemcpyDeviceToHost, st_));
    RTB_CUDA(cudaStreamSynchronize(st_));
  }
  void get_factor(int n, double* h) {
    RTB_CUDA(cudaMemcpyAsync(h, factor(n), shape_[n] * ranks_[n] * 8, cudaMemcpyDeviceToHost, st_));
    RTB_CUDA(cudaStreamSynchronize(st_));
  }
  void update_factor_public(int n) { update_factor(n); }
  void core_sketched_public(uint64_t s, uint64_t seed, uint64_t* idx, double* w) {
    opt_.sample_override = s;
    update_core_sketched(seed);
    if (idx && last_s_) {
      RTB_CUDA(cudaMemcpyAsync(idx, sk_idx_.p, last_s_ * 8, cudaMemcpyDeviceToHost, st_));
      RTB_CUDA(cudaMemcpyAsync(w, sk_w_.p, last_s_ * 8, cudaMemcpyDeviceToHost, st_));
    }
    RTB_CUDA(cudaStreamSynchronize(st_));
  }
  void core_exact_public() { update_core_exact(); }
  void loss_public(double* loss, double* rmse) {
    loss_pass(init_loss_.as<double>(), init_loss_.as<double>() + 1);
    double v[2];
    RTB_CUDA(cudaMemcpyAsync(v, init_loss_.p, 16, cudaMemcpyDeviceToHost, st_));
    RTB_CUDA(cudaStreamSynchronize(st_));
    *loss = v[0];
    *rmse = v[1];
  }
  void reconstruct(double* out_dev) { reconstruct_full(out_dev); }

  double tolerance() const { return opt_.tolerance; }
  double prev_loss_ = 0.0;
  bool have_prev_ = false;
  uint32_t iterations_ = 0;
  bool converged_ = false;
  double sweep_seconds_ = 0.0;
  cudaStream_t st_;

 private:
  const double* x_;  // this process's slab of X (rows lo_ .. lo_ + nloc_ of mode 1)
  long long lo_ = 0, nloc_ = 0;
  std::vector<uint64_t> lshape_;
  uint64_t ltotal_ = 0;
  // a caller that installs the all-reduce callback gets the sharded path, one shard included
  // (P = 1 runs the collective plumbing for real on a single GPU: bench.py --nccl-p1)
  bool sharded() const { return opt_.allreduce != nullptr; }
  void allreduce(double* buf, uint64_t n) {
    if (sharded()) opt_.allreduce(buf, n, st_, opt_.allreduce_user);
  }
  std::vector<uint64_t> shape_, ranks_;
  AlsOptions opt_;
  int N_;
  uint64_t total_, d_;
  int rmax_, eig_stride_;
  uint64_t fac_elems_ = 0;
  std::vector<uint64_t> fac_off_;
  Profiler prof_;

  DevBuf ns_vals_, pinv2_, linv_, spd_ok_;
  // the factor updates' (K K^T + lambda I)^+ scratch: their own slots, so a score step for
  // finished modes can run on a side branch meanwhile (keys_ahead)
  DevBuf fu_linv_, fu_ok_, fu_evals_, fu_evecs_, fu_status_;
  DevBuf core_, fac_, grams_, evals_, evecs_, eig_status_, ns_, pinv_, ranks_dev_;
  DevBuf T_, P_, tmp_a_, tmp_b_, partial_, scal_, hist_, init_loss_, xx_, loss_need_, yq_;
  bool xx_valid_ = false;
  DevBuf scores_, cdf_, sums_, score_off_, rows_dev_, cols_dev_, flag_;
  DevBuf pinv_work_, pinv_rank_;
  DevBuf sk_idx_, sk_w_, draw_work_, gram_work_, G_, rhs_, chol_work_, chol_status_,
      data_draws_, zero_flag_, U_[8], pgram_, pcg_work_, pcg_status_, blocks_, pev_, pvec_, pst_;
  uint64_t sketch_rng_ = 0, sketch_k_ = 0;
  uint64_t factor_rng_ = 0, factor_k_ = 0;
  bool scores_valid_ = false;
  DevBuf fsums_, fsk_idx_, fsk_w_, fsk_work_, hj_ws_;
  DevBuf xrot_[kMaxOrder];  // perf mode: X with mode n moved last (n < N - 1)
  bool xrot_ok_ = std::getenv("RTB_NO_XROT") == nullptr;
  bool t_valid_ = false;
  uint64_t last_s_ = 0;
  int last_rank_deficient_ = 0, last_solver_path_ = 0, last_pcg_iters_ = 0;
  // step events of the sweep in flight: (start, end) per step, F_1..F_N then Core; the
  // Core end event is also the point after which the core verdict is in post_host_
  cudaEvent_t step_ev_[2 * (kMaxOrder + 1)] = {};
  double step_total_[kMaxOrder + 1] = {};
  uint64_t step_count_[kMaxOrder + 1] = {};
  // per-sweep device seeds / counters, the core verdict, CUDA graph of a sweep
  DevBuf seed_dev_, ctr_dev_, post_, warm_dev_, loss_rows_;
  int* post_host_ = nullptr;  // pinned
  bool pcg_path_ = false, deferred_core_ = false, core_pending_ = false;
  bool capturing_ = false, graph_failed_ = false;
  cudaGraphExec_t gexec_ = nullptr;
  unsigned long long graph_kernels_ = 0;
  uint64_t graph_launches_ = 0;
  uint64_t sweeps_enqueued_ = 0;
  size_t core_row_ = 0;
  // history rows (loss, rmse) on the device; grown on demand (copying the rows so far)
  size_t hist_cap_ = 0;
  void ensure_hist(size_t rows) {
    if (rows <= hist_cap_) return;
    const size_t cap = std::max(rows, 2 * hist_cap_);
    DevBuf nb(cap * 16 + 16, st_);
    if (hist_cap_) RTB_CUDA(cudaMemcpyAsync(nb.p, hist_.p, hist_cap_ * 16, cudaMemcpyDeviceToDevice, st_));
    hist_ = std::move(nb);
    hist_cap_ = cap;
  }
  struct HRow {
    uint32_t iter;
    std::string step;
  };
  std::vector<HRow> hist_rows_;
  size_t tmp_elems_ = 0;

  double* factor(int n) { return fac_.as<double>() + fac_off_[n]; }
  double* gram(int n) { return grams_.as<double>() + (size_t)n * eig_stride_; }

  FactorSet factor_set() {
    FactorSet fs{};
    fs.order = N_;
    for (int n = 0; n < N_; ++n) {
      fs.ptr[n] = factor(n);
      fs.rows[n] = (int)shape_[n];
      fs.cols[n] = (int)ranks_[n];
    }
    return fs;
  }

  void allocate() {
    fac_off_.resize(N_);
    for (int n = 0; n < N_; ++n) {
      fac_off_[n] = fac_elems_;
      fac_elems_ += shape_[n] * ranks_[n];
    }
    core_.ensure(d_ * 8, st_);
    fac_.ensure(fac_elems_ * 8, st_);
    grams_.ensure((size_t)N_ * eig_stride_ * 8 + 8, st_);
    pinv_.ensure((size_t)eig_stride_ * 8 + 8, st_);
    pinv2_.ensure((size_t)eig_stride_ * 8 + 8, st_);
    linv_.ensure((size_t)N_ * eig_stride_ * 8 + 8, st_);
    spd_ok_.ensure(64 * 4, st_);
    {
      // eigen_one() may also factor a d <= 64 core Gram into slot 0
      const size_t eb = std::max<size_t>((size_t)N_ * eig_stride_, 64 * 64) * 8 + 8;
      evals_.ensure(eb, st_);
      evecs_.ensure(eb, st_);
      int vals[65];
      for (int i = 0; i < 65; ++i) vals[i] = i;
      ns_vals_.ensure(65 * 4, st_);
      RTB_CUDA(cudaMemcpy(ns_vals_.p, vals, 65 * 4, cudaMemcpyHostToDevice));
    }
    eig_status_.ensure(64 * 4, st_);
    {
      // one-sided Jacobi workspace of the score step (allocated here: the step may run on a
      // side stream)
      long long stride = 0;
      for (int n = 0; n < N_; ++n)
        stride = std::max<long long>(stride, (long long)shape_[n] * (ranks_[n] + (ranks_[n] & 1)));
      hj_ws_.ensure((size_t)N_ * stride * 8 + 64, st_);
    }
    {
      const size_t fb = (size_t)std::max(eig_stride_, 64 * 64) * 8 + 8;
      fu_linv_.ensure(fb, st_);
      fu_evals_.ensure(fb, st_);
      fu_evecs_.ensure(fb, st_);
      fu_ok_.ensure(64 * 4, st_);
      fu_status_.ensure(64 * 4, st_);
    }
    pgram_.ensure((size_t)N_ * eig_stride_ * 8 + 8, st_);
    pev_.ensure((size_t)N_ * eig_stride_ * 8 + 8, st_);
    pvec_.ensure((size_t)N_ * eig_stride_ * 8 + 8, st_);
    pst_.ensure(64 * 4 + 8 * 8, st_);
    pcg_status_.ensure(16, st_);
    ns_.ensure(64 * 4, st_);
    ranks_dev_.ensure(64 * 4, st_);
    // T and P: (this shard's total / I_N) x R_N
    const uint64_t tsz = ltotal_ / shape_[N_ - 1] * ranks_[N_ - 1];
    T_.ensure(tsz * 8, st_);
    P_.ensure(tsz * 8, st_);
    // chain temporaries: largest intermediate of any TTM chain we run, on this shard's slab
    // (a 275 GB C5 tensor is 34 GB per GPU at P = 8: nothing here may scale with the whole)
    uint64_t mx = d_;
    {
      // factor projections and the exact core: X (or T) x_m A_m^T over the other modes
      for (int n = 0; n < N_; ++n) {
        std::vector<uint64_t> dims = lshape_;
        for (int m = 0; m < N_; ++m) {
          if (m == n) continue;
          dims[m] = ranks_[m];
          mx = std::max(mx, prod(dims));
        }
      }
      // P = G x_1 A_1 ... x_{N-1} A_{N-1} (build_P; the last mode stays R_N); the unsharded
      // fast-loss Y chain runs on T, whose intermediates the projections above bound
      std::vector<uint64_t> dims = ranks_;
      for (int m = 0; m + 1 < N_; ++m) {
        dims[m] = lshape_[m];
        mx = std::max(mx, prod(dims));
      }
    }
    for (int n = 0; n < N_; ++n) mx = std::max<uint64_t>(mx, shape_[n] * ranks_[n]);
    mx = std::max<uint64_t>(mx, d_ * d_ <= (1u << 24) ? d_ * d_ : 0);  // pinv fallback scratch
    tmp_elems_ = mx;
    tmp_a_.ensure(mx * 8, st_);
    tmp_b_.ensure(mx * 8, st_);
    const long long nblk = std::max<long long>(
        ttm_last_parts_bound((long long)(total_ / shape_[N_ - 1]), (int)shape_[N_ - 1],
                        (int)ranks_[N_ - 1]),
        kNumSMs * 8);
    partial_.ensure(std::max<size_t>(nblk, kNumSMs * 4) * 8, st_);
    scal_.ensure(4 * 8, st_);
    xx_.ensure(8, st_);
    loss_need_.ensure(8, st_);
    yq_.ensure(2 * (d_ + 1) * 8, st_);
    ensure_hist((size_t)std::max<uint32_t>(opt_.max_iterations, 1) * (N_ + 1));
    init_loss_.ensure(16, st_);
    uint64_t sum_rows = 0;
    for (auto s : shape_) sum_rows += s;
    scores_.ensure(sum_rows * 8, st_);
    cdf_.ensure(sum_rows * 8, st_);
    sums_.ensure(8 * 8, st_);
    score_off_.ensure(8 * 8, st_);
    rows_dev_.ensure(8 * 4, st_);
    cols_dev_.ensure(8 * 4, st_);
    flag_.ensure(4, st_);
    chol_status_.ensure(4, st_);
    data_draws_.ensure(8, st_);
    zero_flag_.ensure(4, st_);
    RTB_CUDA(cudaMemsetAsync(data_draws_.p, 0, 8, st_));
    long long offs[8] = {0};
    int rows[8] = {0}, cols[8] = {0};
    long long o = 0;
    for (int n = 0; n < N_; ++n) {
      offs[n] = o;
      o += (long long)shape_[n];
      rows[n] = (int)shape_[n];
      cols[n] = (int)ranks_[n];
    }
    RTB_CUDA(cudaMemcpyAsync(score_off_.p, offs, 8 * 8, cudaMemcpyHostToDevice, st_));
    RTB_CUDA(cudaMemcpyAsync(rows_dev_.p, rows, 8 * 4, cudaMemcpyHostToDevice, st_));
    RTB_CUDA(cudaMemcpyAsync(cols_dev_.p, cols, 8 * 4, cudaMemcpyHostToDevice, st_));
    int ns[64];
    for (int i = 0; i < 64; ++i) ns[i] = i < N_ ? (int)ranks_[i] : 1;
    RTB_CUDA(cudaMemcpyAsync(ns_.p, ns, 64 * 4, cudaMemcpyHostToDevice, st_));
    seed_dev_.ensure(16 * 8, st_);
    ctr_dev_.ensure(2 * 8, st_);
    post_.ensure(8 * 4, st_);
    warm_dev_.ensure(4, st_);
    loss_rows_.ensure((size_t)(N_ + 1) * 16, st_);
    RTB_CUDA(cudaMemsetAsync(ctr_dev_.p, 0, 16, st_));
    RTB_CUDA(cudaMemsetAsync(warm_dev_.p, 0, 4, st_));
    post_host_ = pinned_slot();
    for (int k = 0; k < 2 * (N_ + 1); ++k) RTB_CUDA(cudaEventCreate(&step_ev_[k]));
    RTB_CUDA(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming));
    RTB_CUDA(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming));
    RTB_CUDA(cudaEventCreateWithFlags(&dfork_ev_, cudaEventDisableTiming));
    RTB_CUDA(cudaEventCreateWithFlags(&kfork_ev_, cudaEventDisableTiming));
    RTB_CUDA(cudaEventCreateWithFlags(&djoin_ev_, cudaEventDisableTiming));
    {
      int rk[8] = {0};
      for (int n = 0; n < N_; ++n) rk[n] = (int)ranks_[n];
      pcg_path_ = opt_.core_solver == 0 && opt_.lambda > 0.0 && rmax_ <= 32 &&
                  pcg_supported((int)d_, N_, rk);
    }
    RTB_CUDA(cudaStreamSynchronize(st_));  // host arrays above go out of scope
  }

  // A_n^T A_n
  void factor_gram(int n) {
    Scope sc(prof_, "factor_gram");
    const int R = (int)ranks_[n];
    FactorSet fs = factor_set();
    // launch for a single mode: offset the set
    FactorSet one{};
    one.order = 1;
    one.ptr[0] = fs.ptr[n];
    one.rows[0] = fs.rows[n];
    one.cols[0] = fs.cols[n];
    dim3 grid(R * R, 1);
    // the kernel indexes grams by mode; write into slot 0 of a view at gram(n)
    k_factor_gram<<<grid, 256, 0, st_>>>(one, gram(n), R);
    RTB_LAUNCH_CHECK();
  }

  // generic mode product on a tensor with dims `dims`: mode m, matrix W (Rn x dims[m])
  // given by strides; writes `out`, updates dims[m] = Rn.
  void mode_product(const double* in, std::vector<uint64_t>& dims, int m, const double* W,
                    long long wr, long long wi, int Rn, double* out, bool w_is_At) {
    const long long O = (long long)prod(dims, 0, m);
    const int I = (int)dims[m];
    const long long J = (long long)prod(dims, m + 1);
    // DMMA paths whenever the reduction is long enough to matter; the scalar
    // generic kernel only for tiny contractions
    const bool dmma = w_is_At && Rn <= 32 && I >= 16 && O * I * J >= 4096;
    if (dmma) {
      if (J == 1) {
        Scope sc(prof_, "ttm_last");
        ttm_last(in, O, I, W, Rn, out, nullptr, nullptr, st_);
      } else if (J >= 2) {
        Scope sc(prof_, "ttm_mid");
        ttm_mid(in, O, I, J, W, Rn, out, st_);
      } else {
        Scope sc(prof_, "ttm_generic");
        ttm_generic(in, O, I, J, W, wr, wi, Rn, out, st_);
      }
    } else {
      Scope sc(prof_, "ttm_generic");
      ttm_generic(in, O, I, J, W, wr, wi, Rn, out, st_);
    }
    dims[m] = Rn;
  }

  // Y for factor n: dims with I_n at n and R_m elsewhere. Returns pointer into tmp.
  const double* factor_projection(int n, std::vector<uint64_t>& dims) {
    dims = lshape_;
    const double* cur = x_;
    double* bufs[2] = {tmp_a_.as<double>(), tmp_b_.as<double>()};
    int which = 0;
    std::vector<int> modes;
    if (n != N_ - 1) {
      if (!t_valid_) compute_T();
      cur = T_.as<double>();
      dims[N_ - 1] = ranks_[N_ - 1];
      for (int m = 0; m < N_ - 1; ++m)
        if (m != n) modes.push_back(m);
    } else {
      for (int m = 0; m < N_ - 1; ++m) modes.push_back(m);
    }
    bool partial = false;
    for (int m : modes) {
      const int R = (int)ranks_[m];
      // mode 1 is sharded: contract with this shard's rows of A_1 -> partial sum
      const double* W = factor(m) + (m == 0 ? (size_t)lo_ * R : 0);
      mode_product(cur, dims, m, W, 1, R, R, bufs[which], true);
      partial |= (m == 0);
      cur = bufs[which];
      which ^= 1;
    }
    if (partial && sharded()) allreduce(const_cast<double*>(cur), prod(dims));
    return cur;
  }

  void compute_T() {
    // T = X x_N A_N^T (O x R_N, this shard's rows), no residual
    const long long O = (long long)(ltotal_ / shape_[N_ - 1]);
    const int I = (int)shape_[N_ - 1], R = (int)ranks_[N_ - 1];
    if (R <= 32) {
      Scope sc(prof_, "ttm_last");
      ttm_last(x_, O, I, factor(N_ - 1), R, T_.as<double>(), nullptr, nullptr, st_);
    } else {
      Scope sc(prof_, "ttm_generic");
      ttm_generic(x_, O, I, 1, factor(N_ - 1), 1, R, R, T_.as<double>(), st_);
    }
    t_valid_ = true;
  }

  // ---- exact factor update (ref tucker.cpp:70-89) ----
  void update_factor(int n) {
    // mode 1 under sharding: this shard computes its own rows of A_1
    const int In = (n == 0) ? (int)nloc_ : (int)shape_[n], Rn = (int)ranks_[n];
    double* pv = pinv2_.as<double>();
    // (KK^T + lambda I)^+ with KK^T = G_(n) (kron_{m!=n} A_m^T A_m) G_(n)^T does not depend on
    // the projection of X (or T) below, so it runs on the side stream -- a parallel branch of
    // the sweep's graph -- while the projection and M = Y_(n) G_(n)^T run on the main stream
    {
      double* qb[2] = {scratch_q(0), scratch_q(1)};  // allocated in main-stream order
      const cudaStream_t ss = fork();
      Scope sc(prof_, "small_linalg");
      double* kk = pinv_.as<double>();
      static const bool no_fused = std::getenv("RTB_NO_FU_KKT") != nullptr;  // experiments
      if (!no_fused && N_ == 3 && rmax_ <= 32) {
        k_fu_kkt3<<<Rn, 256, 0, ss>>>(core_.as<double>(), grams_.as<double>(), eig_stride_, n,
                                      (int)ranks_[0], (int)ranks_[1], (int)ranks_[2], opt_.lambda,
                                      kk);
        RTB_LAUNCH_CHECK();
      } else {
        std::vector<uint64_t> gd = ranks_;
        const double* cur = core_.as<double>();
        int which = 0;
        for (int m = 0; m < N_; ++m) {
          if (m == n) continue;
          const int R = (int)ranks_[m];
          ttm_generic(cur, (long long)prod(gd, 0, m), R, (long long)prod(gd, m + 1), gram(m), R, 1,
                      R, qb[which], ss);
          cur = qb[which];
          which ^= 1;
        }
        const long long O = (long long)prod(ranks_, 0, n);
        const long long J = (long long)prod(ranks_, n + 1);
        contract_except(core_.as<double>(), cur, O, Rn, Rn, J, kk, ss);
        k_add_diag<<<ceil_div(Rn, 64), 64, 0, ss>>>(kk, Rn, opt_.lambda);
        RTB_LAUNCH_CHECK();
      }
      // (KK^T + lambda I)^+ (ref linalg.cpp:8-26): warp Cholesky inverse; if a
      // pivot is below R*eps*max diag the eigen/pinv path (singular values =
      // |eigenvalues|, cutoff R*eps*sigma_max) takes over on the device.
      int* okf = fu_ok_.as<int>();
      const int stride = std::max(eig_stride_, Rn * Rn);
      if (Rn <= 32) {
        spd_small(kk, ns_one(Rn), stride, (double)Rn * DBL_EPSILON, fu_linv_.as<double>(), pv, okf,
                  1, ss, Rn);
        sym_eigen(kk, ns_one(Rn), Rn, stride, fu_evals_.as<double>(), fu_evecs_.as<double>(),
                  fu_status_.as<int>(), 1, ss, okf);
        k_sym_pinv<<<1, 256, 0, ss>>>(fu_evals_.as<double>(), fu_evecs_.as<double>(), ns_one(Rn),
                                       stride, pv, nullptr, okf);
      } else {
        eigen_one(kk, Rn, ss);
        k_sym_pinv<<<1, 256, 0, ss>>>(evals_.as<double>(), evecs_.as<double>(), ns_one(Rn),
                                       stride, pv, nullptr, nullptr);
      }
      RTB_LAUNCH_CHECK();
    }
    // M = Y_(n) G_(n)^T  (I_n x R_n); order 3, modes 1-2, one shard: projection and
    // contraction from T in one launch (k_fu_proj3)
    double* M = tmp_b_.as<double>();
    bool fused = false;
    if (N_ == 3 && n < 2 && !sharded()) {
      if (!t_valid_) compute_T();
      Scope sc(prof_, "ttm_mid");
      const int m = 1 - n;
      fused = fu_proj3(T_.as<double>(), (int)shape_[0], (int)shape_[1], (int)ranks_[2], factor(m),
                       (int)ranks_[m], core_.as<double>(), (int)ranks_[0], (int)ranks_[1], n, M,
                       st_);
    }
    if (!fused) {
      std::vector<uint64_t> dims;
      const double* Y = factor_projection(n, dims);
      M = (Y == tmp_a_.as<double>()) ? tmp_b_.as<double>() : tmp_a_.as<double>();
      Scope sc(prof_, "contract");
      contract_except(Y, core_.as<double>(), (long long)prod(ranks_, 0, n), In, Rn,
                      (long long)prod(ranks_, n + 1), M, st_);
    }
    join();
    {
      Scope sc(prof_, "small_linalg");
      // A_n = M pinv
      const long long tot = (long long)In * Rn;
      if (n == 0 && sharded()) {
        // own rows into a zeroed full-size A_1, then sum over shards = the whole A_1
        double* a1 = factor(0);
        RTB_CUDA(cudaMemsetAsync(a1, 0, shape_[0] * Rn * 8, st_));
        k_rows_times_small<<<ceil_div<long long>(tot, 256), 256, 0, st_>>>(
            M, pv, In, Rn, a1 + (size_t)lo_ * Rn);
        RTB_LAUNCH_CHECK();
        allreduce(a1, shape_[0] * Rn);
      } else {
        k_rows_times_small<<<ceil_div<long long>(tot, 256), 256, 0, st_>>>(M, pv, In, Rn,
                                                                          factor(n));
        RTB_LAUNCH_CHECK();
      }
    }
    factor_gram(n);
    if (n == N_ - 1) t_valid_ = false;
  }

  // ---- side stream: independent work as a parallel branch (fork / join on events) ----
  // Work on the side stream only launches kernels into buffers allocated beforehand on the
  // main stream (every DevBuf is allocated and freed in main-stream order); the side stream
  // itself is per device and lives as long as the process.
  cudaEvent_t fork_ev_ = nullptr, join_ev_ = nullptr;
  // the core sketch's stream decode, run ahead as a second side branch (decode_ahead)
  cudaEvent_t dfork_ev_ = nullptr, djoin_ev_ = nullptr;
  bool decoded_ahead_ = false;
  DevBuf cdraw_work_;
  // keys ahead: mode-1 scores, the Gram's bucket keys and their sort on the same side branch
  // after F1 (order 3, exact factor updates); the first normal_eq of the core step skips them
  cudaEvent_t kfork_ev_ = nullptr;
  bool keys_ahead_ = false, keys_ready_ = false;
  bool forked_ = false;
  bool blocks_ready_ = false;  // the last normal_eq wrote blocks_ (fused contraction epilogue)
  // returns the stream for the branch: the side stream, or the main one when profiling
  cudaStream_t fork() {
    if (opt_.profile || !fork_ev_) return st_;
    const cudaStream_t side = side_stream();
    RTB_CUDA(cudaEventRecord(fork_ev_, st_));
    RTB_CUDA(cudaStreamWaitEvent(side, fork_ev_, 0));
    forked_ = true;
    return side;
  }
  void join() {
    if (!forked_) return;
    RTB_CUDA(cudaEventRecord(join_ev_, side_stream()));
    RTB_CUDA(cudaStreamWaitEvent(st_, join_ev_, 0));
    forked_ = false;
  }

  DevBuf qbuf_[2];
  double* scratch_q(int i) {
    qbuf_[i].ensure((std::max<uint64_t>(d_, (uint64_t)rmax_ * rmax_) + 1) * 8, st_);
    return qbuf_[i].as<double>();
  }
  // device array {0, 1, ..., 64}: ns_one(n) points at the value n
  int* ns_one(int n) { return ns_vals_.as<int>() + n; }

  // eigen of one symmetric n x n matrix (device) into slot 0 of evals/evecs
  void eigen_one(const double* m, int n, cudaStream_t st = nullptr) {
    sym_eigen(m, ns_one(n), n, eig_stride_ > n * n ? eig_stride_ : n * n, evals_.as<double>(),
              evecs_.as<double>(), eig_status_.as<int>(), 1, st ? st : st_);
  }

  // eigen of all factor Grams (batched)
  void eigen_grams() {
    sym_eigen(grams_.as<double>(), ns_.as<int>(), rmax_, eig_stride_, evals_.as<double>(),
              evecs_.as<double>(), eig_status_.as<int>(), N_, st_);
  }

  // ---- sketched core (ref tucker.cpp:141-166, sketch_ridge.cpp:52-151) ----
  uint64_t core_sample_count() const {
    uint64_t s = opt_.sample_override;
    if (s == 0) s = sample_count_formula(0.5, d_, opt_.epsilon, opt_.delta);
    return s;
  }
  DrawSpec core_draw_spec(uint64_t s, uint64_t seed, const unsigned long long* seed_dev) {
    DrawSpec ds{};
    ds.order = N_;
    long long off = 0;
    for (int n = 0; n < N_; ++n) {
      ds.rows[n] = (long long)shape_[n];
      ds.cdf_off[n] = off;
      off += (long long)shape_[n];
    }
    ds.total_rows = total_;
    ds.d = d_;
    ds.seed = seed;
    ds.seed_dev = seed_dev;
    ds.s = s;
    sk_idx_.ensure(s * 8, st_);
    sk_w_.ensure(s * 8, st_);
    // its own workspace: the perf mode's factor sketches reuse draw_work_ while the core
    // sketch's decode runs ahead on a side stream
    cdraw_work_.ensure(draw_work_bytes(ds), st_);
    return ds;
  }

  // The core sketch's stream decode (draw positions: seed, s, d and N only) as a side branch
  // from the start of the sweep, overlapping the factor updates; update_core_sketched joins it.
  void decode_ahead(const unsigned long long* seed_dev) {
    static const bool off = std::getenv("RTB_NO_DECODE_AHEAD") != nullptr;  // experiments
    if (off || !dfork_ev_ || !opt_.sketched) return;
    const DrawSpec ds = core_draw_spec(core_sample_count(), 0, seed_dev);
    // profiled runs keep the same kernels, in line on the main stream (per-family events)
    const cudaStream_t side = opt_.profile ? st_ : side_stream(1);
    if (!opt_.profile) {
      RTB_CUDA(cudaEventRecord(dfork_ev_, st_));
      RTB_CUDA(cudaStreamWaitEvent(side, dfork_ev_, 0));
    }
    {
      Scope sc(prof_, "draw");
      draw_decode(ds, DrawWork{cdraw_work_.p, cdraw_work_.bytes}, side);
    }
    RTB_CUDA(cudaEventRecord(djoin_ev_, side));
    decoded_ahead_ = true;
  }

  // After F1 (A_1 final): on the decode branch, A_1's scores and CDF, every draw's bucket key
  // from A_1's CDF alone (k_draw_keys), the stable key sort, the bucket table and the bucket
  // order -- the Gram's whole sort stage leaves the critical path (it overlaps F2 and F3).
  void keys_ahead() {
    static const bool off = std::getenv("RTB_NO_KEYS_AHEAD") != nullptr;  // experiments
    if (off || !decoded_ahead_ || N_ != 3 || opt_.factor_samples > 0 || rmax_ > 32) return;
    const uint64_t s = core_sample_count();
    const GramSpec gs = gram_spec(s);
    gram_work_.ensure(gram_work_bytes(gs), st_);
    const DrawSpec ds = core_draw_spec(s, 0, seed_dev_.as<unsigned long long>());
    const cudaStream_t side = opt_.profile ? st_ : side_stream(1);
    if (!opt_.profile) {
      RTB_CUDA(cudaEventRecord(kfork_ev_, st_));
      RTB_CUDA(cudaStreamWaitEvent(side, kfork_ev_, 0));
    }
    compute_scores_range(0, 1, side);
    {
      Scope sc(prof_, "gram_sort");
      const GramKeyBufs kb = gram_key_buffers(gs, gram_work_.p);
      gram_keys_reset(gs, gram_work_.p, (unsigned long long*)data_draws_.p, side);
      draw_keys(ds, scores_.as<double>(), cdf_.as<double>(), sums_.as<double>(),
                DrawWork{cdraw_work_.p, cdraw_work_.bytes}, gs.i1_lo, gs.i1_hi, kb.keys, kb.vals,
                kb.counts, kb.aug_count, (unsigned long long*)data_draws_.p, side);
      gram_sort_keys(gs, gram_work_.p, side);
    }
    RTB_CUDA(cudaEventRecord(djoin_ev_, side));
    keys_ahead_ = true;
  }

  void update_core_sketched(uint64_t seed, const unsigned long long* seed_dev = nullptr,
                            bool defer = false) {
    const uint64_t s = core_sample_count();
    last_s_ = s;
    if (keys_ahead_ && seed_dev) {
      // mode 1's scores came with the keys: join that branch, then the other modes
      RTB_CUDA(cudaStreamWaitEvent(st_, djoin_ev_, 0));
      compute_scores_range(1, N_, st_);
      keys_ready_ = true;
    } else {
      compute_scores();
    }
    keys_ahead_ = false;
    const DrawSpec ds = core_draw_spec(s, seed, seed_dev);
    RTB_CUDA(cudaMemsetAsync(flag_.p, 0, 4, st_));
    {
      Scope sc(prof_, "draw");
      const DrawWork dw{cdraw_work_.p, cdraw_work_.bytes};
      if (decoded_ahead_ && seed_dev) {
        RTB_CUDA(cudaStreamWaitEvent(st_, djoin_ev_, 0));
        draw_evaluate(ds, scores_.as<double>(), cdf_.as<double>(), sums_.as<double>(), dw,
                      (unsigned long long*)sk_idx_.p, sk_w_.as<double>(), flag_.as<int>(), st_);
      } else {
        draw_sketch(ds, scores_.as<double>(), cdf_.as<double>(), sums_.as<double>(), dw,
                    (unsigned long long*)sk_idx_.p, sk_w_.as<double>(), flag_.as<int>(), st_);
      }
      decoded_ahead_ = false;
    }
    solve_sketch(s, defer);
  }

  // ---- sketched factor update (perf mode; k_fsketch.cu, orc_update_factor_sketched) ----
  void update_factor_sketched(int n, uint64_t seed,
                              const unsigned long long* seed_dev = nullptr) {
    // under sharding (X split along mode 1): mode 1's fibers are this shard's segments (own
    // rows of A_1, stitched by a zero-padded all-reduce as in update_factor); the other
    // modes' Gram and M are partial sums over this shard's draws, all-reduced
    const int Rn = (int)ranks_[n], In = (n == 0) ? (int)nloc_ : (int)shape_[n];
    if (Rn > 32) {  // the register-tiled gather kernel covers R_n <= 32
      update_factor(n);
      return;
    }
    const uint64_t s = opt_.factor_samples;
    compute_scores();
    DrawSpec ds{};
    ds.order = N_ - 1;
    uint64_t total_o = 1;
    long long off = 0;
    int k = 0;
    for (int m = 0; m < N_; ++m) {
      if (m != n) {
        ds.rows[k] = (long long)shape_[m];
        ds.cdf_off[k] = off;
        total_o *= shape_[m];
        ++k;
      }
      off += (long long)shape_[m];
    }
    ds.total_rows = total_o;
    ds.d = (uint64_t)Rn;
    ds.seed = seed;
    ds.seed_dev = seed_dev;
    ds.s = s;
    fsums_.ensure(8 * 8, st_);
    // score sums of the other modes, in order
    if (n > 0)
      RTB_CUDA(cudaMemcpyAsync(fsums_.p, sums_.p, n * 8, cudaMemcpyDeviceToDevice, st_));
    if (n < N_ - 1)
      RTB_CUDA(cudaMemcpyAsync(fsums_.as<double>() + n, sums_.as<double>() + n + 1,
                               (N_ - 1 - n) * 8, cudaMemcpyDeviceToDevice, st_));
    fsk_idx_.ensure(s * 8, st_);
    fsk_w_.ensure(s * 8, st_);
    draw_work_.ensure(draw_work_bytes(ds), st_);
    RTB_CUDA(cudaMemsetAsync(flag_.p, 0, 4, st_));
    {
      Scope sc(prof_, "draw");
      draw_sketch(ds, scores_.as<double>(), cdf_.as<double>(), fsums_.as<double>(),
                  DrawWork{draw_work_.p, draw_work_.bytes}, (unsigned long long*)fsk_idx_.p,
                  fsk_w_.as<double>(), flag_.as<int>(), st_);
    }
    FactorSketchSpec fs{};
    fs.order = N_;
    fs.mode = n;
    for (int m = 0; m < N_; ++m) {
      fs.rows[m] = (int)shape_[m];
      fs.ranks[m] = (int)ranks_[m];
      fs.factors[m] = factor(m);
    }
    fs.core = core_.as<double>();
    fs.x = x_;
    if (sharded()) {
      fs.shard_lo = (int)lo_;
      fs.shard_rows = (int)nloc_;
      fs.count_aug = opt_.shard_rank == 0 ? 1 : 0;
    }
    // mode-n-last copy of this shard's X (made once per engine): every sampled fiber is
    // contiguous
    if (n != N_ - 1 && xrot_ok_) {
      if (!xrot_[n].p) {
        try {
          xrot_[n].ensure(ltotal_ * 8, st_);
          move_axis_last(x_, (long long)prod(lshape_, 0, n), (int)lshape_[n],
                         (long long)prod(lshape_, n + 1), xrot_[n].as<double>(), st_);
        } catch (const Error&) {
          cudaGetLastError();
          xrot_[n] = DevBuf();
          xrot_ok_ = false;  // no room: keep the strided gathers
        }
      }
      if (xrot_[n].p) {
        fs.x = xrot_[n].as<double>();
        fs.x_mode_last = 1;
      }
    }
    fs.lambda = opt_.lambda;
    fs.s = s;
    fsk_work_.ensure(factor_sketch_work_bytes(fs), st_);
    double* kk = pinv_.as<double>();
    double* M = tmp_a_.as<double>();
    {
      Scope sc(prof_, "factor_sketch");
      factor_sketch_normal_eq(fs, (const unsigned long long*)fsk_idx_.p, fsk_w_.as<double>(),
                              fsk_work_.p, kk, M, st_);
      if (sharded() && n > 0) {  // partial sums over this shard's draws
        allreduce(kk, (size_t)Rn * Rn);
        allreduce(M, (size_t)In * Rn);
      }
    }
    {
      // A_n = M pinv(Gram) (ref sketch_ridge.cpp:130-139 per fiber row), as in update_factor
      Scope sc(prof_, "small_linalg");
      double* pv = pinv2_.as<double>();
      int* okf = fu_ok_.as<int>();
      const int stride = std::max(eig_stride_, Rn * Rn);
      spd_small(kk, ns_one(Rn), stride, (double)Rn * DBL_EPSILON, fu_linv_.as<double>(), pv, okf, 1,
                st_, Rn);
      if (std::getenv("RTB_DEBUG_FSK_SPD")) {
        int okh = -1;
        std::vector<double> kh((size_t)Rn * Rn);
        RTB_CUDA(cudaMemcpyAsync(&okh, okf, 4, cudaMemcpyDeviceToHost, st_));
        RTB_CUDA(cudaMemcpyAsync(kh.data(), kk, kh.size() * 8, cudaMemcpyDeviceToHost, st_));
        RTB_CUDA(cudaStreamSynchronize(st_));
        std::fprintf(stderr, "[fsk] mode %d ok %d diag %.3e %.3e offd %.3e sym %.3e\n", n, okh,
                     kh[0], kh[(size_t)Rn * Rn - 1], kh[1], kh[1] - kh[Rn]);
      }
      sym_eigen(kk, ns_one(Rn), Rn, stride, fu_evals_.as<double>(), fu_evecs_.as<double>(),
                fu_status_.as<int>(), 1, st_, okf);
      k_sym_pinv<<<1, 256, 0, st_>>>(fu_evals_.as<double>(), fu_evecs_.as<double>(), ns_one(Rn),
                                     stride, pv, nullptr, okf);
      RTB_LAUNCH_CHECK();
      const long long tot = (long long)In * Rn;
      if (n == 0 && sharded()) {
        // own rows into a zeroed full-size A_1, then the sum over shards is the whole A_1
        double* a1 = factor(0);
        RTB_CUDA(cudaMemsetAsync(a1, 0, shape_[0] * Rn * 8, st_));
        k_rows_times_small<<<ceil_div<long long>(tot, 256), 256, 0, st_>>>(M, pv, In, Rn,
                                                                          a1 + (size_t)lo_ * Rn);
        RTB_LAUNCH_CHECK();
        allreduce(a1, shape_[0] * Rn);
      } else {
        k_rows_times_small<<<ceil_div<long long>(tot, 256), 256, 0, st_>>>(M, pv, In, Rn,
                                                                          factor(n));
        RTB_LAUNCH_CHECK();
      }
    }
    factor_gram(n);
    scores_valid_ = false;
    if (n == N_ - 1) t_valid_ = false;
  }

  // per-mode classical leverage scores, CDFs and sums of the current factors
  void compute_scores() { compute_scores_range(0, N_, st_); }

  // scores, CDFs and sums of modes [n0, n1) on stream `st`; the zero-rank flag when n1 == N
  void compute_scores_range(int n0, int n1, cudaStream_t st) {
    {
      Scope sc(prof_, "scores");
      // classical scores l_i = a_i^T (A^T A)^+ a_i: Cholesky of each factor Gram
      // (||L^-1 a_i||^2); where a Gram's Cholesky meets a pivot below max(I, R) eps (so
      // sigma_min / sigma_max may be small enough for the reference's cut), the
      // reference's own route: one-sided Jacobi SVD of the factor and the rank cut on its
      // singular values (k_hj_cta; ref kronecker.cpp:18-23, svd.cpp:69-111,
      // leverage.cpp:16-37 at lambda = 0)
      const FactorSet all = factor_set();
      FactorSet fs{};
      const int cnt = n1 - n0;
      fs.order = cnt;
      for (int k = 0; k < cnt; ++k) {
        fs.ptr[k] = all.ptr[n0 + k];
        fs.rows[k] = all.rows[n0 + k];
        fs.cols[k] = all.cols[n0 + k];
      }
      int maxI = 0;
      for (int n = n0; n < n1; ++n) maxI = std::max<int>(maxI, (int)shape_[n]);
      const int* okm = nullptr;
      dim3 grid(ceil_div(maxI, 128), cnt);
      const size_t so = (size_t)n0 * eig_stride_;
      long long* soff = score_off_.as<long long>() + n0;
      int* rkd = ranks_dev_.as<int>() + n0;
      if (rmax_ <= 32) {
        spd_small(grams_.as<double>() + so, ns_.as<int>() + n0, eig_stride_,
                  (double)maxI * DBL_EPSILON, linv_.as<double>() + so, pgram_.as<double>() + so,
                  spd_ok_.as<int>() + n0, cnt, st, rmax_);
        okm = spd_ok_.as<int>() + n0;
        long long stride = 0;
        for (int n = 0; n < N_; ++n)
          stride = std::max<long long>(stride, (long long)shape_[n] * (ranks_[n] + (ranks_[n] & 1)));
        hj_ws_.ensure((size_t)N_ * stride * 8 + 64, st_);
        k_hj_cta<<<cnt, 512, 0, st>>>(fs, hj_ws_.as<double>() + (size_t)n0 * stride, stride, 0.0,
                                      scores_.as<double>(), soff, rkd, okm,
                                      eig_status_.as<int>() + n0);
        RTB_LAUNCH_CHECK();
      } else {
        sym_eigen(grams_.as<double>() + so, ns_.as<int>() + n0, rmax_, eig_stride_,
                  evals_.as<double>() + so, evecs_.as<double>() + so, eig_status_.as<int>() + n0,
                  cnt, st, okm);
        k_leverage_rows<<<grid, 128, 0, st>>>(fs, evals_.as<double>() + so,
                                             evecs_.as<double>() + so, eig_stride_, 0.0,
                                             scores_.as<double>(), soff, rkd, okm);
        RTB_LAUNCH_CHECK();
      }
      if (okm) {
        leverage_chol(fs, linv_.as<double>() + so, eig_stride_, okm, scores_.as<double>(), soff,
                      rkd, maxI, cnt, rmax_, st);
      }
      k_score_cdf<<<cnt, 256, 0, st>>>(scores_.as<double>(), soff, rows_dev_.as<int>() + n0, cnt,
                                       cdf_.as<double>(), sums_.as<double>() + n0);
      RTB_LAUNCH_CHECK();
      if (n1 == N_) {
        k_any_zero_rank<<<1, 32, 0, st>>>(ranks_dev_.as<int>(), N_, zero_flag_.as<int>());
        RTB_LAUNCH_CHECK();
      }
    }
  }

  GramSpec gram_spec(uint64_t s) {
    GramSpec gs{};
    gs.order = N_;
    for (int n = 0; n < N_; ++n) {
      gs.rows[n] = (int)shape_[n];
      gs.ranks[n] = (int)ranks_[n];
      gs.factors[n] = factor(n);
    }
    gs.total_rows = total_;
    gs.d = (int)d_;
    gs.dprime = (int)(d_ / ranks_[0]);
    gs.lambda = opt_.lambda;
    gs.s = s;
    gs.i1_lo = sharded() ? (int)lo_ : 0;
    gs.i1_hi = sharded() ? (int)(lo_ + nloc_) : 0;
    return gs;
  }

 public:
  // normal equations from sk_idx_/sk_w_ (s draws) and solve into the core. With `defer`
  // (a sweep) and the PCG path, nothing waits here: k_core_post writes the verdict (PCG
  // status, zero-factor flag, finiteness of the core) to pinned host memory and the
  // caller's resolve_core() acts on it; otherwise the verdict is resolved right away.
  void solve_sketch(uint64_t s, bool defer = false) {
    GramSpec gs = gram_spec(s);
    gram_work_.ensure(gram_work_bytes(gs), st_);
    rhs_.ensure(d_ * 8, st_);
    int rk[8];
    for (int n = 0; n < N_; ++n) rk[n] = (int)ranks_[n];
    last_s_ = s;
    PcgSpec ps{};
    double* prep = reinterpret_cast<double*>(pst_.as<int>() + 64);
    if (pcg_path_) {
      ps.order = N_;
      for (int n = 0; n < N_; ++n) ps.ranks[n] = rk[n];
      ps.d = (int)d_;
      ps.lambda = opt_.lambda;
      ps.pinv = pgram_.as<double>();  // (A_n^T A_n)^-1 from the score step's Cholesky
      ps.linv_stride = eig_stride_;
      ps.linv_ok = spd_ok_.as<int>();
      ps.grams = grams_.as<double>();
      // the Kronecker preconditioner depends on the factor Grams only: a parallel branch
      // next to the sketched Gram build
      const cudaStream_t ss = fork();
      Scope sc(prof_, "pcg");
      int* eskip = pst_.as<int>() + 32;
      pcg_prepare(ps, prep, eskip, ss);
      sym_eigen(grams_.as<double>(), ns_.as<int>(), rmax_, eig_stride_, pev_.as<double>(),
                pvec_.as<double>(), pst_.as<int>(), N_, ss, eskip);
    }
    // the split-role PCG keeps the compact Gram in shared memory: no block expansion (under
    // sharding it reads the all-reduced compact Gram, the same buffer)
    const bool split = pcg_path_ && pcg_split_ok((int)d_, N_, rk);
    normal_eq(s, !pcg_path_, !split);
    if (!pcg_path_) {
      solve_fallback(s, false);
      return;
    }
    {
      // Kronecker-preconditioned CG on the blocked Gram (k_pcg.cu), verified by its
      // true residual; the Cholesky path (solve_fallback) takes over on failure
      Scope sc(prof_, "pcg");
      // multi-GPU with a large d: the solve is distributed by mode-1 slices (pcg_solve_dist),
      // each shard expands and multiplies its own slices' blocks only
      const bool dist = sharded() && pcg_dist_ok((int)d_, N_, rk);
      int u_lo = 0, u_hi = 0;
      if (dist) {
        const int m1 = rk[0] * (rk[0] + 1) / 2;
        pcg_dist_slices(m1, (int)opt_.shard_rank, (int)opt_.shard_count, &u_lo, &u_hi);
        const long long per = gram_block_elems(gs) / m1;
        blocks_.ensure((size_t)std::max<long long>(1, per * (u_hi - u_lo)) * 8, st_);
        gram_expand_blocks_range(gs, gram_work_.p, blocks_.as<double>(), u_lo, u_hi, st_);
      } else if (!split && !blocks_ready_) {
        blocks_.ensure((size_t)gram_block_elems(gs) * 8, st_);
        gram_expand_blocks(gs, gram_work_.p, blocks_.as<double>(), st_);
      }
      join();
      ps.evals = pev_.as<double>();
      ps.evecs = pvec_.as<double>();
      ps.prep = prep;
      ps.aug_count = gram_aug_counts(gs, gram_work_.p);
      ps.aug_term = gram_aug_term(gs);
      ps.max_iter = 80;
      ps.tol = 1e-15;
      ps.check_tol = 1e-12;
      // warm start from the current core (the previous accepted solve's solution; the
      // first sketch of a run starts cold from the random init): a device flag
      ps.warm_dev = warm_dev_.as<int>();
      pcg_work_.ensure(pcg_work_bytes((int)d_, N_, rk), st_);
      if (dist)
        pcg_solve_dist(ps, blocks_.as<double>(), (int)opt_.shard_rank, (int)opt_.shard_count,
                       rhs_.as<double>(), core_.as<double>(), pcg_work_.p, pcg_status_.as<int>(),
                       st_, [this](double* p, size_t n) { allreduce(p, n); });
      else if (split)
        pcg_solve_compact(ps, gram_compact(gs, gram_work_.p, nullptr), rhs_.as<double>(),
                          core_.as<double>(), pcg_work_.p, pcg_status_.as<int>(), st_);
      else
        pcg_solve(ps, blocks_.as<double>(), rhs_.as<double>(), core_.as<double>(), pcg_work_.p,
                  pcg_status_.as<int>(), st_);
    }
    k_core_post<<<1, 1024, 0, st_>>>(core_.as<double>(), (long long)d_, pcg_status_.as<int>(),
                                     zero_flag_.as<int>(), warm_dev_.as<int>(), post_.as<int>());
    RTB_LAUNCH_CHECK();
    RTB_CUDA(cudaMemcpyAsync(post_host_, post_.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, st_));
    if (defer) {
      deferred_core_ = true;
      return;
    }
    RTB_CUDA(cudaStreamSynchronize(st_));
    finish_core_solve();
  }

  // Acts on the verdict of a PCG core solve (post_host_, after the stream passed
  // k_core_post). Returns true if the core was recomputed by the fallback path.
  bool finish_core_solve() {
    const int* ps = post_host_;
    last_pcg_iters_ = ps[1];
    if (ps[0] == 0 && !ps[2]) {
      if (ps[3]) throw Error(1, "DenseTensor: non-finite entry");  // ref tensor.cpp:32-42
      last_solver_path_ = 2;
      last_rank_deficient_ = 0;
      return false;
    }
    solve_fallback(last_s_, true);
    return true;
  }

  // sketched normal equations of the current draws (compact Gram in the workspace, rhs;
  // with `full` the d x d Gram in G_ as well)
  void normal_eq(uint64_t s, bool full, bool want_blocks = true) {
    GramSpec gs = gram_spec(s);
    // X slab pointer offset so that global flat indices of this shard's draws land in it
    const double* xg = x_ - (sharded() ? lo_ * (long long)(total_ / shape_[0]) : 0);
    Scope sc(prof_, "gram");
    if (full) G_.ensure(d_ * d_ * 8, st_);
    // the PCG's last-mode blocks come out of the contraction itself when it can write them
    // (one shard only: under sharding they follow the all-reduce of the compact Gram)
    double* bl = nullptr;
    if (!full && !sharded() && want_blocks) {
      blocks_.ensure((size_t)gram_block_elems(gs) * 8, st_);
      bl = blocks_.as<double>();
    }
    // the full Gram is expanded after the shard sum of the compact one
    blocks_ready_ = sketch_normal_eq(gs, xg, (const unsigned long long*)sk_idx_.p,
                                     sk_w_.as<double>(), gram_work_.p, gram_work_.bytes,
                                     (full && !sharded()) ? G_.as<double>() : nullptr,
                                     rhs_.as<double>(), (unsigned long long*)data_draws_.p, st_, bl,
                                     keys_ready_);
    keys_ready_ = false;  // a fallback's second normal_eq sorts again
    if (sharded()) {
      size_t ns = 0;
      double* S = gram_compact(gs, gram_work_.p, &ns);
      allreduce(S, ns);
      allreduce(rhs_.as<double>(), d_);
      if (full) gram_expand_full(gs, gram_work_.p, G_.as<double>(), st_);
    }
  }

  // Cholesky of the full Gram (expanded from the compact one when the PCG path built
  // only the blocks), the zero-core rule and the pinv fallback; synchronous (a rare path
  // after a PCG failure, or the solve itself when CG does not apply)
  void solve_fallback(uint64_t s, bool after_pcg) {
    GramSpec gs = gram_spec(s);
    int status[2] = {0, 0};
    RTB_CUDA(cudaMemcpyAsync(&status[1], zero_flag_.p, 4, cudaMemcpyDeviceToHost, st_));
    RTB_CUDA(cudaStreamSynchronize(st_));
    if (status[1]) {  // a zero factor: the minimiser is the zero core (tucker.cpp:148-154)
      RTB_CUDA(cudaMemsetAsync(core_.p, 0, d_ * 8, st_));
      last_solver_path_ = 0;
      last_rank_deficient_ = 0;
      set_warm(0);
      return;
    }
    if (after_pcg) {
      G_.ensure(d_ * d_ * 8, st_);
      gram_expand_full(gs, gram_work_.p, G_.as<double>(), st_);
    }
    chol_work_.ensure(chol_work_bytes((int)d_), st_);
    {
      Scope sc(prof_, "chol");
      chol_solve(G_.as<double>(), (int)d_, rhs_.as<double>(), chol_status_.as<int>(),
                 chol_work_.p, st_);
    }
    RTB_CUDA(cudaMemcpyAsync(&status[0], chol_status_.p, 4, cudaMemcpyDeviceToHost, st_));
    RTB_CUDA(cudaStreamSynchronize(st_));
    last_solver_path_ = 0;
    last_rank_deficient_ = 0;
    if (status[0]) {
      // not positive definite: recompute the Gram and take the pinv route
      normal_eq(s, true);  // Cholesky overwrote G and rhs: rebuild them
      if (d_ > 64) {  // dense eigen pinv with the reference cutoff (k_pinv.cu)
        Scope sc(prof_, "pinv");
        pinv_work_.ensure(pinv_large_work_bytes((int)d_), st_);
        pinv_rank_.ensure(4, st_);
        pinv_solve_large(G_.as<double>(), (int)d_, rhs_.as<double>(), core_.as<double>(),
                         pinv_rank_.as<int>(), pinv_work_.p, pinv_work_.bytes, st_);
        int rank = 0;
        RTB_CUDA(cudaMemcpyAsync(&rank, pinv_rank_.p, 4, cudaMemcpyDeviceToHost, st_));
        RTB_CUDA(cudaStreamSynchronize(st_));
        last_solver_path_ = 1;
        last_rank_deficient_ = rank < (int)d_;
        set_warm(0);
        check_core_finite();
        return;
      }
      eigen_one(G_.as<double>(), (int)d_);
      double* pv = tmp_a_.as<double>();
      k_sym_pinv<<<1, 256, 0, st_>>>(evals_.as<double>(), evecs_.as<double>(), ns_one((int)d_),
                                     eig_stride_ > (int)(d_ * d_) ? eig_stride_ : (int)(d_ * d_),
                                     pv, ranks_dev_.as<int>(), nullptr);
      RTB_LAUNCH_CHECK();
      k_rows_times_small<<<ceil_div<long long>(d_, 256), 256, 0, st_>>>(rhs_.as<double>(), pv, 1,
                                                                        (int)d_, core_.as<double>());
      RTB_LAUNCH_CHECK();
      int rank = 0;
      RTB_CUDA(cudaMemcpyAsync(&rank, ranks_dev_.p, 4, cudaMemcpyDeviceToHost, st_));
      RTB_CUDA(cudaStreamSynchronize(st_));
      last_solver_path_ = 1;
      last_rank_deficient_ = rank < (int)d_;
      set_warm(0);
    } else {
      RTB_CUDA(cudaMemcpyAsync(core_.p, rhs_.p, d_ * 8, cudaMemcpyDeviceToDevice, st_));
      set_warm(1);
    }
    check_core_finite();
  }

  void set_warm(int v) {
    k_set_int<<<1, 1, 0, st_>>>(warm_dev_.as<int>(), v);
    RTB_LAUNCH_CHECK();
  }

  void check_core_finite() {
    RTB_CUDA(cudaMemsetAsync(flag_.p, 0, 4, st_));
    k_check_finite<<<ceil_div<long long>(d_, 256), 256, 0, st_>>>(core_.as<double>(), d_,
                                                                   flag_.as<int>());
    RTB_LAUNCH_CHECK();
    int bad = 0;
    RTB_CUDA(cudaMemcpyAsync(&bad, flag_.p, 4, cudaMemcpyDeviceToHost, st_));
    RTB_CUDA(cudaStreamSynchronize(st_));
    if (bad) throw Error(1, "DenseTensor: non-finite entry");  // ref tensor.cpp:32-42
  }

 private:
  // ---- exact core (ref tucker.cpp:91-129) ----
  void update_core_exact() {
    Scope sc(prof_, "core_exact");
    eigen_grams();
    k_gram_rank<<<1, 32, 0, st_>>>(evals_.as<double>(), eig_stride_, rows_dev_.as<int>(),
                                   cols_dev_.as<int>(), N_, ranks_dev_.as<int>());
    RTB_LAUNCH_CHECK();
    int rk[8];
    RTB_CUDA(cudaMemcpyAsync(rk, ranks_dev_.p, N_ * 4, cudaMemcpyDeviceToHost, st_));
    RTB_CUDA(cudaStreamSynchronize(st_));
    for (int n = 0; n < N_; ++n)
      if (rk[n] == 0) {
        RTB_CUDA(cudaMemsetAsync(core_.p, 0, d_ * 8, st_));
        return;
      }
    // U_n = A_n V_n Sigma_n^-1 (I_n x r_n)
    for (int n = 0; n < N_; ++n) {
      U_[n].ensure(shape_[n] * rk[n] * 8 + 8, st_);
      const long long tot = (long long)shape_[n] * rk[n];
      k_factor_u<<<ceil_div<long long>(tot, 256), 256, 0, st_>>>(
          factor(n), (int)shape_[n], (int)ranks_[n], evecs_.as<double>() + (size_t)n * eig_stride_,
          evals_.as<double>() + (size_t)n * eig_stride_, ranks_dev_.as<int>() + n,
          U_[n].as<double>());
      RTB_LAUNCH_CHECK();
    }
    // W = X x_n U_n^T, last mode first (contiguous), then the others; mode 1 with this
    // shard's rows of U_1 (partial sum over shards)
    std::vector<uint64_t> dims = lshape_;
    double* bufs[2] = {tmp_a_.as<double>(), tmp_b_.as<double>()};
    int which = 0;
    const double* cur = x_;
    std::vector<int> order;
    order.push_back(N_ - 1);
    for (int m = 0; m < N_ - 1; ++m) order.push_back(m);
    for (int m : order) {
      const double* U = U_[m].as<double>() + (m == 0 ? (size_t)lo_ * rk[0] : 0);
      mode_product(cur, dims, m, U, 1, rk[m], rk[m], bufs[which], true);
      cur = bufs[which];
      which ^= 1;
    }
    allreduce(const_cast<double*>(cur), prod(dims));
    // scale by sigma_t / (sigma_t^2 + lambda)
    ScaleSpec sp{};
    sp.order = N_;
    long long n_el = 1;
    for (int m = 0; m < N_; ++m) {
      sp.dims[m] = rk[m];
      sp.mu[m] = evals_.as<double>() + (size_t)m * eig_stride_;
      n_el *= rk[m];
    }
    k_core_scale<<<ceil_div<long long>(n_el, 256), 256, 0, st_>>>(const_cast<double*>(cur), n_el,
                                                                  sp, opt_.lambda);
    RTB_LAUNCH_CHECK();
    // core = W x_n V_n (V_n: R_n x r_n)
    for (int m = 0; m < N_; ++m) {
      const int R = (int)ranks_[m], r = rk[m];
      double* Vt = scratch_q(0);
      k_transpose_small<<<ceil_div(R * r, 256), 256, 0, st_>>>(
          evecs_.as<double>() + (size_t)m * eig_stride_, R, r, Vt);
      RTB_LAUNCH_CHECK();
      double* out = (m == N_ - 1) ? core_.as<double>() : bufs[which];
      // out[.., i, ..] = sum_k V[i][k] W[.., k, ..]: W_mat(R x r) = Vt row-major (wr=r, wi=1)
      ttm_generic(cur, (long long)prod(dims, 0, m), r, (long long)prod(dims, m + 1), Vt, r, 1, R, out,
                  st_);
      dims[m] = R;
      cur = out;
      which ^= 1;
    }
    check_core_finite();
  }

  // P = G x_1 A_1 ... x_{N-1} A_{N-1}  (last mode stays R_N)
  const double* build_P(std::vector<uint64_t>& dims) {
    dims = ranks_;
    const double* cur = core_.as<double>();
    double* bufs[2] = {tmp_a_.as<double>(), tmp_b_.as<double>()};
    int which = 0;
    for (int m = 0; m < N_ - 1; ++m) {
      // mode 1: this shard's rows only (P rows of the local slab)
      const int I = (m == 0) ? (int)nloc_ : (int)shape_[m], R = (int)ranks_[m];
      const double* A = factor(m) + (m == 0 ? (size_t)lo_ * R : 0);
      double* out = (m == N_ - 2) ? P_.as<double>() : bufs[which];
      // out[.., i, ..] = sum_r A[i][r] cur[.., r, ..]  (W = A: wr = R, wi = 1)
      Scope sc(prof_, "ttm_expand");
      const long long Oe = (long long)prod(dims, 0, m), Je = (long long)prod(dims, m + 1);
      if (!ttm_expand(cur, Oe, R, Je, A, I, out, st_))
        ttm_generic(cur, Oe, R, Je, A, R, 1, I, out, st_);
      dims[m] = I;
      cur = out;
      which ^= 1;
    }
    if (N_ == 1) return core_.as<double>();
    return cur;
  }

  // Loss (ref tucker.cpp:216-229). Default: the direct residual, fused with T. Opt-in
  // fast form (opt_.fast_loss; ~1e-12 ||X||^2 absolute error, so not the default):
  // T = X x_N A_N^T (reused by the next sweep's factor updates), Y = T x_{n<N} A_n^T,
  // Q = G x_n (A_n^T A_n); loss from ||X||^2 - 2<Y,G> + <Q,G>, with the direct
  // residual pass (fused with T) enqueued behind it under a device guard for the
  // near-exact-fit case where the cancellation would cost accuracy.
  void loss_pass(double* loss_dev, double* rmse_dev) {
    const int R = (int)ranks_[N_ - 1];
    if (N_ >= 2 && R <= 32 && opt_.fast_loss && !sharded()) {
      if (!xx_valid_) {
        Scope sc(prof_, "loss_norm_x");
        const int nb = kNumSMs * 4;
        k_sumsq_partials<<<nb, 256, 0, st_>>>(x_, (long long)total_, partial_.as<double>());
        RTB_LAUNCH_CHECK();
        sum_partials(partial_.as<double>(), nb, xx_.as<double>(), st_);
        xx_valid_ = true;
      }
      if (!t_valid_) compute_T();
      double* Y = yq_.as<double>();
      double* Q = Y + d_ + 1;
      {
        Scope sc(prof_, "loss_small");
        // Y = T x_1 A_1^T ... x_{N-1} A_{N-1}^T
        std::vector<uint64_t> dims = shape_;
        dims[N_ - 1] = ranks_[N_ - 1];
        const double* cur = T_.as<double>();
        double* bufs[2] = {tmp_a_.as<double>(), tmp_b_.as<double>()};
        int which = 0;
        for (int m = 0; m < N_ - 1; ++m) {
          double* out = (m == N_ - 2) ? Y : bufs[which];
          mode_product(cur, dims, m, factor(m), 1, (int)ranks_[m], (int)ranks_[m], out, true);
          cur = out;
          which ^= 1;
        }
        // Q = G x_n Gram_n (symmetric R_n x R_n)
        std::vector<uint64_t> gd = ranks_;
        const double* gc = core_.as<double>();
        double* qb[2] = {scratch_q(0), scratch_q(1)};
        int w2 = 0;
        for (int m = 0; m < N_; ++m) {
          const int Rm = (int)ranks_[m];
          double* out = (m == N_ - 1) ? Q : qb[w2];
          ttm_generic(gc, (long long)prod(gd, 0, m), Rm, (long long)prod(gd, m + 1), gram(m), Rm,
                      1, Rm, out, st_);
          gc = out;
          w2 ^= 1;
        }
        double* sc2 = scal_.as<double>();
        norms_into(sc2 + 1);
        k_fast_loss<<<1, 1024, 0, st_>>>(Y, Q, core_.as<double>(), (long long)d_, xx_.as<double>(),
                                         sc2 + 1, opt_.lambda, (double)total_, 1e-5, loss_dev,
                                         rmse_dev, loss_need_.as<int>());
        RTB_LAUNCH_CHECK();
      }
      // direct pass, runs only if k_fast_loss set *need
      set_ttm_guard(loss_need_.as<int>());
      try {
        std::vector<uint64_t> dims;
        const double* P = build_P(dims);
        const long long O = (long long)(total_ / shape_[N_ - 1]);
        const int I = (int)shape_[N_ - 1];
        double* partial = partial_.as<double>();
        {
          Scope sc(prof_, "ttm_last_loss");
          ttm_last(x_, O, I, factor(N_ - 1), R, T_.as<double>(), P, partial, st_);
        }
        double* sc2 = scal_.as<double>();
        sum_partials(partial, ttm_last_blocks(O, I, R), sc2, st_);
      } catch (...) {
        set_ttm_guard(nullptr);
        throw;
      }
      set_ttm_guard(nullptr);
      double* sc2 = scal_.as<double>();
      k_finish_loss_guarded<<<1, 1, 0, st_>>>(sc2, sc2 + 1, opt_.lambda, (double)total_, loss_dev,
                                              rmse_dev, loss_need_.as<int>());
      RTB_LAUNCH_CHECK();
      return;
    }
    const long long O = (long long)(ltotal_ / shape_[N_ - 1]);  // this shard's rows
    const int I = (int)shape_[N_ - 1];
    double* partial = partial_.as<double>();
    long long nparts;
    // the ridge term's norms (core and factors are final here) on a side branch next to the
    // X pass
    norms_into(scal_.as<double>() + 1, fork());
    if (kGenerateP && N_ == 3 && ttm_last_pgen_ok(I, R)) {
      // P rows generated inside the pass from W = G x_1 A_1 and A_2 (no P in HBM)
      double* W = tmp_a_.as<double>();
      {
        Scope sc(prof_, "ttm_expand");
        const long long Je = (long long)(ranks_[1] * ranks_[2]);
        if (!ttm_expand(core_.as<double>(), 1, (int)ranks_[0], Je, factor(0), (int)shape_[0], W,
                        st_))
          ttm_generic(core_.as<double>(), 1, (int)ranks_[0], Je, factor(0), (int)ranks_[0], 1,
                      (int)shape_[0], W, st_);
      }
      Scope sc(prof_, "ttm_last_loss");
      ttm_last(x_, O, I, factor(N_ - 1), R, T_.as<double>(), nullptr, partial, st_, W, factor(1),
               (int)shape_[1], (int)ranks_[1]);
      nparts = ttm_last_blocks(O, I, R);
      t_valid_ = true;
    } else if (R <= 32) {
      std::vector<uint64_t> dims;
      const double* P = build_P(dims);
      Scope sc(prof_, "ttm_last_loss");
      // sketched factor updates (R_n <= 32) never read T: the pass computes the residual alone
      bool t_needed = opt_.factor_samples == 0 || N_ < 2;
      for (int n = 0; n < N_; ++n) t_needed |= ranks_[n] > 32;
      if (!t_needed && ttm_last_resid(x_, O, I, factor(N_ - 1), R, P, partial, st_)) {
        t_valid_ = false;
      } else {
        ttm_last(x_, O, I, factor(N_ - 1), R, T_.as<double>(), P, partial, st_);
        t_valid_ = true;
      }
      nparts = ttm_last_blocks(O, I, R);
    } else {
      std::vector<uint64_t> dims;
      const double* P = build_P(dims);
      // generic: full reconstruction then residual
      DevBuf xh(ltotal_ * 8, st_);
      ttm_generic(P, O, R, 1, factor(N_ - 1), R, 1, I, xh.as<double>(), st_);
      k_resid_partials<<<kNumSMs * 8, 256, 0, st_>>>(x_, xh.as<double>(), (long long)ltotal_,
                                                      partial);
      RTB_LAUNCH_CHECK();
      nparts = kNumSMs * 8;
      compute_T();
    }
    double* sc = scal_.as<double>();
    sum_partials(partial, nparts, sc, st_);
    allreduce(sc, 1);  // shard residuals
    join();
    k_finish_loss<<<1, 1, 0, st_>>>(sc, sc + 1, opt_.lambda, (double)total_, loss_dev, rmse_dev);
    RTB_LAUNCH_CHECK();
  }

  // sum of squares of the core and all factors (the ridge term) into *out
  void norms_into(double* out, cudaStream_t st = nullptr) {
    NormSet ns{};
    ns.count = N_ + 1;
    ns.p[0] = core_.as<double>();
    ns.n[0] = (long long)d_;
    for (int n = 0; n < N_; ++n) {
      ns.p[n + 1] = factor(n);
      ns.n[n + 1] = (long long)(shape_[n] * ranks_[n]);
    }
    k_norms<<<1, 1024, 0, st ? st : st_>>>(ns, out);
    RTB_LAUNCH_CHECK();
  }

  void reconstruct_full(double* out) {
    std::vector<uint64_t> dims;
    const double* P = build_P(dims);
    const long long O = (long long)(total_ / shape_[N_ - 1]);
    const int I = (int)shape_[N_ - 1], R = (int)ranks_[N_ - 1];
    ttm_generic(P, O, R, 1, factor(N_ - 1), R, 1, I, out, st_);
  }

};

Session::~Session() { delete e; }

static void validate(const std::vector<uint64_t>& shape, const std::vector<uint64_t>& ranks,
                     const AlsOptions& opt) {
  // ref tucker.cpp:194-199, 182-184; tensor.cpp:7-20
  if (opt.max_iterations == 0) throw Error(1, "als: max_iterations must be >= 1");
  if (ranks.size() != shape.size()) throw Error(1, "als: ranks order != tensor order");
  if (shape.empty() || shape.size() > 8) throw Error(1, "DenseTensor: order must be in [1, 8]");
  for (size_t n = 0; n < shape.size(); ++n)
    if (ranks[n] == 0 || ranks[n] > shape[n])
      throw Error(1, "random_model: rank outside [1, I_n]");
}

Session* session_create(const double* x_dev, const std::vector<uint64_t>& shape,
                        const std::vector<uint64_t>& ranks, const AlsOptions& opt) {
  validate(shape, ranks, opt);
  static const bool trace = std::getenv("RTB_HOST_TRACE") != nullptr;  // debugging aid
  const auto t0 = std::chrono::steady_clock::now();
  auto s = std::make_unique<Session>();
  s->e = new Engine(x_dev, shape, ranks, opt);
  const auto t1 = std::chrono::steady_clock::now();
  s->e->init_model();
  const auto t2 = std::chrono::steady_clock::now();
  s->e->initial_loss();
  if (trace) {
    RTB_CUDA(cudaStreamSynchronize(current_stream()));
    const auto t3 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    std::fprintf(stderr, "[rtb host] engine %.0f us, init %.0f us, initial loss (synced) %.0f us\n",
                 us(t0, t1), us(t1, t2), us(t2, t3));
  }
  return s.release();
}

uint32_t session_run(Session* s, uint32_t n, bool check_tol) {
  Engine& e = *s->e;
  if (check_tol && !e.have_prev_) {
    e.prev_loss_ = e.initial_loss_host();
    e.have_prev_ = true;
  }
  double prev = e.prev_loss_;
  uint32_t run = 0;
  struct Ev {
    cudaEvent_t a = nullptr, b = nullptr;
    ~Ev() {
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } ev;
  cudaEvent_t& a = ev.a;
  cudaEvent_t& b = ev.b;
  RTB_CUDA(cudaEventCreate(&a));
  RTB_CUDA(cudaEventCreate(&b));
  RTB_CUDA(cudaEventRecord(a, e.st_));
  for (uint32_t k = 0; k < n; ++k) {
    e.sweep(e.iterations_ + 1);
    // the core verdict of this sweep (waits only for its core step; the loss pass keeps
    // the GPU busy while the host enqueues the next sweep)
    e.resolve_core();
    ++run;
    if (check_tol) {
      const double loss = e.last_loss_host();
      const double change = std::abs(prev - loss) / std::max(std::abs(prev), 1e-300);
      prev = loss;
      e.prev_loss_ = loss;
      if (change < e.tolerance()) {
        e.converged_ = true;
        break;
      }
    }
  }
  RTB_CUDA(cudaEventRecord(b, e.st_));
  RTB_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  RTB_CUDA(cudaEventElapsedTime(&ms, a, b));
  e.sweep_seconds_ += ms * 1e-3;
  return run;
}

}  // namespace rtb

namespace rtb {

void session_output(Session* s, AlsOutput& out) { s->e->output(out); }

void als_run(const double* x_dev, const std::vector<uint64_t>& shape,
             const std::vector<uint64_t>& ranks, const AlsOptions& opt, AlsOutput& out) {
  static const bool trace = std::getenv("RTB_TRACE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  std::unique_ptr<Session> s(session_create(x_dev, shape, ranks, opt));
  if (trace) RTB_CUDA(cudaStreamSynchronize(current_stream()));
  const auto t1 = now();
  // tolerance <= 0 can never stop early (change < tol is false): no per-sweep sync
  session_run(s.get(), opt.max_iterations, opt.tolerance > 0.0);
  const auto t2 = now();
  session_output(s.get(), out);
  const auto t3 = now();
  s.reset();
  const auto t4 = now();
  if (trace)
    std::fprintf(stderr, "[als_run] create+init+loss %.2f ms, sweeps %.2f ms (device %.2f), "
                 "output %.2f ms, teardown %.2f ms\n", ms(t0, t1), ms(t1, t2),
                 out.sweep_seconds * 1e3, ms(t2, t3), ms(t3, t4));
}

// ---------------------------------------------------------------------------
// single-operation entry points

namespace {
struct HostModel {
  std::vector<uint64_t> shape, ranks;
};
AlsOptions op_opts(double lambda) {
  AlsOptions o;
  o.lambda = lambda;
  o.max_iterations = 1;
  return o;
}
}  // namespace

void model_update_core_sketched(const double* x_dev, const std::vector<uint64_t>& shape,
                                const std::vector<uint64_t>& ranks, const double* core,
                                const double* factors, double lambda, uint64_t s, uint64_t seed,
                                double* core_out, uint64_t* idx_out, double* w_out) {
  validate(shape, ranks, op_opts(lambda));
  AlsOptions o = op_opts(lambda);
  o.sketched = true;
  Engine e(x_dev, shape, ranks, o);
  e.set_model(core, factors);
  e.core_sketched_public(s, seed, idx_out, w_out);
  e.get_core(core_out);
}

void model_update_factor(const double* x_dev, const std::vector<uint64_t>& shape,
                         const std::vector<uint64_t>& ranks, const double* core,
                         const double* factors, double lambda, uint32_t mode, double* out) {
  validate(shape, ranks, op_opts(lambda));
  if (mode < 1 || mode > shape.size()) throw Error(1, "update_factor: mode out of range");
  Engine e(x_dev, shape, ranks, op_opts(lambda));
  e.set_model(core, factors);
  e.update_factor_public((int)mode - 1);
  e.get_factor((int)mode - 1, out);
}

void model_update_core_exact(const double* x_dev, const std::vector<uint64_t>& shape,
                             const std::vector<uint64_t>& ranks, const double* core,
                             const double* factors, double lambda, double* core_out) {
  validate(shape, ranks, op_opts(lambda));
  Engine e(x_dev, shape, ranks, op_opts(lambda));
  e.set_model(core, factors);
  e.core_exact_public();
  e.get_core(core_out);
}

void model_loss(const double* x_dev, const std::vector<uint64_t>& shape,
                const std::vector<uint64_t>& ranks, const double* core, const double* factors,
                double lambda, double* loss, double* rmse) {
  validate(shape, ranks, op_opts(lambda));
  Engine e(x_dev, shape, ranks, op_opts(lambda));
  e.set_model(core, factors);
  e.loss_public(loss, rmse);
}

namespace {
// stream constants of the device generator (documented in engine.h)
constexpr uint64_t kGenCore = 0x243f6a8885a308d3ULL, kGenFactor = 0x13198a2e03707344ULL,
                   kGenNoise = 0xa4093822299f31d0ULL, kGenPareto = 0x082efa98ec4e6c89ULL;

// N(0,1) from stream outputs 2k, 2k + 1 (Box-Muller, cosine branch). Streams: core
// seed ^ kGenCore; factor n sm_at(seed ^ kGenFactor, n) (hashed, so the modes' streams do not
// overlap); Pareto weights of mode n sm_at(seed ^ kGenPareto, n); noise seed ^ kGenNoise at
// the entry's global flat index.
__device__ __forceinline__ double gen_normal(uint64_t stream, uint64_t k) {
  double u1 = u64_to_unit(sm_at(stream, 2 * k));
  const double u2 = u64_to_unit(sm_at(stream, 2 * k + 1));
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

__global__ void k_gen_normal(double* out, long long n, uint64_t stream, long long offset) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = gen_normal(stream, (uint64_t)(offset + e));
}

// factor rows scaled by Pareto(alpha) weights (1 - u)^(-1/alpha), one draw per row
__global__ void k_gen_pareto_rows(double* a, int I, int R, uint64_t stream, double alpha) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I) return;
  const double u = u64_to_unit(sm_at(stream, (uint64_t)i));
  const double wgt = pow(1.0 - u, -1.0 / alpha);
  for (int r = 0; r < R; ++r) a[(size_t)i * R + r] *= wgt;
}

__global__ void k_gen_noise(double* x, long long n, uint64_t stream, long long offset,
                            const double* sigma) {
  const double sg = *sigma;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    x[e] += sg * gen_normal(stream, (uint64_t)(offset + e));
}

// sigma = level * sqrt(<G, Q> / total), Q = G x_n (A_n^T A_n) (so ||X||_F^2 = <G, Q>)
__global__ void k_gen_sigma(const double* G, const double* Q, long long d, double level,
                            double total, double* sigma) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < d; i += blockDim.x) s = fma(G[i], Q[i], s);
  s = block_sum<1024>(s, red);
  if (threadIdx.x == 0) *sigma = level * sqrt(fmax(s, 0.0) / total);
}
}  // namespace

void generate_planted_device(const std::vector<uint64_t>& shape,
                             const std::vector<uint64_t>& ranks, double noise_level,
                             double pareto_alpha, uint64_t seed, uint32_t shard_rank,
                             uint32_t shard_count, double* x_dev, double* core_host,
                             double* factors_host) {
  AlsOptions o = op_opts(0.0);
  validate(shape, ranks, o);
  if (shard_count == 0) shard_count = 1;
  if (shard_rank >= shard_count || shard_count > shape[0])
    throw Error(1, "generate: bad shard (rank >= count or more shards than rows)");
  if (noise_level < 0.0) throw Error(1, "generate: noise level must be non-negative");
  cudaStream_t st = current_stream();
  const int N = (int)shape.size();
  uint64_t d = 1, fe = 0;
  std::vector<uint64_t> foff(N);
  for (int n = 0; n < N; ++n) {
    d *= ranks[n];
    foff[n] = fe;
    fe += shape[n] * ranks[n];
  }
  DevBuf core(d * 8, st), fac(fe * 8, st), sig(8, st);
  const unsigned gb = (unsigned)std::min<uint64_t>(ceil_div<uint64_t>(std::max(d, fe), 256), 1024);
  k_gen_normal<<<gb, 256, 0, st>>>(core.as<double>(), (long long)d, seed ^ kGenCore, 0);
  RTB_LAUNCH_CHECK();
  for (int n = 0; n < N; ++n) {
    const uint64_t cnt = shape[n] * ranks[n];
    k_gen_normal<<<(unsigned)std::min<uint64_t>(ceil_div<uint64_t>(cnt, 256), 1024), 256, 0, st>>>(
        fac.as<double>() + foff[n], (long long)cnt, sm_at(seed ^ kGenFactor, (uint64_t)n), 0);
    RTB_LAUNCH_CHECK();
    if (pareto_alpha > 0.0) {
      k_gen_pareto_rows<<<ceil_div((int)shape[n], 256), 256, 0, st>>>(
          fac.as<double>() + foff[n], (int)shape[n], (int)ranks[n],
          sm_at(seed ^ kGenPareto, (uint64_t)n), pareto_alpha);
      RTB_LAUNCH_CHECK();
    }
  }
  // ||X_planted||^2 = <G, G x_n (A_n^T A_n)> from the full factors (same on every shard)
  {
    DevBuf grams((size_t)N * 64 * 64 * 8, st), q0(d * 8, st), q1(d * 8, st);
    const double* cur = core.as<double>();
    double* qb[2] = {q0.as<double>(), q1.as<double>()};
    std::vector<uint64_t> gd = ranks;
    for (int n = 0; n < N; ++n) {
      const int R = (int)ranks[n];
      FactorSet fs{};
      fs.order = 1;
      fs.ptr[0] = fac.as<double>() + foff[n];
      fs.rows[0] = (int)shape[n];
      fs.cols[0] = R;
      double* gn = grams.as<double>() + (size_t)n * 64 * 64;
      k_factor_gram<<<dim3(R * R, 1), 256, 0, st>>>(fs, gn, R);
      RTB_LAUNCH_CHECK();
      ttm_generic(cur, (long long)prod(gd, 0, n), R, (long long)prod(gd, n + 1), gn, R, 1, R,
                  qb[n & 1], st);
      cur = qb[n & 1];
    }
    k_gen_sigma<<<1, 1024, 0, st>>>(core.as<double>(), cur, (long long)d, noise_level,
                                    (double)prod(shape), sig.as<double>());
    RTB_LAUNCH_CHECK();
  }
  // this shard's rows of mode 1: reconstruct with the slab of A_1, then the noise at the
  // entries' global flat indices
  const uint64_t I1 = shape[0], P = shard_count, r = shard_rank;
  const uint64_t lo = r * I1 / P, hi = (r + 1) * I1 / P;
  std::vector<uint64_t> lshape = shape;
  lshape[0] = hi - lo;
  {
    std::vector<double> ch(d), fh(fe);
    RTB_CUDA(cudaMemcpyAsync(ch.data(), core.p, d * 8, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaMemcpyAsync(fh.data(), fac.p, fe * 8, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaStreamSynchronize(st));
    if (core_host) std::memcpy(core_host, ch.data(), d * 8);
    if (factors_host) std::memcpy(factors_host, fh.data(), fe * 8);
    // slab model: A_1 rows lo..hi
    std::vector<double> fs(fh.begin() + (long long)(lo * ranks[0]),
                           fh.begin() + (long long)(hi * ranks[0]));
    fs.insert(fs.end(), fh.begin() + (long long)(I1 * ranks[0]), fh.end());
    Engine e(x_dev, lshape, ranks, op_opts(0.0));
    e.set_model(ch.data(), fs.data());
    e.reconstruct(x_dev);
  }
  const long long ltot = (long long)prod(lshape);
  const long long inner = (long long)(prod(shape) / I1);
  k_gen_noise<<<(unsigned)std::min<long long>(ceil_div<long long>(ltot, 256), 8 * kNumSMs), 256, 0,
                st>>>(x_dev, ltot, seed ^ kGenNoise, (long long)lo * inner, sig.as<double>());
  RTB_LAUNCH_CHECK();
  RTB_CUDA(cudaStreamSynchronize(st));
}

void model_reconstruct(const std::vector<uint64_t>& shape, const std::vector<uint64_t>& ranks,
                       const double* core, const double* factors, double* out_host) {
  validate(shape, ranks, op_opts(0.0));
  cudaStream_t st = current_stream();
  const uint64_t total = prod(shape);
  DevBuf xd(total * 8, st);
  Engine e(xd.as<double>(), shape, ranks, op_opts(0.0));
  e.set_model(core, factors);
  e.reconstruct(xd.as<double>());
  RTB_CUDA(cudaMemcpyAsync(out_host, xd.p, total * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
}

// Per-factor scores through the same kernels as the ALS core step.
void factor_scores(const double* factor_host, int rows, int cols, double* scores, double* cdf,
                   double* sum, uint64_t* rank) {
  if (rows <= 0 || cols <= 0) throw Error(1, "compact_svd: empty matrix");
  cudaStream_t st = current_stream();
  DevBuf f((size_t)rows * cols * 8, st), sc((size_t)rows * 8, st), cd((size_t)rows * 8, st),
      sm(8, st), off(8, st), rw(4, st), rk(4, st), stat(4, st);
  RTB_CUDA(cudaMemcpyAsync(f.p, factor_host, (size_t)rows * cols * 8, cudaMemcpyHostToDevice, st));
  long long zero = 0;
  RTB_CUDA(cudaMemcpyAsync(off.p, &zero, 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(rw.p, &rows, 4, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemsetAsync(stat.p, 0, 4, st));
  FactorSet fs{};
  fs.order = 1;
  fs.ptr[0] = f.as<double>();
  fs.rows[0] = rows;
  fs.cols[0] = cols;
  if (cols <= 32 && rows >= cols) {
    // same route as the ALS core step: Cholesky of the Gram, one-sided Jacobi SVD behind it
    DevBuf g((size_t)cols * cols * 8, st), ns(4, st), lv((size_t)cols * cols * 8 + 8, st),
        okb(4, st), ws((size_t)rows * (cols + 1) * 8 + 64, st);
    RTB_CUDA(cudaMemcpyAsync(ns.p, &cols, 4, cudaMemcpyHostToDevice, st));
    k_factor_gram<<<dim3(cols * cols, 1), 256, 0, st>>>(fs, g.as<double>(), cols);
    RTB_LAUNCH_CHECK();
    spd_small(g.as<double>(), ns.as<int>(), cols * cols,
              (double)std::max(rows, cols) * DBL_EPSILON, lv.as<double>(), nullptr, okb.as<int>(), 1,
              st);
    k_hj_cta<<<1, 512, 0, st>>>(fs, ws.as<double>(), (long long)rows * (cols + (cols & 1)), 0.0,
                                sc.as<double>(), off.as<long long>(), rk.as<int>(), okb.as<int>(),
                                stat.as<int>());
    RTB_LAUNCH_CHECK();
    leverage_chol(fs, lv.as<double>(), cols * cols, okb.as<int>(), sc.as<double>(),
                  off.as<long long>(), rk.as<int>(), rows, 1, cols, st);
  } else {
    DevBuf ws(hj_work_bytes(rows, cols), st);
    int r = 0;
    hj_ridge_scores(f.as<double>(), rows, cols, 0.0, sc.as<double>(), &r, ws.p, st);
    RTB_CUDA(cudaMemcpyAsync(rk.p, &r, 4, cudaMemcpyHostToDevice, st));
  }
  k_score_cdf<<<1, 256, 0, st>>>(sc.as<double>(), off.as<long long>(), rw.as<int>(), 1,
                                 cd.as<double>(), sm.as<double>());
  RTB_LAUNCH_CHECK();
  int r = 0, es = 0;
  RTB_CUDA(cudaMemcpyAsync(scores, sc.p, (size_t)rows * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(cdf, cd.p, (size_t)rows * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(sum, sm.p, 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(&r, rk.p, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(&es, stat.p, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (es) throw Error(3, "compact_svd: Jacobi sweeps did not converge");
  *rank = (uint64_t)r;
}

void kron_draw(int order, const uint64_t* rows, uint64_t d, const double* scores,
               const double* cdfs, const double* sums, uint64_t seed, uint64_t s, uint64_t* idx,
               double* w) {
  if (order < 1 || order > 8) throw Error(1, "kron_draw: order must be in [1, 8]");
  if (d == 0 || s == 0) throw Error(1, "kron_draw: d and s must be positive");
  cudaStream_t st = current_stream();
  uint64_t sum_rows = 0, total = 1;
  DrawSpec ds{};
  ds.order = order;
  for (int n = 0; n < order; ++n) {
    ds.rows[n] = (long long)rows[n];
    ds.cdf_off[n] = (long long)sum_rows;
    sum_rows += rows[n];
    total *= rows[n];
  }
  ds.total_rows = total;
  ds.d = d;
  ds.seed = seed;
  ds.s = s;
  DevBuf sc(sum_rows * 8, st), cd(sum_rows * 8, st), sm(order * 8, st), ix(s * 8, st),
      ww(s * 8, st), work(draw_work_bytes(ds), st), flag(4, st);
  RTB_CUDA(cudaMemcpyAsync(sc.p, scores, sum_rows * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(cd.p, cdfs, sum_rows * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(sm.p, sums, order * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemsetAsync(flag.p, 0, 4, st));
  draw_sketch(ds, sc.as<double>(), cd.as<double>(), sm.as<double>(), DrawWork{work.p, work.bytes},
              (unsigned long long*)ix.p, ww.as<double>(), flag.as<int>(), st);
  int bad = 0;
  RTB_CUDA(cudaMemcpyAsync(idx, ix.p, s * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(w, ww.p, s * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(&bad, flag.p, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (bad) throw Error(1, "ImplicitKronecker: cannot sample, factor has no nonzero rows");
}

void tensor_fiber_major(const float* x, int I1, int I2, int I3, float* out) {
  cudaStream_t st = current_stream();
  c4_to_fiber_major(x, I1, I2, I3, out, st);
  RTB_CUDA(cudaStreamSynchronize(st));
}

void kron_fiber_sketch(const float* x, bool fiber_major, int I1, int I2, int I3, const double* a2,
                       const double* a3, int R2, int R3, double lambda, uint64_t s, uint64_t seed,
                       double* gram, double* rhs, uint64_t* idx_host, double* w_host,
                       uint64_t* data_draws, uint64_t* unique_rows, double* phase_ms,
                       int shard_rank, int shard_count) {
  if (I1 < 1 || I2 < 1 || I3 < 1 || R2 < 1 || R3 < 1 || R2 > 32 || R3 > 32 || R2 > I2 || R3 > I3)
    throw Error(1, "kron_fiber_sketch: bad shape or ranks (R <= 32, R <= I)");
  if (s == 0) throw Error(1, "solve_sketched_ridge: sample count must be positive");
  if (lambda < 0.0) throw Error(1, "solve_sketched_ridge: lambda must be non-negative");
  cudaStream_t st = current_stream();
  const int rmax = std::max(R2, R3), stride = rmax * rmax, maxI = std::max(I2, I3);
  const uint64_t W = (uint64_t)R2 * R3, total = (uint64_t)I2 * I3;
  cudaEvent_t ev[4];
  for (auto& e : ev) RTB_CUDA(cudaEventCreate(&e));
  RTB_CUDA(cudaEventRecord(ev[0], st));
  // ---- scores (classical, Cholesky route with the eigen fallback) and draws ----
  DevBuf grams(2 * stride * 8, st), linv(2 * stride * 8, st), ok(2 * 4, st), evals(2 * stride * 8, st),
      evecs(2 * stride * 8, st), est(2 * 4 + 64, st), scores((I2 + I3) * 8, st),
      cdf((I2 + I3) * 8, st), sums(2 * 8, st), meta(256, st), flag(4, st);
  FactorSet fs{};
  fs.order = 2;
  fs.ptr[0] = a2;
  fs.ptr[1] = a3;
  fs.rows[0] = I2;
  fs.rows[1] = I3;
  fs.cols[0] = R2;
  fs.cols[1] = R3;
  int hmeta[8] = {R2, R3, I2, I3, R2, R3, 0, 0};  // ns, rows, ranks
  long long hoff[2] = {0, I2};
  char* mp = static_cast<char*>(meta.p);
  int* ns_dev = reinterpret_cast<int*>(mp);
  int* rows_dev = ns_dev + 2;
  int* ranks_dev = ns_dev + 4;
  long long* off_dev = reinterpret_cast<long long*>(mp + 64);
  RTB_CUDA(cudaMemcpyAsync(mp, hmeta, sizeof(hmeta), cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(off_dev, hoff, sizeof(hoff), cudaMemcpyHostToDevice, st));
  k_factor_gram<<<dim3(rmax * rmax, 2), 256, 0, st>>>(fs, grams.as<double>(), rmax);
  RTB_LAUNCH_CHECK();
  spd_small(grams.as<double>(), ns_dev, stride, (double)maxI * DBL_EPSILON, linv.as<double>(), nullptr,
            ok.as<int>(), 2, st, rmax);
  sym_eigen(grams.as<double>(), ns_dev, rmax, stride, evals.as<double>(), evecs.as<double>(),
            est.as<int>(), 2, st, ok.as<int>());
  const dim3 lg(ceil_div(maxI, 128), 2);
  k_leverage_rows<<<lg, 128, 0, st>>>(fs, evals.as<double>(), evecs.as<double>(), stride, 0.0,
                                      scores.as<double>(), off_dev, ranks_dev, ok.as<int>());
  RTB_LAUNCH_CHECK();
  leverage_chol(fs, linv.as<double>(), stride, ok.as<int>(), scores.as<double>(), off_dev,
                ranks_dev, maxI, 2, rmax, st);
  k_score_cdf<<<2, 256, 0, st>>>(scores.as<double>(), off_dev, rows_dev, 2, cdf.as<double>(),
                                 sums.as<double>());
  RTB_LAUNCH_CHECK();
  DrawSpec ds{};
  ds.order = 2;
  ds.rows[0] = I2;
  ds.rows[1] = I3;
  ds.cdf_off[0] = 0;
  ds.cdf_off[1] = I2;
  ds.total_rows = total;
  ds.d = W;
  ds.seed = seed;
  ds.s = s;
  DevBuf ix(s * 8, st), ww(s * 8, st), dwork(draw_work_bytes(ds), st);
  RTB_CUDA(cudaMemsetAsync(flag.p, 0, 4, st));
  draw_sketch(ds, scores.as<double>(), cdf.as<double>(), sums.as<double>(),
              DrawWork{dwork.p, dwork.bytes}, (unsigned long long*)ix.p, ww.as<double>(),
              flag.as<int>(), st);
  RTB_CUDA(cudaEventRecord(ev[1], st));
  // ---- one sort/merge of the draws, then the Gram and the fiber RHS (k_c4.cu) ----
  DevBuf cnt(16, st);
  const bool want_rhs = x && rhs;
  if (gram || want_rhs) {
    DevBuf cw(c4_work_bytes(s, I1, I2, I3, R2, R3, gram != nullptr), st);
    c4_sketch(want_rhs ? x : nullptr, fiber_major, I1, I2, I3, a2, R2, a3, R3,
              (const unsigned long long*)ix.p, ww.as<double>(), s, lambda, cw.p, cw.bytes, gram,
              want_rhs ? rhs : nullptr, cnt.as<unsigned long long>(),
              cnt.as<unsigned long long>() + 1, ev[2], st, shard_rank, shard_count);
  } else {
    RTB_CUDA(cudaMemsetAsync(cnt.p, 0, 16, st));
    RTB_CUDA(cudaEventRecord(ev[2], st));
  }
  RTB_CUDA(cudaEventRecord(ev[3], st));
  int bad = 0;
  RTB_CUDA(cudaMemcpyAsync(&bad, flag.p, 4, cudaMemcpyDeviceToHost, st));
  if (idx_host) RTB_CUDA(cudaMemcpyAsync(idx_host, ix.p, s * 8, cudaMemcpyDeviceToHost, st));
  if (w_host) RTB_CUDA(cudaMemcpyAsync(w_host, ww.p, s * 8, cudaMemcpyDeviceToHost, st));
  uint64_t nd[2] = {0, 0};
  RTB_CUDA(cudaMemcpyAsync(nd, cnt.p, 16, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (bad) throw Error(1, "ImplicitKronecker: cannot sample, factor has no nonzero rows");
  if (data_draws) *data_draws = nd[0];
  if (unique_rows) *unique_rows = nd[1];
  if (phase_ms)
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      RTB_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
      phase_ms[k] = ms;
    }
  for (auto& e : ev) cudaEventDestroy(e);
}

void kron_normal_eq(int order, const uint64_t* rows, const uint64_t* ranks, const double* factors,
                    const double* x_host, double lambda, uint64_t s, const uint64_t* idx,
                    const double* w, double* gram, double* rhs) {
  if (order < 1 || order > 8) throw Error(1, "kron_normal_eq: order must be in [1, 8]");
  if (s == 0) throw Error(1, "solve_sketched_ridge: sample count must be positive");
  for (int n = 0; n < order; ++n)
    if (ranks[n] == 0 || ranks[n] > rows[n] || rows[n] > (uint64_t)INT32_MAX)
      throw Error(1, "kron_normal_eq: rank outside [1, I_n]");
  cudaStream_t st = current_stream();
  std::vector<uint64_t> shape(rows, rows + order), rk(ranks, ranks + order);
  const uint64_t total = prod(shape), d = prod(rk);
  if (d > (uint64_t)INT32_MAX / 2) throw Error(1, "kron_normal_eq: d too large");
  for (uint64_t t = 0; t < s; ++t)
    if (idx[t] >= total + d) throw Error(1, "kron_normal_eq: row index out of range");
  uint64_t fe = 0;
  for (int n = 0; n < order; ++n) fe += shape[n] * rk[n];
  DevBuf xd(total * 8, st), fd(fe * 8, st), ix(s * 8, st), ww(s * 8, st), G(d * d * 8, st),
      r(d * 8, st), dd(8, st);
  RTB_CUDA(cudaMemcpyAsync(xd.p, x_host, total * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(fd.p, factors, fe * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(ix.p, idx, s * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(ww.p, w, s * 8, cudaMemcpyHostToDevice, st));
  GramSpec gs{};
  gs.order = order;
  uint64_t off = 0;
  for (int n = 0; n < order; ++n) {
    gs.rows[n] = (int)shape[n];
    gs.ranks[n] = (int)rk[n];
    gs.factors[n] = fd.as<double>() + off;
    off += shape[n] * rk[n];
  }
  gs.total_rows = total;
  gs.d = (int)d;
  gs.dprime = (int)(d / rk[0]);
  gs.lambda = lambda;
  gs.s = s;
  DevBuf work(gram_work_bytes(gs), st);
  sketch_normal_eq(gs, xd.as<double>(), (const unsigned long long*)ix.p, ww.as<double>(), work.p,
                   work.bytes, G.as<double>(), r.as<double>(), (unsigned long long*)dd.p, st);
  RTB_CUDA(cudaMemcpyAsync(gram, G.p, d * d * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(rhs, r.p, d * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
}

// x = gram^+ rhs: Cholesky, else (d <= 64) eigen pinv with the reference cutoff.
void solve_sym_device(double* G, double* rhs, int d, double* x_dev, int* rank, int* path,
                      cudaStream_t st) {
  DevBuf work(chol_work_bytes(d), st), stat(4, st), copy((size_t)d * d * 8, st);
  RTB_CUDA(cudaMemcpyAsync(copy.p, G, (size_t)d * d * 8, cudaMemcpyDeviceToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(x_dev, rhs, (size_t)d * 8, cudaMemcpyDeviceToDevice, st));
  chol_solve(copy.as<double>(), d, x_dev, stat.as<int>(), work.p, st);
  int status = 0;
  RTB_CUDA(cudaMemcpyAsync(&status, stat.p, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (status == 0) {
    *rank = d;
    *path = 0;
    return;
  }
  if (d > 64) {  // block-Jacobi eigen pinv (k_eig.cu) of G
    RTB_CUDA(cudaMemcpyAsync(copy.p, G, (size_t)d * d * 8, cudaMemcpyDeviceToDevice, st));
    DevBuf pw(pinv_large_work_bytes(d), st), rk(4, st);
    pinv_solve_large(copy.as<double>(), d, rhs, x_dev, rk.as<int>(), pw.p, pw.bytes, st);
    RTB_CUDA(cudaMemcpyAsync(rank, rk.p, 4, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaStreamSynchronize(st));
    *path = 1;
    return;
  }
  DevBuf ev((size_t)d * d * 8 + 8, st), evec((size_t)d * d * 8, st), es(4, st), ns(4, st),
      pv((size_t)d * d * 8, st), rk(4, st);
  RTB_CUDA(cudaMemcpyAsync(ns.p, &d, 4, cudaMemcpyHostToDevice, st));
  sym_eigen(G, ns.as<int>(), d, d * d, ev.as<double>(), evec.as<double>(), es.as<int>(), 1, st);
  k_sym_pinv<<<1, 256, 0, st>>>(ev.as<double>(), evec.as<double>(), ns.as<int>(), d * d,
                                pv.as<double>(), rk.as<int>(), nullptr);
  RTB_LAUNCH_CHECK();
  k_rows_times_small<<<ceil_div(d, 256), 256, 0, st>>>(rhs, pv.as<double>(), 1, d, x_dev);
  RTB_LAUNCH_CHECK();
  int e = 0;
  RTB_CUDA(cudaMemcpyAsync(rank, rk.p, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(&e, es.p, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (e) throw Error(3, "symmetric_eigen: Jacobi sweeps did not converge");
  *path = 1;
}

void sym_eig(const double* a, uint64_t d, double* evals, double* evecs) {
  if (d == 0) throw Error(1, "compact_svd: empty matrix");
  if (d > 46340) throw Error(1, "sym_eig: d too large");
  cudaStream_t st = current_stream();
  const int n = (int)d;
  DevBuf A(d * d * 8, st), ev(d * 8 + 8, st), V(d * d * 8, st);
  RTB_CUDA(cudaMemcpyAsync(A.p, a, d * d * 8, cudaMemcpyHostToDevice, st));
  if (n <= 64) {
    DevBuf es(4, st), ns(4, st);
    RTB_CUDA(cudaMemcpyAsync(ns.p, &n, 4, cudaMemcpyHostToDevice, st));
    sym_eigen(A.as<double>(), ns.as<int>(), n, n * n, ev.as<double>(), V.as<double>(),
              es.as<int>(), 1, st);
    int e = 0;
    RTB_CUDA(cudaMemcpyAsync(&e, es.p, 4, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaMemcpyAsync(evals, ev.p, d * 8, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaMemcpyAsync(evecs, V.p, d * d * 8, cudaMemcpyDeviceToHost, st));
    RTB_CUDA(cudaStreamSynchronize(st));
    if (e) throw Error(3, "symmetric_eigen: Jacobi sweeps did not converge");
    return;  // already sorted non-increasing
  }
  DevBuf work(eig_large_work_bytes(n), st);
  sym_eig_large(A.as<double>(), n, ev.as<double>(), V.as<double>(), work.p, st);
  std::vector<double> mu(d), vv(d * d);
  RTB_CUDA(cudaMemcpyAsync(mu.data(), ev.p, d * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaMemcpyAsync(vv.data(), V.p, d * d * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  std::vector<int> ord(d);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return mu[x] > mu[y]; });
  for (int k = 0; k < n; ++k) {
    evals[k] = mu[ord[k]];
    for (int i = 0; i < n; ++i) evecs[(size_t)i * d + k] = vv[(size_t)i * d + ord[k]];
  }
}

void spd_solve(const double* gram, const double* rhs, uint64_t d, double* x, uint64_t* rank,
               int* path) {
  if (d == 0) throw Error(1, "compact_svd: empty matrix");
  cudaStream_t st = current_stream();
  DevBuf G(d * d * 8, st), r(d * 8, st), xd(d * 8, st);
  RTB_CUDA(cudaMemcpyAsync(G.p, gram, d * d * 8, cudaMemcpyHostToDevice, st));
  RTB_CUDA(cudaMemcpyAsync(r.p, rhs, d * 8, cudaMemcpyHostToDevice, st));
  int rk = 0, pth = 0;
  solve_sym_device(G.as<double>(), r.as<double>(), (int)d, xd.as<double>(), &rk, &pth, st);
  RTB_CUDA(cudaMemcpyAsync(x, xd.p, d * 8, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (rank) *rank = (uint64_t)rk;
  if (path) *path = pth;
}

}  // namespace rtb
