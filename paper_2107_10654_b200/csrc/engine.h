// engine.h -- device-resident sketched Tucker-ALS engine (host C++ side).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

namespace rtb {

// Stream used by the calling thread (default: a library-owned stream per device).
cudaStream_t current_stream();
void set_stream(cudaStream_t s);

// Stream-ordered device buffer (cudaMallocAsync from the device pool).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(size_t b, cudaStream_t s);
  ~DevBuf();
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept;
  void ensure(size_t b, cudaStream_t s);
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct AlsOptions {
  double lambda = 0.001;
  bool sketched = false;
  double epsilon = 0.1;
  double delta = 0.1;
  uint64_t seed = 0;
  uint32_t max_iterations = 50;
  double tolerance = 1e-6;
  uint64_t sample_override = 0;
  bool record_history = false;
  const double* init_core = nullptr;      // host
  const double* init_factors = nullptr;   // host
  bool profile = false;                   // per-kernel-family events
  uint32_t shard_rank = 0, shard_count = 1;
  void (*allreduce)(double*, uint64_t, void*, void*) = nullptr;
  void* allreduce_user = nullptr;
  int core_solver = 0;                    // 0 auto (PCG, Cholesky fallback), 1 Cholesky
  bool fast_loss = false;                 // loss by the expansion formula (see engine.cu)
  uint64_t factor_samples = 0;            // > 0: sketched factor updates (perf mode)
  bool no_graph = false;                  // never run a sweep as a CUDA graph
};

struct HistoryRow {
  uint32_t iteration;
  std::string step;
  double loss, rmse;
};
struct StepTiming {
  std::string step;
  double total = 0.0;
  uint64_t count = 0;
};
struct KernelTiming {
  std::string name;
  double total = 0.0;
  uint64_t launches = 0;
};

struct AlsOutput {
  std::vector<uint64_t> shape, ranks;
  std::vector<double> core;
  std::vector<double> factors;  // concatenated I_n x R_n
  double lambda = 0.0;
  std::vector<HistoryRow> history;
  std::vector<StepTiming> timings;
  std::vector<KernelTiming> kernels;
  uint32_t iterations = 0;
  double final_loss = 0.0, final_rmse = 0.0;
  bool converged = false;
  uint64_t last_sample_count = 0, last_data_draws = 0;
  int last_rank_deficient = 0, last_solver_path = 0, last_pcg_iterations = 0;
  double sweep_seconds = 0.0;  // device time of the sweep loop
  uint64_t graph_launches = 0;  // sweeps that ran as one CUDA graph launch
};

class Engine;  // opaque

// Session: init + initial loss at create; sweeps on demand.
struct Session {
  Engine* e = nullptr;
  ~Session();
};
Session* session_create(const double* x_dev, const std::vector<uint64_t>& shape,
                        const std::vector<uint64_t>& ranks, const AlsOptions& opt);
// Runs up to n sweeps; honours tolerance when check_tol. Returns sweeps run.
uint32_t session_run(Session* s, uint32_t n, bool check_tol);
void session_output(Session* s, AlsOutput& out);

// Whole run with the reference's semantics (ref tucker.cpp:192-276).
void als_run(const double* x_dev, const std::vector<uint64_t>& shape,
             const std::vector<uint64_t>& ranks, const AlsOptions& opt, AlsOutput& out);

// ---- single-operation entry points (parity ladder) ----
void factor_scores(const double* factor_host, int rows, int cols, double* scores, double* cdf,
                   double* sum, uint64_t* rank);
void kron_draw(int order, const uint64_t* rows, uint64_t d, const double* scores,
               const double* cdfs, const double* sums, uint64_t seed, uint64_t s, uint64_t* idx,
               double* w);
// BASELINE C4 microbench on device buffers: scores of A2, A3, s draws from their augmented
// product distribution (d = R2 R3), the W x W Gram (W = R2 R3) and, when x != nullptr,
// the W x I1 fiber RHS (x canonical row-major, or fiber-major: mode 1 fastest).
// phase_ms[3] = scores+draws, Gram (incl. the shared sort/merge of the draws), RHS.
void kron_fiber_sketch(const float* x, bool fiber_major, int I1, int I2, int I3, const double* a2,
                       const double* a3, int R2, int R3, double lambda, uint64_t s, uint64_t seed,
                       double* gram, double* rhs, uint64_t* idx_host, double* w_host,
                       uint64_t* data_draws, uint64_t* unique_rows, double* phase_ms,
                       int shard_rank = 0, int shard_count = 1);
void tensor_fiber_major(const float* x, int I1, int I2, int I3, float* out);
void kron_normal_eq(int order, const uint64_t* rows, const uint64_t* ranks, const double* factors,
                    const double* x_host, double lambda, uint64_t s, const uint64_t* idx,
                    const double* w, double* gram, double* rhs);
void spd_solve(const double* gram, const double* rhs, uint64_t d, double* x, uint64_t* rank,
               int* path);
// Symmetric eigendecomposition of a host d x d matrix on the GPU (d <= 64: CTA Jacobi,
// larger: parallel block Jacobi, k_eig.cu): evals descending, evecs row-major (column k).
void sym_eig(const double* a, uint64_t d, double* evals, double* evecs);
// Model-level ops on a device tensor with a host model.
void model_update_core_sketched(const double* x_dev, const std::vector<uint64_t>& shape,
                                const std::vector<uint64_t>& ranks, const double* core,
                                const double* factors, double lambda, uint64_t s, uint64_t seed,
                                double* core_out, uint64_t* idx_out, double* w_out);
void model_update_factor(const double* x_dev, const std::vector<uint64_t>& shape,
                         const std::vector<uint64_t>& ranks, const double* core,
                         const double* factors, double lambda, uint32_t mode, double* out);
void model_update_core_exact(const double* x_dev, const std::vector<uint64_t>& shape,
                             const std::vector<uint64_t>& ranks, const double* core,
                             const double* factors, double lambda, double* core_out);
void model_loss(const double* x_dev, const std::vector<uint64_t>& shape,
                const std::vector<uint64_t>& ranks, const double* core, const double* factors,
                double lambda, double* loss, double* rmse);
void model_reconstruct(const std::vector<uint64_t>& shape, const std::vector<uint64_t>& ranks,
                       const double* core, const double* factors, double* out_host);
// Dense toolkit (ref capi.cpp:299-362).
void dense_ridge_scores(const double* a, uint64_t n, uint64_t d, double lambda, double* out);
void dense_solve_ridge(const double* a, uint64_t n, uint64_t d, const double* b, double lambda,
                       double* x);
// AugmentedSampler draws (ref sampler.cpp:9-57) of s rows from candidate scores (host)
void aug_draw(const double* cand, uint64_t n, uint64_t d, double d_eff_lower, uint64_t seed,
              uint64_t s, uint64_t* idx_out, double* w_out);
// sketched normal equations of [A; sqrt(lambda) I] from a given RowSketch (host buffers)
void dense_normal_eq(const double* a, uint64_t n, uint64_t d, const double* b, double lambda,
                     uint64_t s, const uint64_t* idx, const double* w, double* gram, double* rhs);
void dense_sketched_ridge(const double* a, uint64_t n, uint64_t d, const double* b,
                          const double* cand, double lambda, double d_eff_lower, double eps,
                          double delta, uint64_t s_override, uint64_t seed, double* x,
                          uint64_t* s_out, double* beta_out);

// Planted synthetic tensor generated on the device (BASELINE configs; counter-based
// SplitMix64 streams, so any shard of rows can be generated independently and a sharded
// generation equals the unsharded one): core and factors i.i.d. N(0,1) (Box-Muller on the
// stream pairs), factor rows optionally scaled by Pareto(alpha) weights (alpha > 0), X = the
// reconstruction plus i.i.d. N(0, sigma^2) noise on every entry, sigma = noise_level
// ||X_planted||_F / sqrt(prod I_n) (the norm from the model: <G, G x_n A_n^T A_n>).
// Writes this shard's rows [r I1 / P, (r + 1) I1 / P) of mode 1 into x_dev; core_host /
// factors_host (optional) receive the planted model.
void generate_planted_device(const std::vector<uint64_t>& shape,
                             const std::vector<uint64_t>& ranks, double noise_level,
                             double pareto_alpha, uint64_t seed, uint32_t shard_rank,
                             uint32_t shard_count, double* x_dev, double* core_host,
                             double* factors_host);

// Property suites of rtucker_verify_suite (verify.cu): name = leverage | kronecker |
// missing | structural | all; JSON report; true when every check passed.
bool verify_suites(const std::string& name, uint64_t seed, std::string& json);

// True when at least one CUDA device is visible (cached).
bool cuda_device_present();
// H2D copy of n doubles on st, then a device-side finiteness scan; synchronises st and
// throws Error(1, "<what>: non-finite entry") like ref tensor.cpp:32-42.
void upload_checked(double* dst, const double* src, uint64_t n, cudaStream_t st, const char* what);
uint64_t sample_count_formula(double beta_prime, uint64_t d, double eps, double delta);

}  // namespace rtb
