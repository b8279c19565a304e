// k_pinv.cu -- pseudo-inverse solve x = G^+ b of a symmetric d x d Gram for d > 64, the
// fallback when the sketched Gram is not numerically positive definite (Cholesky and PCG
// fail), e.g. heavy-tailed (Pareto-scaled) factors where cond(G) reaches 1/eps.
//
// Reference semantics (ref linalg.cpp:8-26 + svd.cpp:87-97): pinv(G) = sum over the singular
// triplets with sigma_k > max(m, n) eps sigma_max (and sigma_k > 0) of v_k u_k^T / sigma_k.
// For symmetric G the singular values are |mu_k| of its eigenpairs (mu_k, v_k) and
// u_k = sign(mu_k) v_k, so x = sum_{|mu_k| > d eps max|mu|} (v_k^T b / mu_k) v_k.
//
// The eigendecomposition is the dense symmetric divide-and-conquer solver of cuSOLVER
// (Dsyevd), loaded with dlopen on first use so the library has no link-time dependency on it;
// it is the rare-path replacement of the reference's one-sided Jacobi SVD of the Gram
// (svd.cpp:21-67), not part of the per-sweep hot path. The two projections run here.
#include <dlfcn.h>

#include <cfloat>
#include <mutex>

#include <cusolverDn.h>

#include "common.cuh"
#include "kernels.h"

namespace rtb {

namespace {

struct Cusolver {
  void* lib = nullptr;
  decltype(&cusolverDnCreate) create = nullptr;
  decltype(&cusolverDnSetStream) set_stream = nullptr;
  decltype(&cusolverDnDsyevd_bufferSize) syevd_bs = nullptr;
  decltype(&cusolverDnDsyevd) syevd = nullptr;
  cusolverDnHandle_t h = nullptr;
  std::string err;
};

Cusolver& cusolver() {
  static Cusolver c;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libcusolver.so.11", "/usr/local/cuda/lib64/libcusolver.so.11",
                           "libcusolver.so"};
    for (const char* n : names)
      if ((c.lib = dlopen(n, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (!c.lib) {
      c.err = "cannot load libcusolver (dense pinv fallback for d > 64)";
      return;
    }
    c.create = reinterpret_cast<decltype(c.create)>(dlsym(c.lib, "cusolverDnCreate"));
    c.set_stream = reinterpret_cast<decltype(c.set_stream)>(dlsym(c.lib, "cusolverDnSetStream"));
    c.syevd_bs = reinterpret_cast<decltype(c.syevd_bs)>(dlsym(c.lib, "cusolverDnDsyevd_bufferSize"));
    c.syevd = reinterpret_cast<decltype(c.syevd)>(dlsym(c.lib, "cusolverDnDsyevd"));
    if (!c.create || !c.set_stream || !c.syevd_bs || !c.syevd) {
      c.err = "libcusolver lacks the Dsyevd entry points";
      return;
    }
    if (c.create(&c.h) != CUSOLVER_STATUS_SUCCESS) c.err = "cusolverDnCreate failed";
  });
  return c;
}

// y[k] = (v_k . b) / mu_k where |mu_k| > cutoff, else 0; one warp per eigenvector (row k of
// the column-major eigenvector matrix read as row-major). rank_out = number kept.
__global__ void k_pinv_project(const double* __restrict__ V, const double* __restrict__ mu, int d,
                               const double* __restrict__ b, double* __restrict__ y,
                               int* __restrict__ rank_out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= d) return;
  const double mmax = fmax(fabs(mu[0]), fabs(mu[d - 1]));  // ascending eigenvalues
  const double cutoff = (double)d * DBL_EPSILON * mmax;
  const double m = mu[warp];
  const bool keep = fabs(m) > cutoff && m != 0.0;
  double acc = 0.0;
  if (keep)
    for (int j = lane; j < d; j += 32) acc += V[(size_t)warp * d + j] * b[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    y[warp] = keep ? acc / m : 0.0;
    if (keep) atomicAdd(rank_out, 1);
  }
}

// x[j] = sum_k y[k] V[k][j] (coalesced over j; fixed k order)
__global__ void k_pinv_expand(const double* __restrict__ V, int d, const double* __restrict__ y,
                              double* __restrict__ x) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    const double yk = y[k];
    if (yk != 0.0) acc += yk * V[(size_t)k * d + j];
  }
  x[j] = acc;
}

}  // namespace

size_t pinv_large_work_bytes(int d) {
  Cusolver& c = cusolver();
  if (!c.err.empty()) throw Error(3, c.err);
  int lwork = 0;
  if (c.syevd_bs(c.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, d, nullptr, d, nullptr,
                 &lwork) != CUSOLVER_STATUS_SUCCESS)
    throw Error(3, "cusolverDnDsyevd_bufferSize failed");
  return ((size_t)lwork + 2 * (size_t)d) * 8 + 256;
}

void pinv_solve_large(double* G, int d, const double* b, double* x, int* rank_dev, void* work,
                      size_t work_bytes, cudaStream_t st) {
  Cusolver& c = cusolver();
  if (!c.err.empty()) throw Error(3, c.err);
  int lwork = 0;
  if (c.syevd_bs(c.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, d, G, d, nullptr,
                 &lwork) != CUSOLVER_STATUS_SUCCESS)
    throw Error(3, "cusolverDnDsyevd_bufferSize failed");
  if (work_bytes < ((size_t)lwork + 2 * (size_t)d) * 8 + 256)
    throw Error(4, "pinv_solve_large: workspace");
  double* mu = static_cast<double*>(work);
  double* y = mu + d;
  double* wk = y + d;
  int* info = reinterpret_cast<int*>(wk + lwork);
  if (c.set_stream(c.h, st) != CUSOLVER_STATUS_SUCCESS) throw Error(3, "cusolverDnSetStream failed");
  // G is symmetric, so its row-major storage is its column-major storage
  if (c.syevd(c.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, d, G, d, mu, wk, lwork, info) !=
      CUSOLVER_STATUS_SUCCESS)
    throw Error(3, "cusolverDnDsyevd failed");
  int hinfo = 0;
  RTB_CUDA(cudaMemcpyAsync(&hinfo, info, 4, cudaMemcpyDeviceToHost, st));
  RTB_CUDA(cudaStreamSynchronize(st));
  if (hinfo != 0) throw Error(3, "Jacobi SVD did not converge (dense eigensolver info != 0)");
  RTB_CUDA(cudaMemsetAsync(rank_dev, 0, 4, st));
  k_pinv_project<<<ceil_div(d * 32, 256), 256, 0, st>>>(G, mu, d, b, y, rank_dev);
  RTB_LAUNCH_CHECK();
  k_pinv_expand<<<ceil_div(d, 256), 256, 0, st>>>(G, d, y, x);
  RTB_LAUNCH_CHECK();
}

}  // namespace rtb
