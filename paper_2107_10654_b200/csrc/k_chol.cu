// k_chol.cu -- on-device Cholesky solve of the sketched normal equations.
//
// The reference solves G x = rhs with a one-sided Jacobi SVD pseudoinverse
// (ref sketch_ridge.cpp:130-139, svd.cpp:21-111): O(sweeps d^3), 186.7 s at
// d = 1024 on one core. G is symmetric positive definite whenever every
// augmented row was drawn at least once (lambda > 0), so we factor G = L L^T:
//
//   for each 64-wide panel k (right looking):
//     k_potrf_diag    one CTA factors the 64x64 diagonal block in smem
//     k_trsm_panel    L_ik = A_ik L_kk^-T for the rows below
//     k_syrk_update   A_ij -= L_ik L_jk^T over the trailing lower tiles,
//                     FP64 tensor cores (DMMA.8x8x4)
//   k_trsv_coop       forward + backward substitution in one cooperative
//                     kernel (grid-wide barrier per 64-row block)
//
// A non-positive pivot stops the factorization and is reported in *status
// (k + 1 for pivot k); the caller then falls back to the eigen/pinv path.
#include "common.cuh"
#include "kernels.h"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace rtb {

namespace {
constexpr int NB = 64;
constexpr int LDB = NB + 4;
}  // namespace

size_t chol_work_bytes(int d) {
  const size_t nbt = (size_t)ceil_div(d, NB);
  return nbt * NB * NB * 8 + (((size_t)d * 8 + 255) & ~size_t(255)) * 2;
}

__global__ void __launch_bounds__(256) k_potrf_diag(double* a, int d, int k, int* status) {
  if (*status) return;
  __shared__ double s[NB][NB + 1];
  const int k0 = k * NB;
  const int nb = min(NB, d - k0);
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int i = e / NB, j = e % NB;
    s[i][j] = (i < nb && j <= i) ? a[(size_t)(k0 + i) * d + k0 + j] : 0.0;
  }
  __syncthreads();
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int j = 0; j < nb; ++j) {
    if (threadIdx.x == 0) {
      const double piv = s[j][j];
      if (!(piv > 0.0)) bad = k0 + j + 1;
      s[j][j] = sqrt(piv);
    }
    __syncthreads();
    if (bad) break;
    const double ljj = s[j][j];
    for (int i = j + 1 + threadIdx.x; i < nb; i += blockDim.x) s[i][j] /= ljj;
    __syncthreads();
    // trailing update of the lower part of columns j+1..nb-1
    const int m = nb - j - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e / m, l = j + 1 + e % m;
      if (l <= i) s[i][l] -= s[i][j] * s[l][j];
    }
    __syncthreads();
  }
  if (bad) {
    if (threadIdx.x == 0) atomicCAS(status, 0, bad);
    return;
  }
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    if (j <= i) a[(size_t)(k0 + i) * d + k0 + j] = s[i][j];
  }
}

// Rows below panel k: solve x L_kk^T = a for each row (64 rows per CTA,
// one thread per row, column-oriented updates in smem).
__global__ void __launch_bounds__(64) k_trsm_panel(double* a, int d, int k, const int* status) {
  if (*status) return;
  extern __shared__ double dyn[];
  double(*L)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dyn);
  double(*X)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dyn + NB * (NB + 1));
  const int k0 = k * NB;
  const int nb = min(NB, d - k0);
  const int r0 = k0 + NB + blockIdx.x * NB;
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 64) {
    const int i = e / NB, j = e % NB;
    L[i][j] = (i < nb && j < nb && j <= i) ? a[(size_t)(k0 + i) * d + k0 + j] : 0.0;
    const int row = r0 + i;
    X[i][j] = (row < d && j < nb) ? a[(size_t)row * d + k0 + j] : 0.0;
  }
  __syncthreads();
  const int row = r0 + tid;
  if (row < d) {
    for (int j = 0; j < nb; ++j) {
      const double xj = X[tid][j] / L[j][j];
      X[tid][j] = xj;
      for (int l = j + 1; l < nb; ++l) X[tid][l] -= xj * L[l][j];
    }
  }
  __syncthreads();
  for (int e = tid; e < NB * NB; e += 64) {
    const int i = e / NB, j = e % NB;
    const int rr = r0 + i;
    if (rr < d && j < nb) a[(size_t)rr * d + k0 + j] = X[i][j];
  }
}

// Trailing update of lower tiles (bi >= bj > k): A_ij -= L_ik L_jk^T.
__global__ void __launch_bounds__(256) k_syrk_update(double* a, int d, int k, const int* status) {
  if (*status) return;
  extern __shared__ __align__(16) double dsm[];
  double(*li)[LDB] = reinterpret_cast<double(*)[LDB]>(dsm);
  double(*lj)[LDB] = reinterpret_cast<double(*)[LDB]>(dsm + NB * LDB);
  const int nbt = ceil_div(d, NB);
  const int first = k + 1;
  // linear block -> (bi, bj) with first <= bj <= bi < nbt
  int rem = blockIdx.x, bj = first;
  while (rem >= nbt - bj) {
    rem -= nbt - bj;
    ++bj;
  }
  const int bi = bj + rem;
  const int k0 = k * NB, i0 = bi * NB, j0 = bj * NB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int mbase = 16 * (warp >> 1), nbase = 32 * (warp & 1);
  const bool vec = (d % 2) == 0;
  for (int e = tid; e < NB * (NB / 2); e += 256) {
    const int r = e / (NB / 2), c = (e % (NB / 2)) * 2;
    const bool oki = (i0 + r < d) && (k0 + c < d);
    const bool okj = (j0 + r < d) && (k0 + c < d);
    if (vec) {
      cp_async16(&li[r][c], oki ? a + (size_t)(i0 + r) * d + k0 + c : a, oki);
      cp_async16(&lj[r][c], okj ? a + (size_t)(j0 + r) * d + k0 + c : a, okj);
    } else {
      for (int q = 0; q < 2; ++q) {
        li[r][c + q] = (i0 + r < d && k0 + c + q < d) ? a[(size_t)(i0 + r) * d + k0 + c + q] : 0.0;
        lj[r][c + q] = (j0 + r < d && k0 + c + q < d) ? a[(size_t)(j0 + r) * d + k0 + c + q] : 0.0;
      }
    }
  }
  cp_async_commit();
  // accumulators start from the current A tile
  double acc[2][4][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int r = i0 + mbase + mt * 8 + g, c = j0 + nbase + nt * 8 + 2 * t4;
      acc[mt][nt][0] = (r < d && c < d) ? a[(size_t)r * d + c] : 0.0;
      acc[mt][nt][1] = (r < d && c + 1 < d) ? a[(size_t)r * d + c + 1] : 0.0;
    }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int ks = 0; ks < NB / 4; ++ks) {
    double af[2], bf[4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) af[mt] = -li[mbase + mt * 8 + g][ks * 4 + t4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = lj[nbase + nt * 8 + g][ks * 4 + t4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int r = i0 + mbase + mt * 8 + g, c = j0 + nbase + nt * 8 + 2 * t4;
      if (r < d && c < d && c <= r) a[(size_t)r * d + c] = acc[mt][nt][0];
      if (r < d && c + 1 < d && c + 1 <= r) a[(size_t)r * d + c + 1] = acc[mt][nt][1];
    }
}

// Inverse of every 64x64 diagonal block of L (one CTA per block, one thread
// per column of the inverse): lets the substitution kernel replace the
// sequential diagonal solve by a 64x64 mat-vec.
__global__ void __launch_bounds__(64) k_tri_inv_diag(const double* a, int d, double* inv,
                                                     const int* status) {
  if (*status) return;
  __shared__ double L[NB][NB + 1];
  const int k0 = blockIdx.x * NB, nb = min(NB, d - k0);
  for (int e = threadIdx.x; e < NB * NB; e += 64) {
    const int i = e / NB, j = e % NB;
    L[i][j] = (i < nb && j <= i) ? a[(size_t)(k0 + i) * d + k0 + j] : 0.0;
  }
  __syncthreads();
  const int c = threadIdx.x;  // column of the inverse: solve L x = e_c
  double* out = inv + (size_t)blockIdx.x * NB * NB;
  double x[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    double v = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int l = 0; l < i; ++l) v -= L[i][l] * x[l];
    x[i] = (i < nb && c < nb && i >= c) ? v / L[i][i] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) out[i * NB + c] = x[i];
}

// Forward (L y = b) then backward (L^T x = y) substitution; x_out receives x,
// b is used as the working vector. Cooperative launch; one grid barrier per
// 64-row block: after it every CTA recomputes the block's solution
// redundantly from the precomputed diagonal-block inverse.
__global__ void __launch_bounds__(256) k_trsv_coop(const double* a, int d, double* b,
                                                   const double* inv, double* ywork,
                                                   double* x_out, const int* status) {
  if (*status) return;
  cg::grid_group grid = cg::this_grid();
  __shared__ double xb[NB];
  __shared__ double bb[NB];
  const int nbt = ceil_div(d, NB);
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gsize = (long long)gridDim.x * blockDim.x;
  // forward: ywork = L^-1 b
  for (int k = 0; k < nbt; ++k) {
    const int k0 = k * NB, nb = min(NB, d - k0);
    const double* iv = inv + (size_t)k * NB * NB;
    if (threadIdx.x < NB) bb[threadIdx.x] = threadIdx.x < nb ? b[k0 + threadIdx.x] : 0.0;
    __syncthreads();
    if (threadIdx.x < nb) {
      double v = 0.0;
      for (int l = 0; l <= (int)threadIdx.x; ++l) v += iv[threadIdx.x * NB + l] * bb[l];
      xb[threadIdx.x] = v;
      if (blockIdx.x == 0) ywork[k0 + threadIdx.x] = v;
    }
    __syncthreads();
    for (long long i = k0 + nb + gtid; i < d; i += gsize) {
      const double* row = a + (size_t)i * d + k0;
      double s = 0.0;
      for (int l = 0; l < nb; ++l) s += row[l] * xb[l];
      b[i] -= s;
    }
    grid.sync();
  }
  // backward: x_k = L_kk^-T (y_k - sum_{i>k} L_ik^T x_i); right looking
  for (int k = nbt - 1; k >= 0; --k) {
    const int k0 = k * NB, nb = min(NB, d - k0);
    const double* iv = inv + (size_t)k * NB * NB;
    if (threadIdx.x < NB) bb[threadIdx.x] = threadIdx.x < nb ? ywork[k0 + threadIdx.x] : 0.0;
    __syncthreads();
    if (threadIdx.x < nb) {
      double v = 0.0;
      for (int l = threadIdx.x; l < nb; ++l) v += iv[l * NB + threadIdx.x] * bb[l];
      xb[threadIdx.x] = v;
      if (blockIdx.x == 0) x_out[k0 + threadIdx.x] = v;
    }
    __syncthreads();
    for (long long j = gtid; j < k0; j += gsize) {
      double s = 0.0;
      for (int r = 0; r < nb; ++r) s += a[(size_t)(k0 + r) * d + j] * xb[r];
      ywork[j] -= s;
    }
    grid.sync();
  }
}

void chol_solve(double* a, int d, double* b, int* status_dev, void* work, cudaStream_t st) {
  RTB_CUDA(cudaMemsetAsync(status_dev, 0, sizeof(int), st));
  const int nbt = ceil_div(d, NB);
  const int trsm_smem = 2 * NB * (NB + 1) * sizeof(double);
  RTB_CUDA(cudaFuncSetAttribute(k_trsm_panel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                trsm_smem));
  const int syrk_smem = 2 * NB * LDB * sizeof(double);
  RTB_CUDA(cudaFuncSetAttribute(k_syrk_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                syrk_smem));
  for (int k = 0; k < nbt; ++k) {
    k_potrf_diag<<<1, 256, 0, st>>>(a, d, k, status_dev);
    RTB_LAUNCH_CHECK();
    const int below = nbt - k - 1;
    if (below > 0) {
      k_trsm_panel<<<below, 64, trsm_smem, st>>>(a, d, k, status_dev);
      RTB_LAUNCH_CHECK();
      const int tiles = below * (below + 1) / 2;
      k_syrk_update<<<tiles, 256, syrk_smem, st>>>(a, d, k, status_dev);
      RTB_LAUNCH_CHECK();
    }
  }
  double* inv = static_cast<double*>(work);
  double* ywork = inv + (size_t)nbt * NB * NB;
  double* xout = ywork + (((size_t)d * 8 + 255) & ~size_t(255)) / 8;
  k_tri_inv_diag<<<nbt, 64, 0, st>>>(a, d, inv, status_dev);
  RTB_LAUNCH_CHECK();
  int dev = 0;
  RTB_CUDA(cudaGetDevice(&dev));
  int per_sm = 0;
  RTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trsv_coop, 256, 0));
  int sms = 0;
  RTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int grid = per_sm > 0 ? sms : 1;
  const int useful = ceil_div(d, 256);
  if (grid > useful) grid = useful;
  if (grid < 1) grid = 1;
  const double* ac = a;
  const double* ic = inv;
  const int* sc = status_dev;
  void* args[] = {(void*)&ac, (void*)&d, (void*)&b, (void*)&ic, (void*)&ywork, (void*)&xout,
                  (void*)&sc};
  RTB_CUDA(cudaLaunchCooperativeKernel((void*)k_trsv_coop, grid, 256, args, 0, st));
  RTB_CUDA(cudaMemcpyAsync(b, xout, (size_t)d * 8, cudaMemcpyDeviceToDevice, st));
}

}  // namespace rtb
