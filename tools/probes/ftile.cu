// factor_tile micro-probe: phase clocks of the 64x64 diagonal-tile Cholesky.
#include <cstdio>
#include <cmath>
#include "k_chol.cu"
namespace rtb {
unsigned long long& launch_counter() { static unsigned long long n = 0; return n; }
__global__ void k_ft(const double* g, double* out, int* status, long long* clk) {
  extern __shared__ __align__(16) double smem[];
  double(*ta)[LDT] = reinterpret_cast<double(*)[LDT]>(smem);
  double(*tb)[LDT] = reinterpret_cast<double(*)[LDT]>(smem + NB * LDT);
  double(*tw)[LDW] = reinterpret_cast<double(*)[LDW]>(smem + 2 * NB * LDT);
  if (threadIdx.x == 0) g_ftclk = clk;
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) { tw[e / 64][e % 64] = g[e]; tb[e / 64][e % 64] = 0.0; }
  __syncthreads();
  __shared__ double sd[64];
  factor_tile(tw, ta, tb, 0, status, sd);
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) { out[e] = ta[e / 64][e % 64]; out[4096 + e] = tb[e / 64][e % 64]; }
}
}
int main() {
  double h[4096];
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j) ? 2.0 : 1.0 / (1 + i + j);
  double *g, *o; int* st; long long* clk;
  cudaMalloc(&g, 4096 * 8); cudaMalloc(&o, 8192 * 8); cudaMalloc(&st, 4); cudaMalloc(&clk, 32 * 8);
  cudaMemcpy(g, h, 4096 * 8, cudaMemcpyHostToDevice); cudaMemset(st, 0, 4);
  const int smem = (2 * 64 * 68 + 64 * 68) * 8;
  cudaFuncSetAttribute(rtb::k_ft, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int r = 0; r < 3; ++r) rtb::k_ft<<<1, 256, smem>>>(g, o, st, clk);
  cudaDeviceSynchronize();
  long long c[32]; cudaMemcpy(c, clk, 32 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"start", "p16 b0", "trsm b0", "syrk b0", "p16 b1", "trsm b1", "syrk b1", "p16 b2", "trsm b2", "syrk b2", "p16 b3", "-", "-", "linv"};
  long long prev = c[0];
  for (int i = 1; i < 14; ++i) { if (i == 11 || i == 12) continue; printf("%-8s %6lld cycles\n", nm[i], c[i] - prev); prev = c[i]; }
  // check L L^T = G and Linv L = I on the host
  double L[8192]; cudaMemcpy(L, o, 8192 * 8, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < 64; ++i) for (int j = 0; j <= i; ++j) { double s = 0; for (int k = 0; k < 64; ++k) s += L[i*64+k]*L[j*64+k]; e1 = fmax(e1, fabs(s - h[i*64+j])); }
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) { double s = 0; for (int k = 0; k < 64; ++k) s += L[4096+i*64+k]*L[k*64+j]; e2 = fmax(e2, fabs(s - (i==j))); }
  printf("max |LL^T - G| %.3e  max |Linv L - I| %.3e  status %d\n", e1, e2, 0);
  printf("potrf16 part of p16 b0: %lld cycles, inverse16 part: %lld\n", c[16] - c[0], c[1] - c[16]);
  printf("total %lld cycles, err %s\n", c[13] - c[0], cudaGetErrorString(cudaGetLastError()));
}
