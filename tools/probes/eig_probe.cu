// k_sym_eigen_warp probe: time + sweeps on random SPD matrices (n = 16).
#include <cstdio>
#include <cstdlib>
#define RTB_EIG_SWEEP_DEBUG 1
#include "k_small.cu"
namespace rtb {
unsigned long long& launch_counter() { static unsigned long long n = 0; return n; }
}
int main() {
  const int n = 16, nm = 4;
  double h[nm * 256];
  unsigned long long s = 7;
  auto rnd = [&]() { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return ((s >> 11) * 0x1.0p-53); };
  for (int b = 0; b < nm; ++b) {
    double F[512 * 16];
    for (int i = 0; i < 512 * 16; ++i) F[i] = rnd();
    for (int p = 0; p < 16; ++p) for (int q = 0; q < 16; ++q) { double a = 0; for (int i = 0; i < 512; ++i) a += F[i*16+p]*F[i*16+q]; h[b*256+p*16+q] = a; }
  }
  double *A, *ev, *evec; int *ns, *st;
  cudaMalloc(&A, sizeof(h)); cudaMalloc(&ev, sizeof(h)); cudaMalloc(&evec, sizeof(h)); cudaMalloc(&ns, 64); cudaMalloc(&st, 64);
  int nh[nm]; for (int b = 0; b < nm; ++b) nh[b] = n;
  cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice); cudaMemcpy(ns, nh, sizeof(nh), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    rtb::sym_eigen(A, ns, n, 256, ev, evec, st, nm, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int sh[nm]; cudaMemcpy(sh, st, sizeof(sh), cudaMemcpyDeviceToHost);
    printf("warp eigen %d mats: %.1f us, status/sweeps %d %d %d %d err %s\n", nm, ms * 1e3, sh[0], sh[1], sh[2], sh[3], cudaGetErrorString(cudaGetLastError()));
  }
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(e0);
    const int np = 16; const size_t smem = (2 * np * (np + 1) + 2 * np) * 8;
    rtb::k_sym_eigen<<<nm, 128, smem>>>(A, ns, 256, ev, evec, st);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int sh[nm]; cudaMemcpy(sh, st, sizeof(sh), cudaMemcpyDeviceToHost);
    printf("cta eigen %d mats: %.1f us, status/sweeps %d %d %d %d\n", nm, ms * 1e3, sh[0], sh[1], sh[2], sh[3]);
  }
}
