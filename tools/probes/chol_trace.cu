// chol_trace: times the tile-DAG Cholesky on a diagonally dominant SPD matrix
// and dumps per-task (grab, ready, end, sm) timestamps for analysis.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2107_10654_b200/csrc \
//   tools/probes/chol_trace.cu paper_2107_10654_b200/csrc/k_chol.cu -o chol_trace
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <unistd.h>
#include <cstring>
#include "kernels.h"
#include "common.cuh"

namespace rtb {
unsigned long long& launch_counter() { static unsigned long long n = 0; return n; }
}

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int d = argc > 1 ? atoi(argv[1]) : 4096;
  const int reps = argc > 2 ? atoi(argv[2]) : 3;
  std::vector<double> g((size_t)d * d), b(d);
  unsigned long long s = 12345;
  auto rnd = [&]() { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return ((s >> 11) * 0x1.0p-53) * 2 - 1; };
  for (int i = 0; i < d; ++i) for (int j = 0; j <= i; ++j) { double v = rnd() / d; g[(size_t)i*d+j] = v; g[(size_t)j*d+i] = v; }
  for (int i = 0; i < d; ++i) { g[(size_t)i*d+i] = 1.5 + rnd() * 0.25; b[i] = rnd(); }
  double *G, *Gw, *B; int* st; void* work;
  cudaMalloc(&G, (size_t)d*d*8); cudaMalloc(&Gw, (size_t)d*d*8); cudaMalloc(&B, d*8); cudaMalloc(&st, 4);
  cudaMalloc(&work, rtb::chol_work_bytes(d));
  cudaMemcpy(G, g.data(), (size_t)d*d*8, cudaMemcpyHostToDevice);
  const int nt = rtb::chol_task_count(d);
  unsigned long long* tr; cudaMalloc(&tr, (size_t)nt * 32);
  cudaStream_t strm; cudaStreamCreate(&strm);
  int* prog_h; cudaHostAlloc(&prog_h, 4096, cudaHostAllocMapped); memset(prog_h, 0, 4096);
  int* prog_d; cudaHostGetDevicePointer(&prog_d, prog_h, 0);
  rtb::chol_set_progress(prog_d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < reps + 1; ++r) {
    if (r == reps) rtb::chol_set_trace(tr);
    cudaMemcpyAsync(Gw, G, (size_t)d*d*8, cudaMemcpyDeviceToDevice, strm);
    cudaMemcpyAsync(B, b.data(), d*8, cudaMemcpyHostToDevice, strm);
    cudaEventRecord(e0, strm);
    printf("launching rep %d\n", r);
    rtb::chol_solve(Gw, d, B, st, work, strm);
    cudaEventRecord(e1, strm);
    for (int it = 0; it < 100 && cudaStreamQuery(strm) == cudaErrorNotReady; ++it) {
      usleep(50000);
      if (it % 20 == 19) printf("  waiting: grabbed %d check %d P-stage %d cta0 %d cta1 %d\n", ((volatile int*)prog_h)[0], ((volatile int*)prog_h)[1], ((volatile int*)prog_h)[2], ((volatile int*)prog_h)[4], ((volatile int*)prog_h)[5]);
    }
    if (cudaStreamQuery(strm) == cudaErrorNotReady) { printf("HUNG\n"); _exit(3); }
    cudaStreamSynchronize(strm);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int status; cudaMemcpy(&status, st, 4, cudaMemcpyDeviceToHost);
    int dbg[4]; rtb::chol_debug(d, work, dbg);
    if (dbg[0]) printf("WATCHDOG: flag %d value %d wanted %d\n", dbg[1], dbg[2], dbg[3]);
    printf("rep %d%s: chol_solve d=%d %.3f ms status %d err %s\n", r, r == reps ? " (traced)" : "", d, ms, status, cudaGetErrorString(cudaGetLastError()));
  }
  // residual check
  std::vector<double> x(d);
  cudaMemcpy(x.data(), B, d*8, cudaMemcpyDeviceToHost);
  double rn = 0, bn = 0;
  for (int i = 0; i < d; ++i) { double r = -b[i]; for (int j = 0; j < d; ++j) r += g[(size_t)i*d+j]*x[j]; rn += r*r; bn += b[i]*b[i]; }
  printf("relative residual %.3e\n", sqrt(rn / bn));
  std::vector<unsigned long long> h((size_t)nt * 4);
  cudaMemcpy(h.data(), tr, (size_t)nt*32, cudaMemcpyDeviceToHost);
  std::vector<int> tab((size_t)nt * 4);
  rtb::chol_task_table(d, tab.data());
  unsigned long long t0 = ~0ULL, t1 = 0;
  for (int t = 0; t < nt; ++t) { t0 = std::min(t0, h[4*t]); t1 = std::max(t1, h[4*t+2]); }
  double wait[4] = {0}, exec[4] = {0}; int cnt[4] = {0};
  for (int t = 0; t < nt; ++t) { int ty = tab[4*t]; wait[ty] += h[4*t+1]-h[4*t]; exec[ty] += h[4*t+2]-h[4*t+1]; cnt[ty]++; }
  const char* nm[4] = {"P", "S", "U", "Urow"};
  printf("DAG span %.3f ms, tasks %d\n", (t1 - t0) * 1e-6, nt);
  for (int ty = 0; ty < 4; ++ty) if (cnt[ty]) printf("  %s: n=%6d  mean wait %8.2f us  mean exec %8.2f us  total exec %.2f ms\n", nm[ty], cnt[ty], wait[ty]/cnt[ty]*1e-3, exec[ty]/cnt[ty]*1e-3, exec[ty]*1e-6);
  // panel timeline
  printf("panel  P_grab   P_ready   P_end (us since start)\n");
  for (int t = 0; t < nt; ++t) if (tab[4*t] == 0 && (tab[4*t+1] % 8 == 0 || tab[4*t+1] > d/64 - 3))
    printf("  P(%2d) %8.1f %8.1f %8.1f\n", tab[4*t+1], (h[4*t]-t0)*1e-3, (h[4*t+1]-t0)*1e-3, (h[4*t+2]-t0)*1e-3);
  // grab-order vs time: how far ahead the front is
  return 0;
}
