// FP64 peak probe: DMMA (mma.sync m8n8k4 f64) vs scalar DFMA, sm_100a.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma16_loop(double* out, int iters) {
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 + threadIdx.x * 1e-4 + j;
  double c[4][4];
  for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) c[j][k] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) s += c[j][k];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
  for (int j = 0; j < 16; ++j) c[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = fma(c[j], b, a);
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += c[j];
  if (s == 12345.0) out[0] = s;
}

// half the warps DMMA, half DFMA: are the FP64 tensor and FP64 FMA pipes independent?
__global__ void mixed_loop(double* out, int iters) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if (w & 1) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-9;
    double c[16];
    for (int j = 0; j < 16; ++j) c[j] = j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 16; ++j) c[j] = fma(c[j], b, a);
    }
    for (int j = 0; j < 16; ++j) s += c[j];
  } else {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
    for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  }
  if (s == 12345.0) out[0] = s;
}

// DMMA fed from shared memory like the TTM kernels: per k-step 2 A + 2 B fragment
// loads (LDS.64) and 4 independent accumulators x 2 (even/odd steps)
__global__ void dmma_lds_loop(double* out, int iters) {
  __shared__ double sm[2][40][68];
  for (int e = threadIdx.x; e < 2 * 40 * 68; e += blockDim.x) (&sm[0][0][0])[e] = e * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  double c[2][4][2] = {};
  for (int it = 0; it < iters; ++it) {
    const double* a = &sm[it & 1][0][0];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      double af[2], bf[2];
#pragma unroll
      for (int m = 0; m < 2; ++m) af[m] = a[(ks * 4 + t) * 68 + m * 8 + g];
#pragma unroll
      for (int n = 0; n < 2; ++n) bf[n] = a[(ks * 4 + t) * 68 + 16 + w * 16 % 48 + n * 8 + g];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 2; ++n)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(c[ks & 1][m * 2 + n][0]), "+d"(c[ks & 1][m * 2 + n][1]) : "d"(af[m]), "d"(bf[n]));
    }
  }
  double s = 0;
  for (int h = 0; h < 2; ++h) for (int j = 0; j < 4; ++j) s += c[h][j][0] + c[h][j][1];
  if (s == 12345.0) out[0] = s;
}

// the same with m16n8k16 (A 8 + B 4 fragment loads per 2 MMAs)
__global__ void dmma16_lds_loop(double* out, int iters) {
  __shared__ double sm[2][40][68];
  for (int e = threadIdx.x; e < 2 * 40 * 68; e += blockDim.x) (&sm[0][0][0])[e] = e * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double c[2][2][4] = {};
  for (int it = 0; it < iters; ++it) {
    const double* a = &sm[it & 1][0][0];
#pragma unroll
    for (int kb = 0; kb < 32; kb += 16) {
      double af[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) af[v] = a[(g + 8 * (v & 1)) * 68 + kb + t + 4 * (v >> 1)];
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        double bf[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) bf[v] = a[(kb + t + 4 * v) * 68 + 32 + n * 8 + g];
        asm("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
            : "+d"(c[kb / 16][n][0]), "+d"(c[kb / 16][n][1]), "+d"(c[kb / 16][n][2]), "+d"(c[kb / 16][n][3])
            : "d"(af[0]), "d"(af[1]), "d"(af[2]), "d"(af[3]), "d"(af[4]), "d"(af[5]), "d"(af[6]), "d"(af[7]),
              "d"(bf[0]), "d"(bf[1]), "d"(bf[2]), "d"(bf[3]));
      }
    }
  }
  double s = 0;
  for (int h = 0; h < 2; ++h) for (int n = 0; n < 2; ++n) for (int j = 0; j < 4; ++j) s += c[h][n][j];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  for (int warps : {4, 8, 16}) {
    int iters = 20000;
    dim3 grid(sms * 2), block(32 * warps);
    dmma_loop<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * grid.x * warps;
    printf("DMMA m8n8k4 warps/CTA=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    dmma16_loop<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dmma16_loop<<<grid, block>>>(out, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * grid.x * warps;
    printf("DMMA m16n8k16 warps/CTA=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    dfma_loop<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * iters * (double)grid.x * block.x;
    printf("DFMA warps/CTA=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int warps : {8, 16}) {
    int iters = 4000;
    dim3 grid(sms), block(32 * warps);
    float ms;
    dmma_lds_loop<<<grid, block>>>(out, 10);
    cudaEventRecord(e0);
    dmma_lds_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 32 * (double)iters * grid.x * warps;
    printf("DMMA m8n8k4 from smem, 1 CTA/SM, warps=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    dmma16_lds_loop<<<grid, block>>>(out, 10);
    cudaEventRecord(e0);
    dmma16_lds_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 2048 * 4 * (double)iters * grid.x * warps;
    printf("DMMA m16n8k16 from smem, 1 CTA/SM, warps=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int warps : {8, 16}) {
    int iters = 20000;
    dim3 grid(sms * 2), block(32 * warps);
    mixed_loop<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    mixed_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // per iteration: DMMA warps 8 x 512 flops per warp, DFMA warps 16 x 2 x 32 flops per warp
    double flops = ((double)8 * 512 + 16 * 2 * 32) * (warps / 2) * iters * (double)grid.x;
    printf("MIXED (half DMMA, half DFMA) warps/CTA=%d: %.2f TFLOP/s combined\n", warps, flops / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
