// Microbenchmark: FFMA (3-register) vs FFMA2 (fma.rn.f32x2) vs DFMA throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define N_ACC 16
#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b) {
  float acc[N_ACC];
  float x = threadIdx.x * 1e-3f, y = 1.0001f + blockIdx.x * 1e-7f;
#pragma unroll
  for (int i = 0; i < N_ACC; ++i) acc[i] = i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < N_ACC; ++i) acc[i] = fmaf(x, acc[i], y);
  }
  float s = 0; for (int i = 0; i < N_ACC; ++i) s += acc[i];
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long acc[N_ACC];
  float xf = threadIdx.x * 1e-3f, yf = 1.0001f + blockIdx.x * 1e-7f;
  unsigned long long x, y;
  asm("mov.b64 %0, {%1,%1};" : "=l"(x) : "f"(xf));
  asm("mov.b64 %0, {%1,%2};" : "=l"(y) : "f"(yf), "f"(yf*2.f));
#pragma unroll
  for (int i = 0; i < N_ACC; ++i) { float f0 = i, f1 = i + 0.5f; asm("mov.b64 %0, {%1,%2};" : "=l"(acc[i]) : "f"(f0), "f"(f1)); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < N_ACC; ++i) asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(acc[i]) : "l"(x), "l"(y));
  }
  float s = 0;
  for (int i = 0; i < N_ACC; ++i) { float f0, f1; asm("mov.b64 {%0,%1}, %2;" : "=f"(f0), "=f"(f1) : "l"(acc[i])); s += f0 + f1; }
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_dfma(float* out, float a, float b) {
  double acc[N_ACC];
  double x = threadIdx.x * 1e-3, y = 1.0001 + blockIdx.x * 1e-7;
#pragma unroll
  for (int i = 0; i < N_ACC; ++i) acc[i] = i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < N_ACC; ++i) acc[i] = fma(x, acc[i], y);
  }
  double s = 0; for (int i = 0; i < N_ACC; ++i) s += acc[i];
  if (s == 1234.5) out[0] = (float)s;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * 2;
    const char* names[3] = {"FFMA", "FFMA2(x2 flops)", "DFMA"};
    for (int k = 0; k < 3; ++k) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (k == 0) k_ffma<<<blocks, threads>>>(d, 1, 2);
        if (k == 1) k_ffma2<<<blocks, threads>>>(d, 1, 2);
        if (k == 2) k_dfma<<<blocks, threads>>>(d, 1, 2);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double fmas = (double)blocks * threads * ITERS * N_ACC * (k == 1 ? 2 : 1);
        if (rep) printf("%-16s threads/blk=%4d : %.2f TFMA/s  (%.1f FMA/clk/SM at %d MHz max)\n", names[k], threads,
               fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
      }
    }
  }
  return 0;
}
