// latency of one solve_block<8> per thread (1 warp) and throughput with many warps
#include <cstdio>
#include "../paper_2410_11625_b200/csrc/flr_solve.cuh"
using namespace flr;
__global__ void k(const double* in, float* out, long long* t, int reps) {
  double m[Dims<8>::KM];
#pragma unroll
  for (int k = 0; k < Dims<8>::KM; ++k) m[k] = in[k * 32 + (threadIdx.x & 31)];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    solve_block<8>([&](int k) { return m[k]; }, 1e-5, 1e-4, out + (threadIdx.x + blockIdx.x * blockDim.x) * 28);
    m[0] += out[(threadIdx.x + blockIdx.x * blockDim.x) * 28] * 1e-30;  // serialise reps
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) t[0] = (t1 - t0) / reps;
}
int main() {
  double h[72 * 32];
  for (int k = 0; k < 72; ++k) for (int l = 0; l < 32; ++l) h[k * 32 + l] = (k == 0 ? 64.0 : (k < 9 ? 32.0 + 0.1 * k : 20.0 + 0.01 * k + (k % 9 == 0 ? 5.0 : 0.0))) + 0.001 * l;
  // make it SPD-ish: diagonal S entries large
  double* d; float* o; long long* t; cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 148 * 1024 * 28 * 4); cudaMalloc(&t, 8);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  long long c;
  k<<<1, 32>>>(d, o, t, 20); cudaMemcpy(&c, t, 8, cudaMemcpyDeviceToHost);
  printf("solve_block<8>: %lld cycles per block (1 warp)\n", c);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w : {4, 8, 16}) {
    cudaEventRecord(a); k<<<148, 32 * w>>>(d, o, t, 20); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); cudaMemcpy(&c, t, 8, cudaMemcpyDeviceToHost);
    printf("  %2d warps/SM: %lld cycles/solve/thread, %.2f ns per block-solve (GPU-wide)\n", w, c, ms * 1e6 / (148.0 * 32 * w * 20));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
