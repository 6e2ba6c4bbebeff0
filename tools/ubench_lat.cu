// dependent-chain latency of DFMA / FFMA / MUFU.RSQ64H / LDS.64 on one warp
#include <cstdio>
__global__ void k(double* out, float* outf, long long* t, double a, double b, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i & 7;
  __syncthreads();
  double x = a + threadIdx.x; float y = (float)a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = fmaf(y, (float)b, (float)a);
  long long t2 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) z = rsqrt(z + 2.0);
  long long t3 = clock64();
  int idx = threadIdx.x & 7; double w = 0;
  for (int i = 0; i < n; ++i) { w += sm[idx]; idx = ((int)w + i) & 1023; }
  long long t4 = clock64();
  double q = x;
  for (int i = 0; i < n; ++i) q = 1.0 / (q + 3.0);
  long long t5 = clock64();
  out[threadIdx.x] = x + z + w + q; outf[threadIdx.x] = y;
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; }
}
int main() {
  double* o; float* of; long long* t; cudaMalloc(&o, 1024*8); cudaMalloc(&of, 4096); cudaMalloc(&t, 64);
  int n = 4096; long long h[5];
  for (int rep = 0; rep < 2; ++rep) { k<<<1, 32>>>(o, of, t, 0.999, 0.5, n); cudaMemcpy(h, t, 40, cudaMemcpyDeviceToHost); }
  printf("latency cycles/op: DFMA %.1f  FFMA %.1f  rsqrt(double)+DADD %.1f  LDS.64+DADD+cvt %.1f  ddiv+DADD %.1f\n",
         h[0]/(double)n, h[1]/(double)n, h[2]/(double)n, h[3]/(double)n, h[4]/(double)n);
  return 0;
}
