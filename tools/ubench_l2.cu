// L2 -> SM read bandwidth on B200: every SM streams an L2-resident buffer of MB megabytes
// (16-byte loads, 4 independent per thread in flight), many passes; compare with a buffer
// far larger than L2 (HBM).  Prints TB/s per buffer size.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench_l2.cu -o tools/ubench_l2
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) k_read(const float4* __restrict__ p, size_t n4, int passes, float* sink)
{
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int ps = 0; ps < passes; ++ps) {
        // rotate the starting SM each pass so no SM keeps re-reading its own slice from L1
        const size_t t0 = ((size_t)((blockIdx.x + ps * 37) % gridDim.x) * blockDim.x + threadIdx.x);
        for (size_t i = t0; i < n4; i += 4 * stride) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const size_t j = i + u * stride;
                v[u] = j < n4 ? __ldcg(p + j) : make_float4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
    }
    if (acc == 1234.5f) sink[0] = acc;
}

int main()
{
    float* buf;
    float* sink;
    const size_t maxb = (size_t)1 << 30;
    cudaMalloc(&buf, maxb);
    cudaMalloc(&sink, 64);
    cudaMemset(buf, 0, maxb);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (size_t mb : {8, 16, 32, 48, 64, 96, 1024}) {
        const size_t bytes = mb << 20, n4 = bytes / 16;
        const int passes = mb >= 1024 ? 2 : (int)(4096 / mb);
        for (int tpb : {512, 1024}) {
            k_read<<<148, tpb>>>(reinterpret_cast<float4*>(buf), n4, 1, sink);
            cudaEventRecord(e0);
            k_read<<<148, tpb>>>(reinterpret_cast<float4*>(buf), n4, passes, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("buffer %5zu MB  threads/SM %4d  %.2f TB/s  (%s)\n", mb, tpb, (double)bytes * passes / (ms * 1e-3) / 1e12,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
