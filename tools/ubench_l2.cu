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

// The fit's access pattern with plain loads: 8 frames of 11 planar 1920 x 1080 fp32 planes;
// warp w of the grid takes items (block row by, 128-px segment sg) round robin and reads, for
// each of the 8 rows and 11 planes, one 512-byte row segment (16 B per lane), SEGW segments
// wide (SEGW = 1: the kernels' 128-px items; 15: whole 1920-px rows).
template <int SEGW>
__global__ void __launch_bounds__(1024, 1) k_items(const float4* __restrict__ p, int nf, float* sink)
{
    const int W4 = 1920 / 4, H = 1080, P = 11, nseg = 15 / SEGW;
    const int per_frame = 135 * nseg, nitems = nf * per_frame;
    const int lane = threadIdx.x & 31, GW = gridDim.x * (blockDim.x >> 5);
    float acc = 0.f;
    for (int it = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < nitems; it += GW) {
        const int f = it / per_frame, rem = it - f * per_frame, by = rem / nseg, sg = rem - by * nseg;
#pragma unroll 1
        for (int r = 0; r < 8; ++r) {
            float4 v[P * SEGW];
#pragma unroll
            for (int q = 0; q < P; ++q)
#pragma unroll
                for (int u = 0; u < SEGW; ++u)
                    v[q * SEGW + u] = __ldcs(p + (((size_t)f * P + q) * H + by * 8 + r) * W4 + (sg * SEGW + u) * 32 + lane);
#pragma unroll
            for (int q = 0; q < P * SEGW; ++q) acc += v[q].x + v[q].w;
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
    {
        const int nf = 8;
        const double bytes = 1920.0 * 1080 * 11 * 4 * nf;
        auto t = [&](auto kern, const char* name, int tpb) {
            kern<<<148, tpb>>>(reinterpret_cast<float4*>(buf), nf, sink);
            cudaEventRecord(e0);
            kern<<<148, tpb>>>(reinterpret_cast<float4*>(buf), nf, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("fit pattern %-22s threads/SM %4d  %.2f TB/s  (%s)\n", name, tpb, bytes / (ms * 1e-3) / 1e12,
                   cudaGetErrorString(cudaGetLastError()));
        };
        for (int tpb : {256, 512, 1024}) t(k_items<1>, "128-px items", tpb);
        for (int tpb : {256, 512}) t(k_items<3>, "384-px items", tpb);
    }
    return 0;
}
