// Compute-only rate of two apply inner-loop schemes (Q = 8, D = 8), guides and models
// resident in shared memory (no TMA, no waits), one CTA of NW warps per SM, 148 CTAs:
//   A  (k_apply_ws today): lane = 4-pixel quad, its two model columns (top, bottom - top)
//      in registers, per row A_y = top + t_y (bottom - top) (28 FFMA2), then per pixel pair
//      2 x 3 x (8 FFMA2) + blend -- 32.5 FFMA2 per pixel, ~208 registers.
//   B  lane = 1 pixel column, the x-blended top and bottom models paired {top, bot} in 27
//      registers pairs (set up once per 8-row band), per row 3 x 8 FFMA2 with the guide
//      broadcast, then o = p.x + t_y (p.y - p.x) -- 24 FFMA2 + 6 FP32 per pixel.
// Prints pixels per clock per SM at the measured clock and the equivalent 1080p time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ubench_apply.cu -o /tmp/ubench_apply
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2410_11625_b200/csrc/flr_pipe.cuh"
using namespace flr;
constexpr int Q = 8, MS = 28, ROWS = 512;  // rows per warp
constexpr int GSM = Q * 128 * 2 * 2;       // floats of two guide stages (2 rows each)

template <int NW, bool STORE = false>
__global__ void __launch_bounds__(NW * 32, 1) k_a(float* sink, float ty0)
{
    extern __shared__ float sm[];
    float* gs = sm;            // [Q][2][128]
    float* ms = sm + GSM;      // [2][18][MS]
    for (int i = threadIdx.x; i < GSM + 2 * 18 * MS; i += blockDim.x) sm[i] = 1e-3f * (i % 97) + 0.25f;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int c0 = lane / 2, c1 = c0 + 1;
    constexpr int MP = MS / 2;
    f2 top0[MP], dlt0[MP], top1[MP], dlt1[MP];
#pragma unroll
    for (int v = 0; v < MS / 4; ++v) {
        const float4 p0 = reinterpret_cast<const float4*>(ms + c0 * MS)[v];
        const float4 q0 = reinterpret_cast<const float4*>(ms + (18 + c0) * MS)[v];
        const float4 p1 = reinterpret_cast<const float4*>(ms + c1 * MS)[v];
        const float4 q1 = reinterpret_cast<const float4*>(ms + (18 + c1) * MS)[v];
        top0[2 * v] = pk2(p0.x, p0.y), top0[2 * v + 1] = pk2(p0.z, p0.w);
        top1[2 * v] = pk2(p1.x, p1.y), top1[2 * v + 1] = pk2(p1.z, p1.w);
        dlt0[2 * v] = sub2(pk2(q0.x, q0.y), top0[2 * v]), dlt0[2 * v + 1] = sub2(pk2(q0.z, q0.w), top0[2 * v + 1]);
        dlt1[2 * v] = sub2(pk2(q1.x, q1.y), top1[2 * v]), dlt1[2 * v + 1] = sub2(pk2(q1.z, q1.w), top1[2 * v + 1]);
    }
    const f2 t2[2] = {pk2(0.0625f, 0.1875f), pk2(0.3125f, 0.4375f)};
    float acc = 0.f;
#pragma unroll 1
    for (int ys = 0; ys < ROWS; ys += 2) {
        float o[2][3][4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const float fy = ((float)(ys + r) + 0.5f) * 0.125f - 0.5f + ty0;
            const f2 ty2 = bc2(fy - floorf(fy));
            float gq[Q][4];
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                const float4 v = reinterpret_cast<const float4*>(gs + ((ys >> 1) & 1) * Q * 256 + (j * 2 + r) * 128)[lane];
                gq[j][0] = v.x; gq[j][1] = v.y; gq[j][2] = v.z; gq[j][3] = v.w;
            }
            float m0[MS], m1[MS];
#pragma unroll
            for (int v = 0; v < MP; ++v) {
                upk2(fma2(ty2, dlt0[v], top0[v]), m0[2 * v], m0[2 * v + 1]);
                upk2(fma2(ty2, dlt1[v], top1[v]), m1[2 * v], m1[2 * v + 1]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                f2 gp[Q];
#pragma unroll
                for (int j = 0; j < Q; ++j) gp[j] = pk2(gq[j][2 * h], gq[j][2 * h + 1]);
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    f2 p0 = bc2(m0[cc]), p1 = bc2(m1[cc]);
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        p0 = fma2(gp[j], bc2(m0[(1 + j) * 3 + cc]), p0);
                        p1 = fma2(gp[j], bc2(m1[(1 + j) * 3 + cc]), p1);
                    }
                    upk2(fma2(t2[h], sub2(p1, p0), p0), o[r][cc][2 * h], o[r][cc][2 * h + 1]);
                }
            }
        }
        if (STORE) {  // like k_apply_ws: 3 planes of a 1920 x 1080 frame, streaming stores
            const int item = blockIdx.x * NW + (threadIdx.x >> 5);
            const int xq = (item % 15) * 128 + lane * 4;
            const int y0 = ((item / 15) * ROWS + ys) % 1080;
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    float* Orow = sink + (size_t)cc * 1920 * 1080 + (size_t)(y0 + r) * 1920 + xq;
                    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(Orow), "f"(o[r][cc][0]), "f"(o[r][cc][1]),
                                 "f"(o[r][cc][2]), "f"(o[r][cc][3])
                                 : "memory");
                }
        } else {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) acc += (o[r][cc][0] + o[r][cc][1]) + (o[r][cc][2] + o[r][cc][3]);
        }
    }
    if (acc == 1234.5f) sink[threadIdx.x] = acc;
}

// B: RR rows per step, lane = one pixel column of a 32-px slice (4 slices per 128-px stage)
template <int NW, int RR>
__global__ void __launch_bounds__(NW * 32, 1) k_b(float* sink, float ty0)
{
    extern __shared__ float sm[];
    float* gs = sm;        // [Q][RR][128]
    float* ms = sm + 2 * Q * RR * 128;  // [2][18][MS]
    for (int i = threadIdx.x; i < 2 * Q * RR * 128 + 2 * 18 * MS; i += blockDim.x) sm[i] = 1e-3f * (i % 97) + 0.25f;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, sl = w & 3;
    const int x = sl * 32 + lane;
    const float fx = (x + 0.5f) * 0.125f - 0.5f;
    const int ib = (int)floorf(fx);
    const float tx = fx - ib;
    const int c0 = max(ib, 0), c1 = min(ib + 1, 16);
    float acc = 0.f;
#pragma unroll 1
    for (int band = 0; band < ROWS / 8; ++band) {
        f2 tb[27];  // {top, bottom} of the x-blended model, component k
#pragma unroll
        for (int k = 0; k < 27; ++k) {
            const float a0 = ms[c0 * MS + k], a1 = ms[c1 * MS + k];
            const float b0 = ms[(18 + c0) * MS + k], b1 = ms[(18 + c1) * MS + k];
            tb[k] = fma2(bc2(tx), sub2(pk2(a1, b1), pk2(a0, b0)), pk2(a0, b0));
        }
#pragma unroll 1
        for (int r0 = 0; r0 < 8; r0 += RR) {
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                const float fy = ((float)(band * 8 + r0 + r) + 0.5f) * 0.125f - 0.5f + ty0;
                const float ty = fy - floorf(fy);
                float g[Q];
#pragma unroll
                for (int j = 0; j < Q; ++j) g[j] = gs[((r0 / RR) & 1) * Q * RR * 128 + (j * RR + r) * 128 + x];
                f2 p[3];
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) p[cc] = tb[cc];
#pragma unroll
                for (int j = 0; j < Q; ++j)
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) p[cc] = fma2(bc2(g[j]), tb[(1 + j) * 3 + cc], p[cc]);
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    float lo, hi;
                    upk2(p[cc], lo, hi);
                    acc += fmaf(ty, hi - lo, lo);
                }
            }
        }
    }
    if (acc == 1234.5f) sink[threadIdx.x] = acc;
}

template <class K>
static void run(const char* name, K kern, int nw, int px_per_warp, size_t smem)
{
    float* sink;
    cudaMalloc(&sink, 3 * 1920 * 1088 * 4);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) kern<<<148, nw * 32, smem>>>(sink, 0.f);
    cudaEventRecord(e0);
    const int REP = 20;
    for (int i = 0; i < REP; ++i) kern<<<148, nw * 32, smem>>>(sink, 0.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double sec = ms * 1e-3 / REP;
    const double px = 148.0 * nw * px_per_warp;
    const double pxclk = px / 148.0 / (sec * 1.965e9);
    printf("%-4s NW=%2d regs=%3d spill=%zu  %.3f px/clk/SM  1080p-equivalent %.2f us  (%s)\n", name, nw, fa.numRegs,
           (size_t)fa.localSizeBytes, pxclk, 2073600.0 / (pxclk * 148 * 1.965e9) * 1e6, cudaGetErrorString(cudaGetLastError()));
    cudaFree(sink);
}

int main()
{
    const size_t sa = (GSM + 2 * 18 * MS) * 4;
    run("A", k_a<4>, 4, ROWS * 128, sa);
    run("A", k_a<7>, 7, ROWS * 128, sa);
    run("A", k_a<8>, 8, ROWS * 128, sa);
    run("A", k_a<12>, 12, ROWS * 128, sa);
    run("A", k_a<16>, 16, ROWS * 128, sa);
    run("As", k_a<7, true>, 7, ROWS * 128, sa);
    run("As", k_a<8, true>, 8, ROWS * 128, sa);
    run("As", k_a<12, true>, 12, ROWS * 128, sa);
    const size_t sb2 = (2 * Q * 2 * 128 + 2 * 18 * MS) * 4, sb4 = (2 * Q * 4 * 128 + 2 * 18 * MS) * 4;
    run("B2", k_b<4, 2>, 4, ROWS * 32, sb2);
    run("B2", k_b<8, 2>, 8, ROWS * 32, sb2);
    run("B2", k_b<12, 2>, 12, ROWS * 32, sb2);
    run("B2", k_b<16, 2>, 16, ROWS * 32, sb2);
    run("B2", k_b<24, 2>, 24, ROWS * 32, sb2);
    run("B2", k_b<32, 2>, 32, ROWS * 32, sb2);
    run("B4", k_b<8, 4>, 8, ROWS * 32, sb4);
    run("B4", k_b<16, 4>, 16, ROWS * 32, sb4);
    run("B4", k_b<24, 4>, 24, ROWS * 32, sb4);
    return 0;
}
