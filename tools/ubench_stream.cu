// Microbenchmark: how fast can one SM-resident ring pipeline stream planar fp32 data?
//   (a) LDG.128 grid-stride read (reference)
//   (b) per-warp rings fed by 3-D TMA boxes {128 px, R rows, P planes}, S stages, NW warps/CTA
// Reads n_frames x P planes of W x H floats; reports GB/s.  Build: nvcc -arch=sm_100a -O3 -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2410_11625_b200/csrc/flr_pipe.cuh"

using namespace flr;

__global__ void k_ldg(const float4* __restrict__ p, size_t n4, float* out)
{
    float acc = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "l"(p + i));
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

struct Args {
    CUtensorMap tm;
    int W, H, P, nframes, rows_per_box, rows_per_item;
};

// each warp walks items = (frame, row-group, segment) round-robin; a stage = one box
template <int S>
__global__ void __launch_bounds__(512, 1) k_tma(const __grid_constant__ Args a, int nw, int stg_floats, float* out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* stages = reinterpret_cast<float*>(sm) + (size_t)w * S * stg_floats;
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(sm) + (size_t)nw * S * stg_floats) + w * S;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    __syncthreads();
    const int nseg = a.W / 128, ngrp = a.H / (a.rows_per_box * a.rows_per_item);
    const int per_frame = nseg * ngrp, nitems = per_frame * a.nframes;
    int prow = 0;
    const int GW = gridDim.x * nw, first = blockIdx.x * nw + w;
    const unsigned bytes = 128 * a.rows_per_box * a.P * 4;
    const uint64_t pol = policy_evict_first();
    int pit = first;
    unsigned prod = 0, cons = 0;
    auto issue = [&]() {
        while (prod < cons + S && pit < nitems) {
            const int f = pit / per_frame, rem = pit % per_frame;
            uint64_t* b = &bars[prod % S];
            mbar_arrive_expect_tx(b, bytes);
            tma_load_3d(stages + (size_t)(prod % S) * stg_floats, &a.tm, (rem % nseg) * 128,
                        ((rem / nseg) * a.rows_per_item + prow) * a.rows_per_box, f * a.P, b, pol);
            ++prod;
            if (++prow == a.rows_per_item) {
                prow = 0;
                pit += GW;
            }
        }
    };
    if (lane == 0) issue();
    float acc = 0.f;
    const int my_items = first < nitems ? (nitems - first + GW - 1) / GW : 0;
    for (int st_i = 0; st_i < my_items * a.rows_per_item; ++st_i) {
        mbar_wait(&bars[cons % S], (cons / S) & 1);
        const float* st = stages + (size_t)(cons % S) * stg_floats;
        for (int i = lane; i < stg_floats / 4; i += 32) {
            const float4 v = reinterpret_cast<const float4*>(st)[i];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        ++cons;
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue();
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv)
{
    const int W = 1920, H = 1080, P = 11, NF = 8;
    const size_t n = (size_t)W * H * P * NF;
    float *d, *o;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&o, 4);
    cudaMemset(d, 0, n * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_ldg<<<sms * 4, 512>>>(reinterpret_cast<const float4*>(d), n / 4, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("LDG.128 grid-stride: %.0f GB/s\n", n * 4 / ms / 1e6);

    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    for (int rpi : {1, 8}) {
        for (int nf : {1, 8}) {
            for (int S : {2, 3, 4}) {
                for (int nw : {4, 8, 12}) {
                    const int rpb = 1;
                    Args a;
                    a.W = W, a.H = H, a.P = P, a.nframes = nf, a.rows_per_box = rpb, a.rows_per_item = rpi;
                    const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)P * NF};
                    const cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
                    const cuuint32_t box[3] = {128, (cuuint32_t)rpb, (cuuint32_t)P};
                    const cuuint32_t es[3] = {1, 1, 1};
                    enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                    const int stg = 128 * rpb * P;
                    const size_t smem = (size_t)nw * S * stg * 4 + nw * S * 8;
                    if (smem > 227 * 1024) continue;
                    auto kern = S == 2 ? k_tma<2> : S == 3 ? k_tma<3> : S == 4 ? k_tma<4> : k_tma<6>;
                    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    for (int rep = 0; rep < 4; ++rep) {
                        cudaEventRecord(e0);
                        kern<<<sms, nw * 32, smem>>>(a, nw, stg, o);
                        cudaEventRecord(e1);
                        cudaEventSynchronize(e1);
                        cudaEventElapsedTime(&ms, e0, e1);
                    }
                    cudaError_t err = cudaGetLastError();
                    const double bytes = (double)W * (H / (rpi * rpb) * rpi * rpb) * P * 4 * nf;
                    printf("rows/item=%d frames=%d S=%d warps=%2d: %7.1f us/frame %6.0f GB/s %s\n", rpi, nf, S, nw,
                           1e3 * ms / nf, bytes / ms / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
                }
            }
        }
    }
    return 0;
}
