// Per-SM TMA read rate: G CTAs, each with NW warps; lane 0 of each warp keeps S stages of
// one 3-D box in flight (box {BX px, BY rows, 11 planes} of planar fp32 1080p frames), the
// warp touches one float per lane of each stage and releases it.  No math: the rate one SM's
// TMA path sustains for a given box shape and bytes in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda tools/t_tma_rate.cu -o tools/t_tma_rate
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2410_11625_b200/csrc/flr_pipe.cuh"
using namespace flr;

struct Args {
    CUtensorMap tm, tm2;  // tm2: second tensor (split mode: planes P1.. of the stage)
    int W, H, P, nf, bx, by, rpi, split;  // rpi: consecutive box rows per item; split: planes in tm
};

__global__ void __launch_bounds__(512, 1) k_tma(const __grid_constant__ Args a, int nw, int S, int stg_floats, float* out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* stages = reinterpret_cast<float*>(sm) + (size_t)w * S * stg_floats;
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(sm) + (size_t)nw * S * stg_floats) + w * S;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    __syncthreads();
    const int nseg = a.W / a.bx, nrow = a.H / (a.by * a.rpi);
    const int per_frame = nseg * nrow, nitems = per_frame * a.nf;
    const int GW = gridDim.x * nw, first = blockIdx.x * nw + w;
    const unsigned bytes = a.bx * a.by * a.P * 4;
    const uint64_t pol = policy_evict_first();
    int pit = first, prow = 0;
    unsigned prod = 0, cons = 0;
    auto issue = [&]() {
        while (prod < cons + S && pit < nitems) {
            const int f = pit / per_frame, rem = pit % per_frame;
            uint64_t* b = &bars[prod % S];
            mbar_arrive_expect_tx(b, bytes);
            const int x = (rem % nseg) * a.bx, y = ((rem / nseg) * a.rpi + prow) * a.by;
            float* dst = stages + (size_t)(prod % S) * stg_floats;
            if (a.split) {
                tma_load_3d(dst, &a.tm, x, y, f * a.split, b, pol);
                tma_load_3d(dst + a.bx * a.by * a.split, &a.tm2, x, y, f * (a.P - a.split), b, pol);
            } else {
                tma_load_3d(dst, &a.tm, x, y, f * a.P, b, pol);
            }
            ++prod;
            if (++prow == a.rpi) {
                prow = 0;
                pit += GW;
            }
        }
    };
    if (lane == 0) issue();
    float acc = 0.f;
    const int mine = first < nitems ? (nitems - first + GW - 1) / GW * a.rpi : 0;
    for (int i = 0; i < mine; ++i) {
        mbar_wait(&bars[cons % S], (cons / S) & 1);
        acc += stages[(size_t)(cons % S) * stg_floats + lane];
        __syncwarp();
        ++cons;
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue();
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

// warp-specialised: warp NC = producer, lane c feeds consumer warp c (full/empty mbarriers,
// non-blocking test_wait round robin, like k_fit_ws); consumers wait, touch, release
__global__ void __launch_bounds__(512, 1) k_ws(const __grid_constant__ Args a, int NC, int S, int stg_floats, float* out,
                                              int spin)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(sm) + (size_t)NC * S * stg_floats);
    uint64_t* empty = full + NC * S;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NC * S; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int nseg = a.W / a.bx, nrow = a.H / (a.by * a.rpi);
    const int per_frame = nseg * nrow, nitems = per_frame * a.nf;
    const int GW = gridDim.x * NC;
    const unsigned bytes = a.bx * a.by * a.P * 4;
    const uint64_t pol = policy_evict_first();
    if (w == NC) {
        if (lane >= NC) return;
        const int c = lane;
        int it = blockIdx.x * NC + c, prow = 0, k = 0;
        const unsigned mask = (1u << NC) - 1;
        while (__any_sync(mask, it < nitems)) {
            const int slot = k % S;
            if (it < nitems && (k < S || mbar_test_wait(&empty[c * S + slot], ((k / S) - 1) & 1))) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const int f = it / per_frame, rem = it % per_frame;
                uint64_t* b = &full[c * S + slot];
                mbar_arrive_expect_tx(b, bytes);
                const int x = (rem % nseg) * a.bx, y = ((rem / nseg) * a.rpi + prow) * a.by;
                float* dst = reinterpret_cast<float*>(sm) + (size_t)(c * S + slot) * stg_floats;
                tma_load_3d(dst, &a.tm, x, y, f * a.split, b, pol);
                tma_load_3d(dst + a.bx * a.by * a.split, &a.tm2, x, y, f * (a.P - a.split), b, pol);
                ++k;
                if (++prow == a.rpi) {
                    prow = 0;
                    it += GW;
                }
            }
        }
        return;
    }
    float acc = 0.f;
    const int first = blockIdx.x * NC + w;
    const int mine = first < nitems ? (nitems - first + GW - 1) / GW * a.rpi : 0;
    for (int k = 0; k < mine; ++k) {
        const int slot = k % S;
        mbar_wait(&full[w * S + slot], (k / S) & 1);
        acc += reinterpret_cast<float*>(sm)[(size_t)(w * S + slot) * stg_floats + lane];
        if (spin > 0) {
            for (int i = 0; i < spin; ++i) acc = fmaf(acc, 1.0001f, 0.5f);
        } else if (spin < 0) {  // issue-heavy hold: -spin rounds of 32 independent FFMA2 (the fit's mix)
            f2 h[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) h[j] = pk2(acc + j, acc - j);
            for (int i = 0; i < -spin; ++i)
#pragma unroll
                for (int j = 0; j < 32; ++j) h[j] = fma2(h[j], h[(j + 1) & 31], h[j]);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += lo2(h[j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[w * S + slot]);
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main()
{
    const int W = 1920, H = 1080, P = 11, NF = 8;
    const size_t n = (size_t)W * H * P * NF;
    float *d, *d2, *o;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&d2, n * 4);
    cudaMemset(d2, 0, n * 4);
    cudaMalloc(&o, 4);
    cudaMemset(d, 0, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    struct Cfg { int bx, by, nw, S, rpi, split; };
    const Cfg cfgs[] = {{128, 1, 8, 4, 1, 0}, {128, 1, 8, 4, 8, 0}, {128, 1, 8, 4, 1, 8}, {128, 1, 8, 4, 8, 8},
                        {128, 1, 16, 2, 8, 8}, {128, 1, 12, 3, 8, 8}, {256, 1, 8, 2, 8, 8}, {128, 2, 8, 2, 4, 8},
                        {64, 1, 16, 4, 8, 8}, {128, 1, 4, 8, 8, 8}};
    cudaFuncSetAttribute(k_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const bool spins = getenv("TMA_SPINS") != nullptr;  // the fit's protocol with a per-stage hold time
    for (int G : {37, 148}) {
        struct WC { int NC, S, rb; };
        const std::vector<int> spin_list = spins ? std::vector<int>{0, 400, -4, -6, -8, -10} : std::vector<int>{0};
        const std::vector<WC> wc_list = spins ? std::vector<WC>{WC{7, 2, 2}}
                                              : std::vector<WC>{WC{7, 4, 1}, WC{7, 2, 2}, WC{6, 3, 2}, WC{7, 1, 4}, WC{3, 2, 4}, WC{5, 2, 2}};
        for (int spin : spin_list) {
            for (WC wc : wc_list) {
            const int NC = wc.NC, S = wc.S;
            Args a;
            a.W = W, a.H = H, a.P = P, a.nf = NF, a.bx = 128, a.by = wc.rb, a.rpi = 8 / wc.rb, a.split = 8;
            const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)P * NF};
            const cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
            const cuuint32_t box[3] = {128, (cuuint32_t)wc.rb, 8}, box2[3] = {128, (cuuint32_t)wc.rb, 3}, es[3] = {1, 1, 1};
            enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            enc(&a.tm2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d2, dims, str, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int stg = 128 * 11 * wc.rb;
            const size_t smem = (size_t)NC * S * stg * 4 + 2 * NC * S * 8;
            if (smem > 227 * 1024) { printf("skip\n"); continue; }
            float ms = 0;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                k_ws<<<G, (NC + 1) * 32, smem>>>(a, NC, S, stg, o, spin);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            const double bytes = (double)n * 4;
            printf("WS   G=%3d consumers %2d S %d rows/box %d spin %3d: %6.0f GB/s = %5.1f GB/s/SM %s\n", G, NC, S, wc.rb, spin,
                   bytes / ms / 1e6, bytes / ms / 1e6 / G, cudaGetErrorString(cudaGetLastError()));
            }
        }
        if (spins) continue;
        for (const Cfg& c : cfgs) {
            Args a;
            a.W = W, a.H = H, a.P = P, a.nf = NF, a.bx = c.bx, a.by = c.by, a.rpi = c.rpi, a.split = c.split;
            const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)P * NF};
            const cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
            const cuuint32_t box[3] = {(cuuint32_t)c.bx, (cuuint32_t)c.by, (cuuint32_t)(c.split ? c.split : P)};
            const cuuint32_t box2[3] = {(cuuint32_t)c.bx, (cuuint32_t)c.by, (cuuint32_t)(P - c.split)};
            const cuuint32_t es[3] = {1, 1, 1};
            enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (c.split)
                enc(&a.tm2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d2, dims, str, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int stg = c.bx * c.by * P;
            const size_t smem = (size_t)c.nw * c.S * stg * 4 + c.nw * c.S * 8;
            if (smem > 227 * 1024) {
                printf("skip bx=%d by=%d nw=%d S=%d (smem %zu)\n", c.bx, c.by, c.nw, c.S, smem);
                continue;
            }
            float ms = 0;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                k_tma<<<G, c.nw * 32, smem>>>(a, c.nw, c.S, stg, o);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            const double bytes = (double)n * 4;
            printf("G=%3d box {%3d,%d,11} rpi %d split %d warps %2d S %d (%3.0f KB in flight/SM): %6.0f GB/s = %5.1f GB/s/SM %s\n",
                   G, c.bx, c.by, c.rpi, c.split, c.nw, c.S, c.nw * c.S * stg * 4 / 1024.0, bytes / ms / 1e6, bytes / ms / 1e6 / G,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
