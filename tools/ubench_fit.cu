// Microbenchmark of the streaming FIT / APPLY kernels on one 1080p Q=8 frame set (no Python).
// Variants are selected at compile time (see tools/ubench_fit.sh).
#include <cstdio>
#include <vector>

#include "../paper_2410_11625_b200/csrc/flr_launch.h"
#include "../paper_2410_11625_b200/csrc/flr_persist.cuh"

using namespace flr;
#ifdef FLR_DBG_TIMES
namespace flr {
__device__ unsigned long long g_flr_wait_cycles[4096];
__device__ unsigned long long g_flr_total_cycles[4096];
__device__ int g_flr_items[4096];
}
#endif

int main()
{
    constexpr int Q = 8, D = 8;
    const int W = 1920, H = 1080, NF = 4;
    const int Bx = W / D, By = (H + D - 1) / D;
    const size_t plane = (size_t)W * H;
    float *G, *Y, *M, *O;
    double* mom;
    cudaMalloc(&G, plane * Q * NF * 4);
    cudaMalloc(&Y, plane * 3 * NF * 4);
    cudaMalloc(&O, plane * 3 * NF * 4);
    cudaMalloc(&M, (size_t)Bx * By * NF * Dims<Q>::MSTRIDE * 4);
    cudaMalloc(&mom, (size_t)Bx * By * NF * Dims<Q>::KM * 8);
    std::vector<float> h(plane * Q * NF);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)((i * 2654435761u) % 1000) * 1e-3f;
    cudaMemcpy(G, h.data(), plane * Q * NF * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(Y, h.data(), plane * 3 * NF * 4, cudaMemcpyHostToDevice);
    cudaMemset(M, 0, (size_t)Bx * By * NF * Dims<Q>::MSTRIDE * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);

    FitArgs fa;
    make_tmap_planes(&fa.tg, G, W, H, NF * Q, kSeg, Q);
    make_tmap_planes(&fa.ty, Y, W, H, NF * 3, kSeg, 3);
    fa.mom = mom, fa.W = W, fa.H = H, fa.Bx = Bx, fa.Bxp = mom_pitch(Bx), fa.By = By, fa.nseg = W / kSeg;
    using FC = FitCfg<Q>;
    cudaFuncSetAttribute(k_fit_stream<Q, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FC::SMEM);
    float ms = 0;
    for (int nf : {1, 4}) {
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            k_fit_stream<Q, D><<<sms, FC::THREADS, FC::SMEM>>>(fa, nf);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("fit   nf=%d warps=%d S=%d: %7.1f us/frame  %6.0f GB/s (%s)\n", nf, FC::NSW, FC::S, 1e3 * ms / nf,
               plane * (Q + 3) * 4.0 * nf / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
#ifdef FLR_DBG_TIMES
        {
            static unsigned long long w[4096], tt[4096];
            static int it[4096];
            cudaMemset(g_flr_wait_cycles, 0, 0);
            unsigned long long zero[4096] = {};
            cudaMemcpyToSymbol(g_flr_wait_cycles, zero, sizeof(zero));
            k_fit_stream<Q, D><<<sms, FC::THREADS, FC::SMEM>>>(fa, nf);
            cudaDeviceSynchronize();
            cudaMemcpyFromSymbol(w, g_flr_wait_cycles, sizeof(w));
            cudaMemcpyFromSymbol(tt, g_flr_total_cycles, sizeof(tt));
            cudaMemcpyFromSymbol(it, g_flr_items, sizeof(it));
            double sw = 0, st = 0, mx = 0; int n = 0, hist[8] = {};
            for (int b = 0; b < sms; ++b)
                for (int ww = 0; ww < FC::NSW; ++ww) {
                    const int i = b * 32 + ww;
                    sw += w[i]; st += tt[i]; ++n; if (tt[i] > mx) mx = tt[i]; hist[it[i] < 8 ? it[i] : 7]++;
                }
            printf("   per-warp: mean total %.0f cyc, mean wait %.0f cyc (%.0f%%), max total %.0f; items/warp hist:",
                   st / n, sw / n, 100 * sw / st, mx);
            for (int k = 0; k < 8; ++k) printf(" %d", hist[k]);
            printf("\n");
        }
#endif
    }
    {
        FitLdgArgs la{G, Y, mom, W, H, Bx, mom_pitch(Bx), By, W / kSeg};
        for (int nf : {1, 4}) {
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                k_fit_ldg<Q, D><<<sms, kFitLdgWarps * 32>>>(la, nf);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            printf("fitldg nf=%d warps=%d: %7.1f us/frame  %6.0f GB/s (%s)\n", nf, kFitLdgWarps, 1e3 * ms / nf,
                   plane * (Q + 3) * 4.0 * nf / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    ApplyArgs aa;
    make_tmap_planes(&aa.tg, G, W, H, NF * Q, kSeg, Q);
    aa.models = M, aa.out = O, aa.W = W, aa.H = H, aa.D = D, aa.Bx = Bx, aa.By = By;
    aa.nseg = (W + kSeg - 1) / kSeg, aa.nband = apply_nband(H, D, By), aa.nsub = 1;
    using AC = ApplyCfg<Q>;
    cudaFuncSetAttribute(k_apply_stream<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AC::SMEM);
    for (int nf : {1, 4}) {
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            k_apply_stream<Q><<<sms, AC::THREADS, AC::SMEM>>>(aa, nf);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("apply nf=%d warps=%d S=%d: %7.1f us/frame  %6.0f GB/s (%s)\n", nf, AC::NSW, AC::S, 1e3 * ms / nf,
               plane * (Q + 3) * 4.0 * nf / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
