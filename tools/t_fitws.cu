// Standalone timing of the warp-specialised fit and apply kernels on synthetic 1080p Q=8
// frames (back-to-back launches after a clock warm-up).  Variants via -D macros.
#include <cstdio>
#include <vector>
#include "../paper_2410_11625_b200/csrc/flr_launch.h"
#include "../paper_2410_11625_b200/csrc/flr_fitws.cuh"
#include "../paper_2410_11625_b200/csrc/flr_applyws.cuh"
using namespace flr;
int main()
{
    constexpr int Q = 8, D = 8;
    const int W = 1920, H = 1080, NF = 8, Bx = W / D, By = (H + D - 1) / D;
    const size_t plane = (size_t)W * H;
    float *G, *Y, *M, *O;
    double* mom;
    cudaMalloc(&G, plane * Q * NF * 4);
    cudaMalloc(&Y, plane * 3 * NF * 4);
    cudaMalloc(&O, plane * 3 * NF * 4);
    cudaMalloc(&M, (size_t)Bx * By * NF * Dims<Q>::MSTRIDE * 4);
    cudaMalloc(&mom, (size_t)mom_pitch(Bx) * By * NF * Dims<Q>::KM * 8);
    cudaMemset(G, 0, plane * Q * NF * 4);
    cudaMemset(Y, 0, plane * 3 * NF * 4);
    cudaMemset(M, 0, (size_t)Bx * By * NF * Dims<Q>::MSTRIDE * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    using FC = FitWsCfg<Q>;
    using AC = ApplyWsCfg<Q>;
    cudaFuncSetAttribute(k_fit_ws<Q, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FC::SMEM);
    cudaFuncSetAttribute(k_apply_ws<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AC::SMEM);
    for (int nf : {1, 8}) {
        FitArgs fa{};
        make_tmap_planes(&fa.tg, G, W, H, nf * Q, kSeg, Q);
        make_tmap_planes(&fa.ty, Y, W, H, nf * 3, kSeg, 3);
        fa.keep_y0 = H, fa.mom = mom, fa.W = W, fa.H = H, fa.Bx = Bx, fa.Bxp = mom_pitch(Bx), fa.By = By, fa.nseg = W / kSeg;
        ApplyArgs aa{};
        make_tmap_planes(&aa.tg, G, W, H, nf * Q, kSeg, Q);
        aa.models = M, aa.out = O, aa.W = W, aa.H = H, aa.D = D, aa.Bx = Bx, aa.By = By;
        aa.nseg = W / kSeg, aa.nband = apply_nband(H, D, By), aa.nsub = 2;
        const int gf = min(sms, (nf * By * fa.nseg + FC::NC - 1) / FC::NC);
        const int ga = min(sms, (nf * aa.nband * 2 * aa.nseg + AC::NC - 1) / AC::NC);
        float ms = 0;
        const int reps = nf == 1 ? 2000 : 300;
        for (int k = 0; k < 2; ++k) {
            cudaEventRecord(e0);
            for (int r = 0; r < reps; ++r) k_fit_ws<Q, D><<<gf, FC::THREADS, FC::SMEM>>>(fa, nf);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("fit_ws   nf=%d S=%d: %6.2f us/frame (%s)\n", nf, FC::S, 1e3 * ms / reps / nf,
               cudaGetErrorString(cudaGetLastError()));
        for (int k = 0; k < 2; ++k) {
            cudaEventRecord(e0);
            for (int r = 0; r < reps; ++r) k_apply_ws<Q><<<ga, AC::THREADS, AC::SMEM>>>(aa, nf);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("apply_ws nf=%d S=%d: %6.2f us/frame (%s)\n", nf, AC::S, 1e3 * ms / reps / nf,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
