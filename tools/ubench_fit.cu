// Microbenchmark of the streaming FIT / APPLY kernels on one 1080p Q=8 frame set (no Python).
// Variants are selected at compile time (see tools/ubench_fit.sh).
#include <cstdio>
#include <vector>

#include "../paper_2410_11625_b200/csrc/flr_launch.h"
#include "../paper_2410_11625_b200/csrc/flr_persist.cuh"

using namespace flr;

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
    }
    ApplyArgs aa;
    make_tmap_planes(&aa.tg, G, W, H, NF * Q, kSeg, Q);
    aa.models = M, aa.out = O, aa.W = W, aa.H = H, aa.D = D, aa.Bx = Bx, aa.By = By;
    aa.nseg = (W + kSeg - 1) / kSeg, aa.nband = apply_nband(H, D, By);
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
