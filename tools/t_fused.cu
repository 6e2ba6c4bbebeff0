// standalone timing of the fused kernel on synthetic 1080p Q=8 frames (no Python)
#include <cstdio>
#include <vector>
#include "../paper_2410_11625_b200/csrc/flr_launch.h"
#include "../paper_2410_11625_b200/csrc/flr_fused.cuh"
using namespace flr;
int main(int argc, char** argv)
{
    constexpr int Q = 8, D = 8, R = 3;
    const int W = 1920, H = 1080, NF = 4, Bx = W / D, By = (H + D - 1) / D, Bxp = mom_pitch(Bx);
    const int lag = argc > 1 ? atoi(argv[1]) : 40;
    const size_t plane = (size_t)W * H;
    float *G, *Y, *M, *O;
    double* mom;
    int* flags;
    cudaMalloc(&G, plane * Q * NF * 4);
    cudaMalloc(&Y, plane * 3 * NF * 4);
    cudaMalloc(&O, plane * 3 * NF * 4);
    cudaMalloc(&M, (size_t)Bx * By * NF * Dims<Q>::MSTRIDE * 4);
    cudaMalloc(&mom, (size_t)Bxp * By * NF * Dims<Q>::KM * 8);
    cudaMalloc(&flags, 4 * NF * (By + By));
    std::vector<float> h(plane * Q * NF);
    for (size_t i = 0; i < h.size(); ++i) h[i] = 0.2f + (float)((i * 2654435761u) % 1000) * 6e-4f;
    cudaMemcpy(G, h.data(), plane * Q * NF * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(Y, h.data(), plane * 3 * NF * 4, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int nf : {1, 4}) {
        FusedArgs a;
        memset(&a, 0, sizeof(a));
        make_tmap_planes(&a.fit.tg, G, W, H, nf * Q, kSeg, Q);
        make_tmap_planes(&a.fit.ty, Y, W, H, nf * 3, kSeg, 3);
        make_tmap_planes(&a.app.tg, G, W, H, nf * Q, kSeg, Q);
        make_tmap_3d(&a.tmom, mom, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, Bx, By, Bxp, nf * Dims<Q>::KM, halo_x(R),
                     kTileTY + 2 * R, kFusedG);
        a.fit.mom = mom, a.fit.W = W, a.fit.H = H, a.fit.Bx = Bx, a.fit.Bxp = Bxp, a.fit.By = By, a.fit.nseg = W / kSeg;
        a.app.models = M, a.app.out = O, a.app.W = W, a.app.H = H, a.app.D = D, a.app.Bx = Bx, a.app.By = By;
        a.app.nseg = W / kSeg, a.app.nband = apply_nband(H, D, By), a.app.nsub = 1;
        a.taps.R = R;
        for (int i = -R; i <= R; ++i) a.taps.g[R + i] = 1.0;
        a.nrt = (By + 3) / 4, a.ncx = (Bx + 31) / 32, a.fit_done = flags, a.solve_done = flags + nf * By, a.n = nf;
        a.lag = lag, a.eps_add = 1e-5, a.eps_mul = 1e-4;
        using C = FusedCfg<Q, R>;
        cudaFuncSetAttribute(k_flr_fused<Q, D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float ms = 0;
        for (int rep = 0; rep < 4; ++rep) {
            cudaMemset(flags, 0, 4 * nf * 2 * By);
            cudaEventRecord(e0);
            void* args[] = {&a};
            cudaLaunchCooperativeKernel((void*)k_flr_fused<Q, D, R>, sms, kFusedThreads, args, C::SMEM);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("fused lag=%d nf=%d: %.1f us/frame (%s)\n", lag, nf, 1e3 * ms / nf, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
