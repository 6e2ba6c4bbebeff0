// Standalone timing of the K2 kernels (row-strip blur + row solve) on a synthetic 1080p Q=8
// moment field, with optional per-CTA phase stamps (-DFLR_DBG_PHASES).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_2410_11625_b200/csrc/flr_launch.h"
#include "../paper_2410_11625_b200/csrc/flr_tiles.cuh"
#include "../paper_2410_11625_b200/csrc/flr_k2.cuh"

using namespace flr;
namespace flr {
__device__ long long g_flr_phase[10 * 65536];
}
int main(int argc, char** argv)
{
    constexpr int Q = 8, R = 3, KM = Dims<Q>::KM;
    const int Bx = 240, By = 135, Bxp = mom_pitch(Bx), n = argc > 1 ? atoi(argv[1]) : 1;
    std::vector<double> h((size_t)n * KM * By * Bxp);
    for (size_t i = 0; i < h.size(); ++i) h[i] = 1.0 + 1e-3 * (double)(i % 977);
    for (int f = 0; f < n; ++f)
        for (int y = 0; y < By; ++y)
            for (int x = 0; x < Bxp; ++x) h[((size_t)f * KM * By + y) * Bxp + x] = 64.0;
    double *mom, *hb;
    float* models;
    cudaMalloc(&mom, h.size() * 8);
    cudaMalloc(&hb, h.size() * 8);
    cudaMalloc(&models, (size_t)n * Bx * By * Dims<Q>::MSTRIDE * 4);
    cudaMemcpy(mom, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    Taps t{};
    t.R = R;
    for (int i = -R; i <= R; ++i) t.g[R + i] = std::exp(-(double)(i * i) / (2.0 * 1.25 * 1.25));
    const size_t sb = blur_rows_smem(Bx, R), ss = solve_rows_smem<Q>();
    cudaFuncSetAttribute(k_blur_rows<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    cudaFuncSetAttribute(k_solve_rows<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ss);
    cudaEvent_t e[3];
    for (auto& x : e) cudaEventCreate(&x);
    const dim3 gb(cdiv(By, kRowsCH), n * KM), gs(cdiv(Bx, kSolveRowN), By, n);
    float tb = 0, tsv = 0;
    for (int rep = 0; rep < 3000; ++rep) {  // ~100 ms: let the SM clock ramp up
        k_blur_rows<R><<<gb, kRowsThreads, sb>>>(mom, Bx, Bxp, By, hb, t);
        k_solve_rows<Q><<<gs, kSolveRowN, ss>>>(Bx, Bxp, By, hb, models, 1e-5, 1e-4);
    }
    for (int rep = 0; rep < 20; ++rep) {
        cudaEventRecord(e[0]);
        k_blur_rows<R><<<gb, kRowsThreads, sb>>>(mom, Bx, Bxp, By, hb, t);
        cudaEventRecord(e[1]);
        k_solve_rows<Q><<<gs, kSolveRowN, ss>>>(Bx, Bxp, By, hb, models, 1e-5, 1e-4);
        cudaEventRecord(e[2]);
        cudaEventSynchronize(e[2]);
        cudaEventElapsedTime(&tb, e[0], e[1]);
        cudaEventElapsedTime(&tsv, e[1], e[2]);
    }
    {
        using KG = K2WsGeom<Q, R>;
        cudaFuncSetAttribute(k_blur_solve_tile<Q, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)KG::SMEM);
        const dim3 gt(cdiv(Bx, kK2TX), cdiv(By, kK2TY), n);
        CUtensorMap tmk;
        make_tmap_3d(&tmk, mom, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, Bx, By, Bxp, n * KM, KG::HX, KG::NVB, KG::G);
        float tt = 0;
        for (int rep = 0; rep < 2000; ++rep) {
            if (rep == 1990) cudaEventRecord(e[0]);
            k_blur_solve_tile<Q, R><<<gt, kK2WsThreads, KG::SMEM>>>(tmk, Bx, By, models, Dims<Q>::MSTRIDE, 1e-5, 1e-4, t);
        }
        cudaEventRecord(e[1]);
        cudaEventSynchronize(e[1]);
        cudaEventElapsedTime(&tt, e[0], e[1]);
        printf("n=%d blur_solve_tile %.2f us/frame (back-to-back) (%s)\n", n, 1e3 * tt / 10 / n,
               cudaGetErrorString(cudaGetLastError()));
#ifdef FLR_DBG_PHASES
        std::vector<long long> ph(64);
        cudaMemcpyFromSymbol(ph.data(), g_flr_phase, 64 * 8);
        printf("  tile phases (cycles):");
        for (int i = 0; i < ph[63]; ++i) printf(" %lld", ph[i]);
        printf("\n");
        {
            const int nc = gt.x * gt.y * gt.z;
            std::vector<long long> g(1000 + 4 * nc);
            cudaMemcpyFromSymbol(g.data(), g_flr_phase, g.size() * 8);
            long long e0 = g[1000], e1 = g[1000], x0 = g[1001], x1 = g[1001];
            double cyc = 0;
            for (int c = 0; c < nc; ++c) {
                e0 = std::min(e0, g[1000 + 4 * c]), e1 = std::max(e1, g[1000 + 4 * c]);
                x0 = std::min(x0, g[1001 + 4 * c]), x1 = std::max(x1, g[1001 + 4 * c]);
                cyc += g[1002 + 4 * c];
            }
            printf("  CTA entry spread %.2f us, exits %.2f..%.2f us after first entry, mean in-CTA cycles %.0f\n",
                   (e1 - e0) * 1e-3, (x0 - e0) * 1e-3, (x1 - e0) * 1e-3, cyc / nc);
        }
#endif
    }
    printf("n=%d blur_rows %.2f us/frame  solve_rows %.2f us/frame (%s)\n", n, 1e3 * tb / n, 1e3 * tsv / n,
           cudaGetErrorString(cudaGetLastError()));
#ifdef FLR_DBG_PHASES
    const int nc = gb.x * gb.y;
    std::vector<long long> ph((size_t)10 * nc);
    cudaMemcpyFromSymbol(ph.data(), g_flr_phase, ph.size() * 8);
    double acc[5] = {}, dur = 0;
    long long smin = ph[8], emax = ph[7], emin = ph[7], smax = ph[8];
    for (int c = 0; c < nc; ++c) {
        const long long* q = &ph[10 * c];
        for (int k = 0; k < 5; ++k) acc[k] += q[k + 1] - q[k];
        smin = std::min(smin, q[8]), smax = std::max(smax, q[8]);
        emin = std::min(emin, q[7]), emax = std::max(emax, q[7]);
        dur += q[7] - q[8];
    }
    printf("blur_rows per-CTA cycles: load+v %.0f  sync %.0f  h %.0f  sync %.0f  store %.0f\n", acc[0] / nc,
           acc[1] / nc, acc[2] / nc, acc[3] / nc, acc[4] / nc);
    printf("  CTA start spread %.2f us, first end %.2f us, last end %.2f us, mean CTA %.2f us, clock %.0f MHz\n",
           (smax - smin) * 1e-3, (emin - smin) * 1e-3, (emax - smin) * 1e-3, dur / nc * 1e-3,
           (acc[0] + acc[1] + acc[2] + acc[3] + acc[4]) / dur * 1e3 / 1e3);
#endif
    return 0;
}
