// Per-SM streaming rate of the warp-specialised fit and apply kernels: 8 distinct 1080p Q=8
// frames (730 MB of inputs, > L2) processed with the grid restricted to G CTAs (one per SM),
// G = 148 ... 37.  If the kernels are HBM-bound, time stays flat as G shrinks until the
// per-SM rate limit is reached; the knee gives the rate one SM can stream at.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -lcuda tools/t_rate.cu -o tools/t_rate
#include <cstdio>
#ifndef T_NSUB
#define T_NSUB 2  // APPLY sub-bands per block row (the library: 2 at D = 8)
#endif
#include "../paper_2410_11625_b200/csrc/flr_launch.h"
#include "../paper_2410_11625_b200/csrc/flr_fitws.cuh"
#include "../paper_2410_11625_b200/csrc/flr_applyws.cuh"
namespace flr {
// K1 with self-feeding consumer warps (experiment): no producer warp; lane 0
// of each of kFitSelfW warps issues its own 2-row stages, the next one into the slot it has
// just read, so a stage's round trip is the TMA latency alone.
#ifndef FLR_FITSELF_W
#define FLR_FITSELF_W 8
#endif
#ifndef FLR_FITSELF_S
#define FLR_FITSELF_S 2
#endif
constexpr int kFitSelfW = FLR_FITSELF_W, kFitSelfS = FLR_FITSELF_S;
template <int Q>
struct FitSelfCfg {
    using FC = FitWsCfg<Q>;
    static constexpr int STG = FC::STG, S = kFitSelfS, NW = kFitSelfW, THREADS = NW * 32;
    static constexpr size_t BAR_OFF = (size_t)NW * S * STG * sizeof(float);
    static constexpr size_t SMEM = BAR_OFF + NW * S * sizeof(uint64_t);
    static_assert(SMEM <= 232448, "self-feeding fit exceeds 227 KB of shared memory");
};
template <int Q, int D>
__global__ void __launch_bounds__(FitSelfCfg<Q>::THREADS, 1) k_fit_self(const __grid_constant__ FitArgs a, int n)
{
    using C = FitSelfCfg<Q>;
    using FC = FitWsCfg<Q>;
    constexpr int S = C::S, STG = C::STG, NW = C::NW, RB = FC::RB;
    static_assert(FC::S == S || true, "");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* ring = reinterpret_cast<float*>(smem_raw) + (size_t)w * S * STG;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + C::BAR_OFF) + w * S;
    if (lane == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    const int per_frame = a.By * a.nseg, nitems = n * per_frame, GW = gridDim.x * NW;
    const uint64_t pg = policy_evict_first(), py = policy_evict_first();
    int pit = blockIdx.x * NW + w, prow = 0, prows = 0, pf = 0, pby = 0, psg = 0;  // issue cursor (lane 0)
    auto decode = [&]() {
        if (pit >= nitems) return;
        pf = pit / per_frame;
        const int rem = pit - pf * per_frame;
        pby = rem / a.nseg;
        psg = rem - pby * a.nseg;
        prows = min(D, a.H - pby * D);
    };
    auto issue = [&](int slot) {
        if (pit >= nitems) return;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        fit_issue_row<Q, D, false, false, kFS, RB>(a, pf, pby, psg, prow, ring + slot * STG, &full[slot], pg, py);
        if ((prow += RB) >= prows) {
            prow = 0;
            pit += GW;
            decode();
        }
    };
    if (lane == 0) {
        decode();
        for (int s = 0; s < S; ++s) issue(s);
    }
    __syncwarp();
    int k = 0;
    bool waited = true;
    for (int it = blockIdx.x * NW + w; it < nitems; it += GW)
        fit_consume_item_rel<Q, D, false, false, false>(a, it, per_frame, ring, full, issue, k, lane, waited);
}

}  // namespace flr
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
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    using FC = FitWsCfg<Q>;
    using AC = ApplyWsCfg<Q>;
    cudaFuncSetAttribute(k_fit_ws<Q, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FC::SMEM);
    cudaFuncSetAttribute(k_apply_ws<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AC::SMEM);
    const int nf = NF;
    FitArgs fa{};
    make_tmap_planes(&fa.tg, G, W, H, nf * Q, kFS, Q, FitWsCfg<Q>::RB);
    make_tmap_planes(&fa.ty, Y, W, H, nf * 3, kFS, 3, FitWsCfg<Q>::RB);
    fa.keep_y0 = H, fa.mom = mom, fa.W = W, fa.H = H, fa.Bx = Bx, fa.Bxp = mom_pitch(Bx), fa.By = By, fa.nseg = W / kFS;
    ApplyArgs aa{};
    make_tmap_planes(&aa.tg, G, W, H, nf * Q, kSeg, Q, ApplyWsCfg<Q>::RB);
    aa.models = M, aa.out = O, aa.W = W, aa.H = H, aa.D = D, aa.Bx = Bx, aa.By = By;
    aa.nseg = W / kSeg, aa.nband = apply_nband(H, D, By), aa.nsub = T_NSUB;
    const double fit_bytes = (double)plane * (Q + 3) * 4 * nf, app_bytes = (double)plane * (Q + 3) * 4 * nf;
    for (int g : {148, 136, 120, 104, 88, 74, 60, 48, 37}) {
        float ms = 0;
        const int reps = 30;
        for (int k = 0; k < 2; ++k) {
            cudaEventRecord(e0);
            for (int r = 0; r < reps; ++r) k_fit_ws<Q, D><<<g, FC::THREADS, FC::SMEM>>>(fa, nf);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        const double tf = 1e-3 * ms / reps;
        double tself = 0;
#ifndef FLR_FITWS_NOWAIT  // (self-fed warps would exit with stages in flight)
        {
            using SC = FitSelfCfg<Q>;
            static bool once = false;
            if (!once) cudaFuncSetAttribute(k_fit_self<Q, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SC::SMEM), once = true;
            for (int k = 0; k < 2; ++k) {
                cudaEventRecord(e0);
                for (int r = 0; r < reps; ++r) k_fit_self<Q, D><<<g, SC::THREADS, SC::SMEM>>>(fa, nf);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            tself = 1e-3 * ms / reps;
        }
#endif
        for (int k = 0; k < 2; ++k) {
            cudaEventRecord(e0);
            for (int r = 0; r < reps; ++r) k_apply_ws<Q><<<g, AC::THREADS, AC::SMEM>>>(aa, nf);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        const double ta = 1e-3 * ms / reps;
        printf("G=%3d  fit %7.2f us/frame %6.0f GB/s (%5.1f GB/s/SM)  self-fed fit %7.2f us/frame (%5.1f GB/s/SM)   apply %7.2f us/frame %6.0f GB/s (%5.1f GB/s/SM)  %s\n",
               g, 1e6 * tf / nf, fit_bytes / tf / 1e9, fit_bytes / tf / 1e9 / g, 1e6 * tself / nf, fit_bytes / tself / 1e9 / g,
               1e6 * ta / nf, app_bytes / ta / 1e9,
               app_bytes / ta / 1e9 / g, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
