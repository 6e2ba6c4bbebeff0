// flr_k2.cuh -- K2 as one tile kernel: separable Gaussian of the moment field (P:334,
// R1-R3) and the appendix's normalised, regularised per-block solve, for a
// 32 x 8 tile of blocks per CTA (one thread per block in the solve).
//
// The moment field is read ONCE per tile from L2 (plus the R-block halo): every byte
// moved between L2 and the SM costs about as much as an HBM byte on B200 (measured
// ~32 B/clk/SM each way), so K2 avoids any blurred-field round trip through global
// memory.  Per group of G components:
//   TMA     one 3-D box {HX columns, TY + 2R rows, G planes} per group into a 3-stage
//           ring (issued 3 groups ahead; out-of-field rows/columns arrive as zeros = R3);
//   v-pass  one thread per (component, halo column): TY + 2R values -> TY outputs -> vb;
//   h-pass  one thread per (component, row, 8 consecutive columns): 8 + 2RE values
//           (16-byte shared loads, bank-padded layout) -> 8 outputs -> stage;
//   gather  thread (tx, ty) moves its G values of the group from stage to registers.
// All fp64 (the cancellation in S/n - mu mu^T needs it); DP throughput (~64 FMA/clk/SM)
// then bounds the kernel: ~1.1k DP ops of blur + ~0.7k of solve per block.
#pragma once
#include "flr_common.cuh"
#include "flr_pipe.cuh"
#include "flr_solve.cuh"

namespace flr {

#ifndef FLR_K2_TY
#define FLR_K2_TY 8
#endif
constexpr int kK2TX = 32, kK2TY = FLR_K2_TY, kK2Threads = kK2TX * kK2TY;
constexpr int kK2MinBlocks = kK2TY <= 4 ? 2 : 1;  // CTAs per SM the register budget allows

template <int Q, int R>
struct K2Geom {
    static constexpr int RE = (R + 1) & ~1;     // x halo, even: 16-byte aligned pairs in vb
    static constexpr int HX = kK2TX + 2 * RE;   // halo columns
    static constexpr int NV = kK2TY + 2 * R;    // values per v-pass column task
    static constexpr int VT = R <= 5 ? 2 : 1;   // v-pass column tasks per thread
    static constexpr int G = VT * kK2Threads / HX;  // components per group
    static constexpr int NG = (Dims<Q>::KM + G - 1) / G;
    static constexpr int CWH = G * kK2TY * (kK2TX / 8) <= kK2Threads ? 8 : 16;  // h-pass outputs per task
    static constexpr int NCH = kK2TX / CWH;     // h-pass chunks per row
    static constexpr int S = VT == 2 ? 2 : 3;   // TMA ring stages
    // vb: [G][TY][VP], halo column u at u + 2 (u / 8); stage: [G][TY][SP], column x at
    // x + 2 (x / 8).  Pitches = 8 (mod 16) doubles: the h-pass's 16-byte accesses of the
    // 8 lanes of a quarter warp then fall on distinct bank groups.
    static constexpr int VPMIN = HX + 2 * ((HX - 1) / 8);
    static constexpr int VP = ((VPMIN - 8 + 15) / 16) * 16 + 8;
    static constexpr int SP = 40;
    static constexpr size_t BOXD = (size_t)G * NV * HX;    // doubles per TMA box
    static constexpr size_t BOX = (BOXD + 15) / 16 * 16;  // stage pitch: TMA needs 128-byte aligned smem
    static constexpr size_t VB = (size_t)G * kK2TY * VP;
    static constexpr size_t ST = (size_t)G * kK2TY * SP;
    static constexpr size_t MODB = (size_t)kK2Threads * Dims<Q>::MSTRIDE * sizeof(float);
    static constexpr size_t DATA = (S * BOX + VB + ST) * sizeof(double);
    static constexpr size_t BAR_OFF = (DATA > MODB ? DATA : MODB);
    static constexpr size_t SMEM = BAR_OFF + S * sizeof(uint64_t);
    static_assert(G >= 1 && G * kK2TY * NCH <= kK2Threads && G <= 256, "tile geometry");
    static_assert(SMEM <= 232448, "K2 tile exceeds 227 KB of shared memory");
};

// One TX x TY tile of output blocks (frame f, first block (bx0, by0)), run by the kK2Threads
// threads of the CTA (tid = threadIdx.x).  smk: KG::BAR_OFF bytes of shared memory, bar: S
// mbarriers, initialised here (every earlier use of them must have completed).
// tm: the fp64 moment field [n*KM][By][Bxp] with box {HX, TY + 2R, G} (K2Geom).
template <int Q, int R>
__device__ __forceinline__ void k2_tile(const CUtensorMap* tmp, int f, int bx0, int by0, int Bx, int By,
                                        float* __restrict__ models, int mstride, double eps_add, double eps_mul,
                                        const Taps& t, double* smk, uint64_t* bar, uint64_t kpol)
{
    using Dm = Dims<Q>;
    using KG = K2Geom<Q, R>;
    constexpr int KM = Dm::KM, G = KG::G, NG = KG::NG, HX = KG::HX, NV = KG::NV, RE = KG::RE, S = KG::S, VT = KG::VT;
    constexpr int TX = kK2TX, TY = kK2TY, VP = KG::VP, SP = KG::SP, NCH = KG::NCH, MS = Dm::MSTRIDE;
    double* ring = smk;
    double* vb = smk + S * KG::BOX;
    double* st = vb + KG::VB;
    const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
    const CUtensorMap& tm = *tmp;
    auto issue = [&](int grp) {
        uint64_t* b = &bar[grp % S];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the stage before
        mbar_arrive_expect_tx(b, KG::BOXD * sizeof(double));
        tma_load_3d(ring + (grp % S) * KG::BOX, &tm, bx0 - RE, by0 - R, f * KM + grp * G, b, kpol);
    };
    if (tid == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int g = 0; g < S && g < NG; ++g) issue(g);
#ifdef FLR_DBG_PHASES
    long long tsg[NG + 3];
    tsg[0] = clock64();
#endif
    double blur[KM];
#pragma unroll
    for (int grp = 0; grp < NG; ++grp) {
#ifdef FLR_DBG_PHASES
        tsg[grp + 1] = clock64();
#endif
        mbar_wait(&bar[grp % S], (grp / S) & 1);
        {  // v-pass, one column task at a time (keeps the live set to NV values besides blur[])
            const double* box = ring + (grp % S) * KG::BOX;
#pragma unroll
            for (int q = 0; q < VT; ++q) {
                const int task = tid + q * kK2Threads, gv = task / HX, u = task - gv * HX;
                if (gv < G) {
                    double v[NV];
#pragma unroll
                    for (int i = 0; i < NV; ++i) v[i] = box[(gv * NV + i) * HX + u];
                    double* o = vb + gv * TY * VP + u + 2 * (u / 8);
#pragma unroll
                    for (int r = 0; r < TY; ++r) {
                        double a = t.g[R] * v[r + R];
#pragma unroll
                        for (int d = 1; d <= R; ++d) a = fma(t.g[R + d], v[r + R - d] + v[r + R + d], a);
                        o[r * VP] = a;
                    }
                }
            }
        }
        __syncthreads();  // vb complete, stage grp % S consumed (and the previous gather done)
        if (tid == 0 && grp + S < NG) issue(grp + S);
        if (tid < G * TY * NCH) {
            constexpr int CW = KG::CWH, NW = CW + 2 * RE;
            const int c = tid % NCH, r = (tid / NCH) % TY, g = tid / (NCH * TY);
            // u = CW c + i lives at CW c + i + 2 ((CW c + i) / 8) = (CW + CW / 4) c + i + 2 (i / 8)
            const double* h = vb + (g * TY + r) * VP + c * (CW + CW / 4);
            double w[NW];
#pragma unroll
            for (int i = 0; i < NW; i += 2) {
                const double2 q = *reinterpret_cast<const double2*>(h + i + 2 * (i / 8));
                w[i] = q.x;
                w[i + 1] = q.y;
            }
            double* o = st + (g * TY + r) * SP + c * (CW + CW / 4);
#pragma unroll
            for (int e = 0; e < CW; e += 2) {
                double a = t.g[R] * w[e + RE], b = t.g[R] * w[e + 1 + RE];
#pragma unroll
                for (int d = 1; d <= R; ++d) {
                    a = fma(t.g[R + d], w[e + RE - d] + w[e + RE + d], a);
                    b = fma(t.g[R + d], w[e + 1 + RE - d] + w[e + 1 + RE + d], b);
                }
                *reinterpret_cast<double2*>(o + e + 2 * (e / 8)) = make_double2(a, b);
            }
        }
        __syncthreads();  // stage complete (and vb free for the next v-pass)
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int k = grp * G + g;
            if (k < KM) blur[k] = st[(g * TY + ty) * SP + tx + 2 * (tx / 8)];
        }
    }
    __syncthreads();  // every gather done: smem now stages the models
#ifdef FLR_DBG_PHASES
    tsg[NG + 1] = clock64();
#endif
    float* mstage = reinterpret_cast<float*>(smk);
    const int bx = bx0 + tx, by = by0 + ty;
    if (bx < Bx && by < By) {
        solve_block<Q>([&](int k) { return blur[k]; }, eps_add, eps_mul, mstage + tid * MS);
#pragma unroll
        for (int i = 3 * (Q + 1); i < MS; ++i) mstage[tid * MS + i] = 0.0f;
    }
    __syncthreads();
#ifdef FLR_DBG_PHASES
    tsg[NG + 2] = clock64();
    if (tid == 0 && blockIdx.x == 2 && blockIdx.y == 2 && blockIdx.z == 0) {
        extern __device__ long long g_flr_phase[];
        for (int i = 0; i < NG + 3; ++i) g_flr_phase[i] = tsg[i] - tsg[0];
        g_flr_phase[63] = NG + 3;
    }
#endif
    const int nbx = min(TX, Bx - bx0), nrow = min(TY, By - by0);
    static_assert(MS % 4 == 0, "padded models are whole float4s");
    if (mstride == MS && (reinterpret_cast<uintptr_t>(models) & 15) == 0) {  // rows: contiguous aligned runs
        const int q = nbx * (MS / 4);
        for (int i = tid; i < nrow * q; i += kK2Threads) {
            const int r = i / q, j = i - r * q;
            reinterpret_cast<float4*>(models + ((size_t)(f * By + by0 + r) * Bx + bx0) * MS)[j] =
                reinterpret_cast<const float4*>(mstage + r * TX * MS)[j];
        }
    } else {  // the ABI's packed [Q+1][3] models (flr_fit): runs of nbx * mstride floats, 4-byte aligned
        const int q = nbx * mstride;
        for (int i = tid; i < nrow * q; i += kK2Threads) {
            const int r = i / q, j = i - r * q, b = j / mstride;
            models[((size_t)(f * By + by0 + r) * Bx + bx0) * mstride + j] = mstage[(r * TX + b) * MS + j - b * mstride];
        }
    }
}

template <int Q, int R>
__global__ void __launch_bounds__(kK2Threads, kK2MinBlocks)
    k_blur_solve_tile(const __grid_constant__ CUtensorMap tm, int Bx, int By, float* __restrict__ models,
                      int mstride, double eps_add, double eps_mul, const __grid_constant__ Taps t)
{
    using KG = K2Geom<Q, R>;
    extern __shared__ __align__(1024) double smk[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(smk) + KG::BAR_OFF);
    if (threadIdx.x == 0) FLR_TL(1, 0);
    pdl_wait();  // the moment field comes from the previous grid
    pdl_trigger();  // dependents launch only once we are past our own wait
    if (threadIdx.x == 0) FLR_TL(1, 1);
    k2_tile<Q, R>(&tm, blockIdx.z, blockIdx.x * kK2TX, blockIdx.y * kK2TY, Bx, By, models, mstride, eps_add, eps_mul, t,
                  smk, bar, policy_evict_normal());
    if (threadIdx.x == 0) FLR_TL(1, 2);
}

}  // namespace flr
