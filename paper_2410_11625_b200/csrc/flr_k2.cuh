// flr_k2.cuh -- K2 as one tile kernel: separable Gaussian of the moment field (P:334,
// R1-R3) and the appendix's normalised, regularised per-block solve, for a
// 32 x 8 tile of blocks per CTA (one thread per block in the solve).
//
// The moment field is read ONCE per tile from L2 (plus the R-block halo): every byte
// moved between L2 and the SM costs about as much as an HBM byte on B200, so K2 avoids any
// blurred-field round trip through global memory.  Per group of G components:
//   TMA     one 3-D box {HX columns, TY + 2R rows, G planes} per group into a 2-3-stage
//           ring (issued S groups ahead; out-of-field rows/columns arrive as zeros = R3);
//   v-pass  one thread per (component, halo column): TY + 2R values -> TY outputs -> vb;
//   h-pass  one thread per (component, row, CWH consecutive columns): CWH + 2RE values
//           (16-byte shared loads, bank-padded layout) -> CWH outputs -> stage;
//   gather  thread (tx, ty) moves its G values of the group from stage to registers.
// All fp64 (the cancellation in S/n - mu mu^T needs it).
//
// k_blur_solve_tile (the staged schedule) is warp-specialised: BLUR warps run TMA, v-pass
// and h-pass group after group into a 2-deep stage ring while the 8 SOLVE warps (one
// thread per block) gather each group as it lands and factor the system as soon as its
// components (n, u, S, Y: the first C_XY) are in -- under the blur of the cross moments --
// so the blur, bound by shared-memory bandwidth (~75 B per block-component), overlaps the
// fp64 solve instead of alternating with it.  k2_tile (used by the one-kernel wave schedule,
// whose CTAs have 8 warps) runs the same passes with every warp in lock step.
#pragma once
#include "flr_common.cuh"
#include "flr_pipe.cuh"
#include "flr_solve.cuh"

namespace flr {

#ifndef FLR_K2_TY
#define FLR_K2_TY 8
#endif
#ifndef FLR_K2_BLUR_WARPS
#define FLR_K2_BLUR_WARPS 4
#endif
constexpr int kK2TX = 32, kK2TY = FLR_K2_TY, kK2Threads = kK2TX * kK2TY;
constexpr int kK2BlurThreads = 32 * FLR_K2_BLUR_WARPS, kK2WsThreads = kK2Threads + kK2BlurThreads;

// WS: the geometry of the warp-specialised kernel (k_blur_solve_tile): NST = 2 stages
// between the blur and the solve warps, G reduced until everything fits in 227 KB, and
// 8-column h-pass tasks (bank-conflict free; the 128 blur threads have tasks to spare).
// model staging stride in shared memory: MSTRIDE + 1 floats (odd: the solve threads' stores
// of one model component fall on 32 distinct banks)
template <int Q>
constexpr int k2_msp = Dims<Q>::MSTRIDE + 1;
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

template <int Q, int R, bool WS = false>
struct K2Geom {
    static constexpr int RE = (R + 1) & ~1;     // x halo, even: 16-byte aligned pairs in vb
    static constexpr int HX = kK2TX + 2 * RE;   // halo columns
    static constexpr int NV = kK2TY + 2 * R;    // values per v-pass column task
    // TMA box rows: NV + 1 where that makes the box's plane pitch HX * NVB = HX (mod 16
    // doubles): a half warp of v-pass lanes crossing from one plane's last columns into the
    // next plane's first then still hits 16 distinct 8-byte bank pairs (R = 3, 4)
    static constexpr int NVB = (HX * (NV - 1)) % 16 != 0 && (HX * NV) % 16 == 0 ? NV + 1 : NV;
    static constexpr int VT = R <= 5 ? 2 : 1;   // v-pass column tasks per thread (256 threads)
    static constexpr int S = VT == 2 ? 2 : 3;   // TMA ring stages
    static constexpr int NST = WS ? 2 : 1;      // blur -> solve stages
    // vb: [G] planes of pitch PV, row r at r VP, halo column u at u; stage: [G][TY][SP].
    // Shared-memory bank rules (8-byte accesses: 16 lanes per wavefront; 16-byte: 8):
    //  * row pitches VP, SP = 2 (mod 4) doubles: the h-pass's quarter warps (8 rows of one
    //    column chunk) then read vb and write the stage on 8 distinct 16-byte bank groups;
    //  * rows hold their columns contiguously: the v-pass stores and the gather (consecutive
    //    columns per lane) are conflict free;
    //  * plane pitch PV = HX (mod 16): v-pass half warps crossing planes stay conflict free.
    static constexpr int VP = (HX + 1) / 4 * 4 + 2;
    static constexpr int PV = kK2TY * VP + ((HX - kK2TY * VP) % 16 + 16) % 16;
    static constexpr int SP = 34;
    static constexpr int G0 = VT * kK2Threads / HX;
    static constexpr int PER_G = S * NVB * HX + PV + NST * kK2TY * SP;  // doubles per component
    static constexpr int GFIT = (232448 - 64 - 16 * 8 * S) / (8 * PER_G);
    static constexpr int G = WS && GFIT < G0 ? GFIT : G0;  // components per group
    static constexpr int NG = (Dims<Q>::KM + G - 1) / G;
#ifndef FLR_K2_WS_CWH
#define FLR_K2_WS_CWH 8
#endif
    static constexpr int CWH = WS ? FLR_K2_WS_CWH : G * kK2TY * (kK2TX / 8) <= kK2Threads ? 8 : 16;  // h-pass outputs per task
    static constexpr int NCH = kK2TX / CWH;     // h-pass chunks per row
    static constexpr size_t BOXD = (size_t)G * NVB * HX;   // doubles per TMA box
    static constexpr size_t BOX = (BOXD + 15) / 16 * 16;  // stage pitch: TMA needs 128-byte aligned smem
    static constexpr size_t VB = (size_t)G * PV;
    static constexpr size_t ST = (size_t)G * kK2TY * SP;
    static constexpr int MSP = k2_msp<Q>;
    static constexpr size_t MODB = (size_t)kK2Threads * MSP * sizeof(float);
    static constexpr size_t RING = S * BOX;  // doubles
    static constexpr size_t DATA = (RING + VB + NST * ST) * sizeof(double);
    // k2_tile stages the models over everything; the warp-specialised kernel in the ring
    static constexpr size_t BAR_OFF = WS ? DATA : (DATA > MODB ? DATA : MODB);
    static constexpr size_t SMEM = BAR_OFF + (S + 2 * NST) * sizeof(uint64_t);
    // the solve warps factor once group KF (holding component C_XY - 1) is in
    static constexpr int KF = (Dims<Q>::C_XY - 1) / G;
    static_assert(G >= 1 && G <= 256 && (WS || G * kK2TY * NCH <= kK2Threads), "tile geometry");
    static_assert(!WS || MODB <= RING * sizeof(double), "models stage in the TMA ring");
    static_assert(SMEM <= 232448, "K2 tile exceeds 227 KB of shared memory");
};
template <int Q, int R>
using K2WsGeom = K2Geom<Q, R, true>;

// v-pass of one group (thread i0 of NT): per (component, halo column) task, TY + 2R values
// of the TMA box -> TY outputs in vb.
template <class KG, int R, int NT>
__device__ __forceinline__ void k2_vpass(const double* __restrict__ box, double* __restrict__ vb, const Taps& t, int i0)
{
    constexpr int G = KG::G, HX = KG::HX, NV = KG::NV, NVB = KG::NVB, TY = kK2TY, VP = KG::VP, PV = KG::PV;
    constexpr int NQ = (G * HX + NT - 1) / NT;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {  // one column task at a time (keeps the live set to NV values)
        const int task = i0 + q * NT, gv = task / HX, u = task - gv * HX;
        if (gv < G) {
            double v[NV];
#pragma unroll
            for (int i = 0; i < NV; ++i) v[i] = box[(gv * NVB + i) * HX + u];
            double* o = vb + gv * PV + u;
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

// h-pass of one group (thread i0 of NT): per (component, row, CWH consecutive columns)
// task, CWH + 2RE values of vb (16-byte shared loads, bank-padded layout) -> stage st.
template <class KG, int R, int NT>
__device__ __forceinline__ void k2_hpass(const double* __restrict__ vb, double* __restrict__ st, const Taps& t, int i0)
{
    constexpr int G = KG::G, RE = KG::RE, TY = kK2TY, VP = KG::VP, PV = KG::PV, SP = KG::SP, NCH = KG::NCH;
    constexpr int CW = KG::CWH, NW = CW + 2 * RE, NTASK = G * TY * NCH, NQ = (NTASK + NT - 1) / NT;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int task = i0 + q * NT;
        if (task < NTASK) {
            const int r = task % TY, c = (task / TY) % NCH, g = task / (NCH * TY);  // rows fastest
            const double* h = vb + g * PV + r * VP + c * CW;
            double w[NW];
#pragma unroll
            for (int i = 0; i < NW; i += 2) {
                const double2 qq = *reinterpret_cast<const double2*>(h + i);
                w[i] = qq.x;
                w[i + 1] = qq.y;
            }
            double* o = st + (g * TY + r) * SP + c * CW;
#pragma unroll
            for (int e = 0; e < CW; e += 2) {
                double x0 = t.g[R] * w[e + RE], x1 = t.g[R] * w[e + 1 + RE];
#pragma unroll
                for (int d = 1; d <= R; ++d) {
                    x0 = fma(t.g[R + d], w[e + RE - d] + w[e + RE + d], x0);
                    x1 = fma(t.g[R + d], w[e + 1 + RE - d] + w[e + 1 + RE + d], x1);
                }
                *reinterpret_cast<double2*>(o + e) = make_double2(x0, x1);
            }
        }
    }
}

// thread (tx, ty)'s G values of group GRP: stage -> registers blur[GRP G ...]
template <int Q, class KG, int GRP>
__device__ __forceinline__ void k2_gather(const double* __restrict__ st, double (&blur)[Dims<Q>::KM], int tx, int ty)
{
#pragma unroll
    for (int g = 0; g < KG::G; ++g) {
        const int k = GRP * KG::G + g;
        if (k < Dims<Q>::KM) blur[k] = st[(g * kK2TY + ty) * KG::SP + tx];
    }
}

// the tile's models (staged in shared memory, k2_msp floats per block) -> global, by the
// kK2Threads threads tid of the tile
template <int Q>
__device__ __forceinline__ void k2_store_models(const float* mstage, float* __restrict__ models, int mstride, int f,
                                                int bx0, int by0, int Bx, int By, int tid)
{
    constexpr int TX = kK2TX, TY = kK2TY, MS = Dims<Q>::MSTRIDE, MSP = k2_msp<Q>;
    const int nbx = min(TX, Bx - bx0), nrow = min(TY, By - by0);
    static_assert(MS % 4 == 0, "padded models are whole float4s");
    if (mstride == MS && (reinterpret_cast<uintptr_t>(models) & 15) == 0) {  // rows: contiguous aligned runs
        const int q = nbx * (MS / 4);
        for (int i = tid; i < nrow * q; i += kK2Threads) {
            const int r = i / q, j = i - r * q, b = 4 * j / MS;  // float4 j lies in block b
            const float* m = mstage + (r * TX + b) * MSP + 4 * j - b * MS;
            reinterpret_cast<float4*>(models + ((size_t)(f * By + by0 + r) * Bx + bx0) * MS)[j] =
                make_float4(m[0], m[1], m[2], m[3]);
        }
    } else {  // the ABI's packed [Q+1][3] models (flr_fit): runs of nbx * mstride floats, 4-byte aligned
        const int q = nbx * mstride;
        for (int i = tid; i < nrow * q; i += kK2Threads) {
            const int r = i / q, j = i - r * q, b = j / mstride;
            models[((size_t)(f * By + by0 + r) * Bx + bx0) * mstride + j] = mstage[(r * TX + b) * MSP + j - b * mstride];
        }
    }
    (void)TY;
}

// One TX x TY tile of output blocks (frame f, first block (bx0, by0)), run by the kK2Threads
// threads of the CTA (tid = threadIdx.x) in lock step.  smk: KG::BAR_OFF bytes of shared
// memory, bar: S mbarriers, initialised here (every earlier use of them must have completed).
// tm: the fp64 moment field [n*KM][By][Bxp] with box {HX, TY + 2R, G} (K2Geom).
template <int Q, int R>
__device__ __forceinline__ void k2_tile(const CUtensorMap* tmp, int f, int bx0, int by0, int Bx, int By,
                                        float* __restrict__ models, int mstride, double eps_add, double eps_mul,
                                        const Taps& t, double* smk, uint64_t* bar, uint64_t kpol)
{
    using Dm = Dims<Q>;
    using KG = K2Geom<Q, R>;
    constexpr int KM = Dm::KM, G = KG::G, NG = KG::NG, RE = KG::RE, S = KG::S;
    constexpr int TX = kK2TX, MS = Dm::MSTRIDE;
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
    double blur[KM];
    static_for<NG>([&](auto GRP) {
        constexpr int grp = decltype(GRP)::value;
        mbar_wait(&bar[grp % S], (grp / S) & 1);
        k2_vpass<KG, R, kK2Threads>(ring + (grp % S) * KG::BOX, vb, t, tid);
        __syncthreads();  // vb complete, stage grp % S consumed (and the previous gather done)
        if (tid == 0 && grp + S < NG) issue(grp + S);
        k2_hpass<KG, R, kK2Threads>(vb, st, t, tid);
        __syncthreads();  // stage complete (and vb free for the next v-pass)
        k2_gather<Q, KG, grp>(st, blur, tx, ty);
    });
    __syncthreads();  // every gather done: smem now stages the models
    float* mstage = reinterpret_cast<float*>(smk);
    const int bx = bx0 + tx, by = by0 + ty;
    if (bx < Bx && by < By) {
        solve_block<Q>([&](int k) { return blur[k]; }, eps_add, eps_mul, mstage + tid * KG::MSP);
#pragma unroll
        for (int i = 3 * (Q + 1); i < MS; ++i) mstage[tid * KG::MSP + i] = 0.0f;
    }
    __syncthreads();
    k2_store_models<Q>(mstage, models, mstride, f, bx0, by0, Bx, By, tid);
}

// the SOLVE warps' side of k_blur_solve_tile: gather each group as the blur warps publish
// it (st_full), release the stage (st_empty), factor as the components arrive (DirectSolve:
// row by row; TikhonovSolve: after group KF), finish after the last.
// MODE 0: DirectSolve, 1: TikhonovSolve (raw models; the centred layout takes the row
// kernels), 2: gather everything, then solve_block (the FLR_SOLVE_NORMALISED build).
template <int Q, int R, int MODE>
__device__ __forceinline__ void k2_solve_role(const double* st, uint64_t* sfull, uint64_t* sempty, bool active,
                                              float* out, double eps_add, double eps_mul, int tx, int ty)
{
    using KG = K2WsGeom<Q, R>;
    using WG = KG;
    constexpr int NG = KG::NG, NST = WG::NST;
#ifdef FLR_DBG_PHASES
    long long tsg[NG + 3];
    tsg[0] = clock64();
#endif
    double blur[Dims<Q>::KM];
    auto m = [&](int k) { return blur[k]; };
    std::conditional_t<MODE == 1, TikhonovSolve<Q>, DirectSolve<Q>> sv;
    static_for<NG>([&](auto GRP) {
        constexpr int grp = decltype(GRP)::value;
        mbar_wait(&sfull[grp % NST], (grp / NST) & 1);
#ifdef FLR_DBG_PHASES
        tsg[grp + 1] = clock64();
#endif
        k2_gather<Q, KG, grp>(st + (grp % NST) * KG::ST, blur, tx, ty);
        mbar_arrive(&sempty[grp % NST]);
        if constexpr (MODE == 0) {  // factor row by row as the rows of S arrive, then the
                                    // forward substitution as the cross moments arrive
            using Dm = Dims<Q>;
            constexpr int G = KG::G, BEGIN = (Dm::C_S - 1) / G;  // n and u are in
            constexpr int RHS = cmax(Dm::s_idx(Q - 1, Q - 1) / G, (Dm::C_Y + 2) / G);  // S and Y are in
            if (active) {
                if constexpr (grp == BEGIN) sv.begin(m);
                static_for<Q>([&](auto K) {
                    constexpr int k = decltype(K)::value;
                    if constexpr (cmax(Dm::s_idx(k, Q - 1) / G, BEGIN) == grp) sv.template row<k>(m, eps_add, eps_mul);
                });
                if constexpr (grp == RHS) sv.rhs_begin(m);
                static_for<Q>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    if constexpr (cmax((Dm::C_XY + 3 * i + 2) / G, RHS) == grp) sv.template fwd<i>(m);
                });
            }
        } else if constexpr (MODE == 1 && grp == WG::KF) {
            if (active) sv.factor(m, eps_add);
        }
    });
    if (active) {
        if constexpr (MODE == 0) sv.back_out(out);
        else if constexpr (MODE == 1) sv.finish(m, out, false);
        else solve_block<Q>(m, eps_add, eps_mul, out);
#pragma unroll
        for (int i = 3 * (Q + 1); i < Dims<Q>::MSTRIDE; ++i) out[i] = 0.0f;
    }
#ifdef FLR_DBG_PHASES
    tsg[NG + 1] = clock64();
    tsg[NG + 2] = tsg[NG + 1];
    if (tx == 0 && ty == 0 && blockIdx.x == 2 && blockIdx.y == 2 && blockIdx.z == 0) {
        extern __device__ long long g_flr_phase[];
        for (int i = 0; i < NG + 3; ++i) g_flr_phase[i] = tsg[i] - tsg[0];
        g_flr_phase[63] = NG + 3;
    }
#endif
}

template <int Q, int R>
__global__ void __launch_bounds__(kK2WsThreads, 1)
    k_blur_solve_tile(const __grid_constant__ CUtensorMap tm, int Bx, int By, float* __restrict__ models,
                      int mstride, double eps_add, double eps_mul, const __grid_constant__ Taps t)
{
    using Dm = Dims<Q>;
    using KG = K2WsGeom<Q, R>;
    using WG = KG;
    constexpr int KM = Dm::KM, G = KG::G, NG = KG::NG, RE = KG::RE, S = KG::S, NST = WG::NST;
    extern __shared__ __align__(1024) double smk[];
    double* ring = smk;
    double* vb = smk + WG::RING;
    double* st = vb + KG::VB;
    uint64_t* tfull = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(smk) + WG::BAR_OFF);
    uint64_t* sfull = tfull + S;
    uint64_t* sempty = sfull + NST;
    const int tid = threadIdx.x;
    if (tid == 0) FLR_TL(1, 0);
    pdl_wait();  // the moment field comes from the previous grid
    pdl_trigger();  // dependents launch only once we are past our own wait
    if (tid == 0) {
        FLR_TL(1, 1);
        for (int i = 0; i < S; ++i) mbar_init(&tfull[i], 1);
        for (int i = 0; i < NST; ++i) {
            mbar_init(&sfull[i], kK2BlurThreads);
            mbar_init(&sempty[i], kK2Threads);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int f = blockIdx.z, bx0 = blockIdx.x * kK2TX, by0 = blockIdx.y * kK2TY;
    if (tid >= kK2Threads) {  // ---------------- blur warps ----------------
        const int bt = tid - kK2Threads;
        const uint64_t kpol = policy_evict_last();  // the moment field stays in L2 (see k_fit_ws)
        auto issue = [&](int grp) {
            uint64_t* b = &tfull[grp % S];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the stage before
            mbar_arrive_expect_tx(b, KG::BOXD * sizeof(double));
            tma_load_3d(ring + (grp % S) * KG::BOX, &tm, bx0 - RE, by0 - R, f * KM + grp * G, b, kpol);
        };
        if (bt == 0)
            for (int g = 0; g < S && g < NG; ++g) issue(g);
#pragma unroll 1
        for (int grp = 0; grp < NG; ++grp) {
            mbar_wait(&tfull[grp % S], (grp / S) & 1);
            k2_vpass<KG, R, kK2BlurThreads>(ring + (grp % S) * KG::BOX, vb, t, bt);
            named_bar_sync(1, kK2BlurThreads);  // vb complete, ring slot grp % S consumed
            if (bt == 0 && grp + S < NG) issue(grp + S);
            if (grp >= NST) mbar_wait(&sempty[grp % NST], ((grp / NST) - 1) & 1);
            k2_hpass<KG, R, kK2BlurThreads>(vb, st + (grp % NST) * KG::ST, t, bt);
            mbar_arrive(&sfull[grp % NST]);
            named_bar_sync(1, kK2BlurThreads);  // every h-pass read of vb done before the next v-pass
        }
        return;
    }
    // ---------------- solve warps: thread (tx, ty) owns block (bx0 + tx, by0 + ty) ----------------
    const int tx = tid % kK2TX, ty = tid / kK2TX;
    const bool active = bx0 + tx < Bx && by0 + ty < By;
    // the models stage in the TMA ring: free once the last group has been published (its
    // v-pass, which read the last ring slot, precedes its h-pass)
    float* mstage = reinterpret_cast<float*>(smk);
    float* out = mstage + tid * KG::MSP;
#ifdef FLR_SOLVE_NORMALISED
    k2_solve_role<Q, R, 2>(st, sfull, sempty, active, out, eps_add, eps_mul, tx, ty);
#else
    if (eps_mul < 0.0) k2_solve_role<Q, R, 1>(st, sfull, sempty, active, out, eps_add, eps_mul, tx, ty);
    else k2_solve_role<Q, R, 0>(st, sfull, sempty, active, out, eps_add, eps_mul, tx, ty);
#endif
    named_bar_sync(2, kK2Threads);  // the tile's models are staged
    k2_store_models<Q>(mstage, models, mstride, f, bx0, by0, Bx, By, tid);
    if (tid == 0) FLR_TL(1, 2);
}

}  // namespace flr
