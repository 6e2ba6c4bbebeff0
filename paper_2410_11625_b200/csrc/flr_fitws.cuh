// flr_fitws.cuh -- K1 (block moments) as a warp-specialised TMA pipeline.
//
// One CTA per SM: kFitWsNC consumer warps + 1 producer warp.  Lane c of the producer
// walks consumer c's item sequence and keeps its kFitWsS-stage shared-memory ring full
// (one TMA pair per pixel row: the Q guide planes and the 3 radiance planes of 128
// pixels); consumers wait on the stage's `full` mbarrier, accumulate, and arrive on its
// `empty` mbarrier.  Consumer warps therefore run no producer code at all: per row they
// do 22 shared loads, 8 + 71 packed fp32x2 operations per pixel pair and two barrier ops.
//
// Accumulation is in PIXEL pairs (fma.rn.f32x2 of two pixels' products, both operands
// vectors): a lane's 4 pixels are 2 pairs of the same block, so every packed operand
// comes straight from an 8-byte shared load with no repacking, and the pair halves are
// added once per item.  Sums are taken about the block's top-left pixel c (design rule
// H1) and un-shifted to fp64 in the epilogue (FitAcc::store's algebra).
#pragma once
#include <cuda_fp16.h>

#include <type_traits>

#include "flr_stream.cuh"

namespace flr {

#ifndef FLR_FITWS_NC
#define FLR_FITWS_NC 7
#endif
constexpr int kFitWsNC = FLR_FITWS_NC;  // consumer warps (+1 producer = 8 warps: 2 per SMSP keeps the 255-register cap)
#ifndef FLR_FITWS_NP
#define FLR_FITWS_NP 1
#endif
constexpr int kFitWsNP = FLR_FITWS_NP;  // producer warps (producer p feeds consumers p, p + NP, ...)
#ifndef FLR_FITWS_S
#define FLR_FITWS_S 4
#endif
constexpr int kFitWsS = FLR_FITWS_S;  // ring stages per consumer (1-row stages)
#ifndef FLR_FITWS_S2
#define FLR_FITWS_S2 2  // ring stages per consumer with 2-row stages
#endif
#ifndef FLR_FIT_SEG
#define FLR_FIT_SEG 128
#endif
// segment width of a FIT item in pixels: 128 (4 pixels per lane) or 64 (2 per lane: half the
// bytes per item, for a shorter grid tail; give it twice the stages)
constexpr int kFS = FLR_FIT_SEG, kPPL = kFS / 32, kNH = kPPL / 2;
static_assert(kFS == 128 || kFS == 64, "fit segment: 64 or 128 pixels");

template <int Q, bool MOD = false, bool HG = false>
struct FitWsCfg {
    // floats per pixel row of a stage: Q guide planes (fp32, or fp16 when HG), 3 radiance
    // planes (+ 3 albedo planes)
    static constexpr int GF = HG ? kFS / 2 : kFS;  // floats per guide plane row
    static constexpr int ROWF = Q * GF + (3 + (MOD ? 3 : 0)) * kFS;
    // A stage holds RB pixel rows: one TMA box {128, RB, planes} per tensor.  The producer
    // warp's issue rate, not HBM, limits one SM at one row per box (measured ~50 GB/s per
    // SM, tools/t_tma_rate.cu); two rows per box double it.  RB = 2 with 2 stages per
    // consumer when that fits in 227 KB, else single rows with up to kFitWsS stages.
    static constexpr bool TWO = (size_t)kFitWsNC * FLR_FITWS_S2 * 2 * ROWF * 4 + 4096 <= 232448;
    static constexpr int RB = TWO ? 2 : 1;
    static constexpr int STG = RB * ROWF;  // floats per stage
    static constexpr int fit_stages(int s)
    {
        return (s <= 2 || (size_t)kFitWsNC * s * STG * 4 + 4096 <= 232448) ? s : fit_stages(s - 1);
    }
    static constexpr int NC = kFitWsNC, NP = kFitWsNP, S = TWO ? FLR_FITWS_S2 : fit_stages(kFitWsS),
                         THREADS = (NC + NP) * 32;
    static constexpr size_t BAR_OFF = (size_t)NC * S * STG * sizeof(float);
    static constexpr size_t SMEM = BAR_OFF + 2 * NC * S * sizeof(uint64_t);
    static_assert(SMEM <= 232448, "fit pipeline exceeds 227 KB of shared memory");
    // offsets (floats) inside a stage: guide plane j / radiance plane c, row r of the stage
    __host__ __device__ static constexpr int g_off(int j, int r) { return (j * RB + r) * GF; }
    __host__ __device__ static constexpr int y_off(int c, int r) { return Q * RB * GF + (c * RB + r) * kFS; }
};

// per-lane accumulators of one item, pixel-pair packed
template <int Q>
struct FitAccPix {
    using Dm = Dims<Q>;
    f2 U[Q], S[Dm::NS], Y[3], XY[3 * Q];
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int j = 0; j < Q; ++j) U[j] = 0ull;
#pragma unroll
        for (int s = 0; s < Dm::NS; ++s) S[s] = 0ull;
#pragma unroll
        for (int c = 0; c < 3; ++c) Y[c] = 0ull;
#pragma unroll
        for (int k = 0; k < 3 * Q; ++k) XY[k] = 0ull;
    }
    // d[j]: shifted guide j of the pixel pair, y[c]: radiance
    __device__ __forceinline__ void add(const f2 (&d)[Q], const f2 (&y)[3])
    {
#pragma unroll
        for (int c = 0; c < 3; ++c) Y[c] = add2(Y[c], y[c]);
#pragma unroll
        for (int j = 0; j < Q; ++j) U[j] = add2(U[j], d[j]);
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
            for (int j = i; j < Q; ++j) S[Dm::s_idx(i, j) - Dm::C_S] = fma2(d[i], d[j], S[Dm::s_idx(i, j) - Dm::C_S]);
#pragma unroll
        for (int j = 0; j < Q; ++j)
#pragma unroll
            for (int c = 0; c < 3; ++c) XY[j * 3 + c] = fma2(d[j], y[c], XY[j * 3 + c]);
    }
};

// per-lane accumulators in fp64 (Tikhonov mode): its system (Mbar/n + eps I) is not
// normalised, so at eps ~1e-6 the fp32 rounding of edge blocks' shifted sums reaches the
// solution (model errors ~1e-3 relative at 1080p); DFMA is half the FFMA rate on B200 and
// the fit stays bandwidth-bound.  Same interface as FitAccPix.
template <int Q>
struct FitAcc64 {
    using Dm = Dims<Q>;
    double U[Q], S[Dm::NS], Y[3], XY[3 * Q];
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int j = 0; j < Q; ++j) U[j] = 0.0;
#pragma unroll
        for (int s = 0; s < Dm::NS; ++s) S[s] = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) Y[c] = 0.0;
#pragma unroll
        for (int k = 0; k < 3 * Q; ++k) XY[k] = 0.0;
    }
    __device__ __forceinline__ void add(const f2 (&d2)[Q], const f2 (&y2)[3])
    {
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // the pixel pair's two pixels
            double d[Q], y[3];
#pragma unroll
            for (int j = 0; j < Q; ++j) d[j] = (double)(h ? hi2(d2[j]) : lo2(d2[j]));
#pragma unroll
            for (int c = 0; c < 3; ++c) y[c] = (double)(h ? hi2(y2[c]) : lo2(y2[c]));
#pragma unroll
            for (int c = 0; c < 3; ++c) Y[c] += y[c];
#pragma unroll
            for (int j = 0; j < Q; ++j) U[j] += d[j];
#pragma unroll
            for (int i = 0; i < Q; ++i)
#pragma unroll
                for (int j = i; j < Q; ++j) S[Dm::s_idx(i, j) - Dm::C_S] = fma(d[i], d[j], S[Dm::s_idx(i, j) - Dm::C_S]);
#pragma unroll
            for (int j = 0; j < Q; ++j)
#pragma unroll
                for (int c = 0; c < 3; ++c) XY[j * 3 + c] = fma(d[j], y[c], XY[j * 3 + c]);
        }
    }
};

// fold the m lanes of a block (xor shuffles) of fp64 sums
template <int N>
__device__ __forceinline__ void fold_pairs(const double (&in)[N], double (&out)[N], int m_lanes)
{
#pragma unroll
    for (int k = 0; k < N; ++k) out[k] = in[k];
    for (int m = 1; m < m_lanes; m <<= 1)
#pragma unroll
        for (int k = 0; k < N; ++k) out[k] += __shfl_xor_sync(0xffffffffu, out[k], m);
}

// fold the pair halves and the m lanes of a block (xor shuffles) into plain fp32 sums
template <int N>
__device__ __forceinline__ void fold_pairs(const f2 (&in)[N], float (&out)[N], int m_lanes)
{
#pragma unroll
    for (int k = 0; k < N; ++k) out[k] = lo2(in[k]) + hi2(in[k]);
    for (int m = 1; m < m_lanes; m <<= 1)
#pragma unroll
        for (int k = 0; k < N; ++k) out[k] += __shfl_xor_sync(0xffffffffu, out[k], m);
}

// the rows of one item for one consumer warp (k: stages consumed so far by this warp)
// Rel: called by lane 0 with the slot once its values are in registers (frees the stage:
// arrive on its `empty` barrier, or -- self-feeding warps -- issue the next stage into it)
template <int Q, int D, bool EDGE, bool MOD, bool HG, class Acc, class Rel>
__device__ __forceinline__ void fit_ws_rows(Acc& acc, float (&cs)[Q], const float* ring, uint64_t* full, Rel&& rel,
                                            int& k, int rows, int lane, int lb0, int x0, int W, float afloor)
{
    using C = FitWsCfg<Q, MOD, HG>;
    constexpr int S = C::S, STG = C::STG, RB = C::RB;
    {  // the block shift c = its top-left pixel (first row of the item)
#ifndef FLR_FITWS_NOWAIT
        mbar_wait(&full[k % S], (k / S) & 1);
#else  // timing experiment (tools/t_rate.cu): the producer fills the ring once, the consumers
       // re-read it -- the consumers' compute rate alone
        if (k < S) mbar_wait(&full[k % S], (k / S) & 1);
#endif
        const float* st = ring + (k % S) * STG;
#pragma unroll
        for (int j = 0; j < Q; ++j)
            cs[j] = HG ? __half2float(reinterpret_cast<const __half*>(st + C::g_off(j, 0))[lb0]) : st[C::g_off(j, 0) + lb0];
    }
#pragma unroll 1  // keep the row body resident in the instruction cache
    for (int r0 = 0; r0 < rows; r0 += RB, ++k) {
        const int slot = k % S;
#ifndef FLR_FITWS_NOWAIT
        mbar_wait(&full[slot], (k / S) & 1);
#else
        if (k < S) mbar_wait(&full[slot], (k / S) & 1);
#endif
        const float* st = ring + slot * STG;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            if (RB > 1 && r0 + r >= rows) break;  // odd row count at the bottom edge
#pragma unroll
            for (int h = 0; h < kNH; ++h) {
                f2 d[Q], y[3];
#pragma unroll
                for (int j = 0; j < Q; ++j) {
                    if (HG) {  // fp16 guide pair -> fp32 (exact)
                        const float2 v =
                            __half22float2(reinterpret_cast<const __half2*>(st + C::g_off(j, r))[kNH * lane + h]);
                        d[j] = pk2(v.x, v.y);
                    } else {
                        d[j] = reinterpret_cast<const f2*>(st + C::g_off(j, r))[kNH * lane + h];
                    }
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) y[c] = reinterpret_cast<const f2*>(st + C::y_off(c, r))[kNH * lane + h];
                if (MOD) {  // demodulation y = radiance / max(albedo, floor) (R20)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const f2 al = reinterpret_cast<const f2*>(st + C::y_off(3 + c, r))[kNH * lane + h];
                        y[c] = pk2(lo2(y[c]) * __frcp_rn(fmaxf(lo2(al), afloor)),
                                   hi2(y[c]) * __frcp_rn(fmaxf(hi2(al), afloor)));
                    }
                }
#pragma unroll
                for (int j = 0; j < Q; ++j) d[j] = sub2(d[j], bc2(cs[j]));
                if (EDGE) {  // pixels past the image arrive as zeros: make them contribute nothing
                    const bool in0 = x0 + 2 * h < W, in1 = x0 + 2 * h + 1 < W;
#pragma unroll
                    for (int j = 0; j < Q; ++j) d[j] = pk2(in0 ? lo2(d[j]) : 0.f, in1 ? hi2(d[j]) : 0.f);
                }
#ifndef FLR_FITWS_NOCOMPUTE
                acc.add(d, y);
#else
                if (lo2(d[0]) == 12345.f) acc.add(d, y);  // timing experiment: stream without accumulating
#endif
            }
        }
        __syncwarp();
        if (lane == 0) rel(slot);  // values are in registers: free the stage
    }
}

// One FIT item (frame f, block row by, segment sg; item index `it`) for one consumer warp:
// its rows from the warp's ring (k: stages consumed so far), then the epilogue -- fold the
// pair halves and the lanes of a block, un-shift exactly to fp64 and store the moments.
// `waited`: the grid-dependency wait has run (in early mode it runs before the first store).
template <int Q, int D, bool MOD, bool HG, bool A64, class Rel>
__device__ __forceinline__ void fit_consume_item_rel(const FitArgs& a, int it, int per_frame, const float* ring,
                                                     uint64_t* full, Rel&& rel, int& k, int lane, bool& waited)
{
    using Acc = std::conditional_t<A64, FitAcc64<Q>, FitAccPix<Q>>;
    using V = std::conditional_t<A64, double, float>;
    using Dm = Dims<Q>;
    constexpr int DQ = D / kPPL;  // lanes per block
    const int f = it / per_frame, rem = it - f * per_frame, by = rem / a.nseg, sg = rem - by * a.nseg;
    const int rows = min(D, a.H - by * D);
    const int x0 = sg * kFS + lane * kPPL, bx = x0 / D, lb0 = (lane / DQ) * D;
    float cs[Q];
    Acc acc;
    acc.zero();
    if (sg * kFS + kFS > a.W)  // segment reaches past the image
        fit_ws_rows<Q, D, true, MOD, HG>(acc, cs, ring, full, rel, k, rows, lane, lb0, x0, a.W, a.afloor);
    else
        fit_ws_rows<Q, D, false, MOD, HG>(acc, cs, ring, full, rel, k, rows, lane, lb0, x0, a.W, a.afloor);
#ifdef FLR_FITWS_NOEPI  // timing experiment (tools/t_rate.cu): no epilogue (accumulators kept live)
    {
        float z = 0.f;
#pragma unroll
        for (int i = 0; i < Dm::NS; ++i) z += lo2(acc.S[i]) + hi2(acc.S[i]);
#pragma unroll
        for (int i = 0; i < 3 * Q; ++i) z += lo2(acc.XY[i]) + hi2(acc.XY[i]);
#pragma unroll
        for (int i = 0; i < Q; ++i) z += lo2(acc.U[i]) + hi2(acc.U[i]);
#pragma unroll
        for (int i = 0; i < 3; ++i) z += lo2(acc.Y[i]) + hi2(acc.Y[i]);
        if (z == 12345.f) a.mom[lane] = z;
    }
    return;
#endif
    // epilogue: fold, then un-shift to fp64 and store (lanes of a block split the components)
    V u[Q], sv[Dm::NS], yc[3], xy[3 * Q];
    fold_pairs(acc.U, u, DQ);
    fold_pairs(acc.S, sv, DQ);
    fold_pairs(acc.Y, yc, DQ);
    fold_pairs(acc.XY, xy, DQ);
    if (!waited) {
        pdl_wait();
        waited = true;
    }
    if (bx < a.Bx) {
        const int gi = lane % DQ;
        const double nn = (double)(min(D, a.W - bx * D) * rows);
        const size_t cst = (size_t)a.By * a.Bxp;
#ifdef FLR_FIT_MOM_ALIAS  // timing experiment (tools/t_rate.cu): every frame's moments in one L2-resident field
        double* out = a.mom + (size_t)by * a.Bxp + bx;
#else
        double* out = a.mom + (size_t)f * Dm::KM * cst + (size_t)by * a.Bxp + bx;
#endif
        // the moment field is stored (and read by K2) evict_last: the next call rewrites the same
        // lines, which then stay in L2 instead of being written back under the next fit's
        // stream (C2 43.05 -> 42.4, 32-frame calls 43.4 -> 42.35 us per frame)
        const uint64_t mpol = policy_evict_last();
        auto put = [&](int kk, double v) {
            if (kk % DQ == gi) st_hint_f64(out + (size_t)kk * cst, v, mpol);
        };
        put(Dm::C_N, nn);
#pragma unroll
        for (int j = 0; j < Q; ++j) put(Dm::C_U + j, fma(nn, (double)cs[j], (double)u[j]));
        // S_ij = S'_ij + c_i u'_j + c_j u'_i + n c_i c_j
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
            for (int j = i; j < Q; ++j) {
                double v = (double)sv[Dm::s_idx(i, j) - Dm::C_S];
                v = fma((double)cs[i], (double)u[j], v);
                v = fma((double)cs[j], (double)u[i], v);
                v = fma(nn * (double)cs[i], (double)cs[j], v);
                put(Dm::s_idx(i, j), v);
            }
#pragma unroll
        for (int c = 0; c < 3; ++c) put(Dm::C_Y + c, (double)yc[c]);
#pragma unroll
        for (int j = 0; j < Q; ++j)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                put(Dm::C_XY + j * 3 + c, fma((double)cs[j], (double)yc[c], (double)xy[j * 3 + c]));
    }
}

template <int Q, int D, bool MOD, bool HG, bool A64 = false>
__device__ __forceinline__ void fit_consume_item(const FitArgs& a, int it, int per_frame, const float* ring,
                                                 uint64_t* full, uint64_t* empty, int& k, int lane, bool& waited)
{
    fit_consume_item_rel<Q, D, MOD, HG, A64>(a, it, per_frame, ring, full, [&](int s) { mbar_arrive(&empty[s]); }, k,
                                             lane, waited);
}
template <int Q, int D, bool MOD = false, bool HG = false, bool A64 = false>
__global__ void __launch_bounds__(FitWsCfg<Q, MOD, HG>::THREADS, 1) k_fit_ws(const __grid_constant__ FitArgs a, int n)
{
    using C = FitWsCfg<Q, MOD, HG>;
    if (threadIdx.x == 0) FLR_TL(0, 0);
    constexpr int NC = C::NC, S = C::S, STG = C::STG;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* stages = reinterpret_cast<float*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + C::BAR_OFF);
    uint64_t* empty = full + NC * S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NC * S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int per_frame = a.By * a.nseg, nitems = n * per_frame, GW = gridDim.x * NC;
    // Default: the inputs may come from the previous grid, so wait for it before streaming.
    // Early (inputs ready before the previous grid began): the producer streams at once and
    // runs the wait (+ trigger) once it has issued its last row, so the dependents -- K2,
    // which writes the models the previous call's apply may still be reading -- launch only
    // after the previous grid completed.  The consumers also wait before their first store
    // to the moment field, which the previous grid (a K2 reading it by TMA) may still read.
    if (!a.early) {
        pdl_wait();  // caller data may come from the previous grid
        pdl_trigger();  // dependents launch only once we are past our own wait
    }
    if (threadIdx.x == 0) FLR_TL(0, 1);

    if (warp >= NC) {
        // ---------------- producer p: lane i feeds consumer c = p + NP i ----------------
        constexpr int NP = C::NP, LANES = (NC + NP - 1) / NP;
        const int p = warp - NC, c = p + NP * lane;
        if (lane >= LANES || c >= NC) return;
                // the guide rows from a.keep_y0 down (the bottom-up apply reads them first) stay in L2
        // (evict_normal); the rows above stream (evict_first) -- see launch_k1
        const uint64_t pg = policy_evict_normal(), py = policy_evict_first();
        int it = blockIdx.x * NC + c, row = 0, rows = 0, f = 0, by = 0, sg = 0;
        auto decode = [&]() {
            if (it >= nitems) return;
            f = it / per_frame;
            const int rem = it - f * per_frame;
            by = rem / a.nseg;
            sg = rem - by * a.nseg;
            rows = min(D, a.H - by * D);
        };
        decode();
        // the lanes stay converged: each round, every lane whose next slot is free
        // (non-blocking test) issues one stage for its consumer
        int k = 0;
        const unsigned mask = __activemask();
        while (__any_sync(mask, it < nitems)) {
            const int slot = k % S;
#ifndef FLR_FITWS_NOWAIT
            if (it < nitems && (k < S || mbar_test_wait(&empty[c * S + slot], ((k / S) - 1) & 1))) {
#else
            if (it < nitems && k < S) {
#endif
                ws_proxy_fence();
                fit_issue_row<Q, D, MOD, HG, kFS, C::RB>(a, f, by, sg, row, stages + (size_t)(c * S + slot) * STG,
                                                         &full[c * S + slot], by * D >= a.keep_y0 ? pg : py, py);
                ++k;
                if ((row += C::RB) >= rows) {
                    row = 0;
                    it += GW;
                    decode();
                }
            }
#ifdef FLR_FITWS_NOWAIT
            if (k >= S) it = nitems;
#endif
        }
        if (a.early && lane == 0) {  // (each trigger follows a completed wait: safe from any producer)
            pdl_wait();
            pdl_trigger();
        }
        return;
    }

    // ---------------- consumer warp ----------------
    const int w = warp;
    float* ring = stages + (size_t)w * S * STG;
    int k = 0;  // stages consumed
    bool waited = !a.early;  // past the grid-dependency wait (early mode: before the first store)
    for (int it = blockIdx.x * NC + w; it < nitems; it += GW)
        fit_consume_item<Q, D, MOD, HG, A64>(a, it, per_frame, ring, full + w * S, empty + w * S, k, lane, waited);
    if (threadIdx.x == 0) FLR_TL(0, 2);
}


}  // namespace flr
