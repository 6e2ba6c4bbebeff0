// flr_applyws.cuh -- K3 (apply the blended per-block models, R4) as a
// warp-specialised TMA pipeline, like flr_fitws.cuh.
//
// One CTA per SM: kApplyWsNC consumer warps + 1 producer warp.  Lane c of the producer
// walks consumer c's APPLY items (sub-band of D/nsub output rows x 128 pixels) and keeps
// two rings full: the items' 2 x 18 staged models (two 1-D bulk copies per item, kApplyWsM
// stages, running ahead of the rows: a stage is free once its models are in registers) and
// the guide rows (one 3-D TMA box {128, RB, Q} per stage; 2 or 3 stages of 2 rows at Q = 8).  Consumers run no
// producer code: per item each lane keeps its two model columns (top row and bottom-top
// difference) in registers; per row it forms A_y = top + t_y (bottom - top), reads its
// pixel quad of the Q guide planes, and applies I = (1 - t_x) x~.A_y(i0) + t_x x~.A_y(i1)
// with packed fp32x2 FMAs, streaming the 3 output planes out (st.global.cs).
#pragma once
#include <cuda_fp16.h>

#include "flr_stream.cuh"

#ifndef FLR_OUT_ST
#define FLR_OUT_ST "st.global.cs.v4.f32"
#endif

namespace flr {

#ifndef FLR_APPLYWS_NC
#define FLR_APPLYWS_NC 7
#endif
#ifndef FLR_APPLYWS_S
#define FLR_APPLYWS_S 4
#endif
constexpr int kApplyWsNC = FLR_APPLYWS_NC;  // consumer warps (+1 producer = 8 warps, 255-register cap)
constexpr int kApplyWsS = FLR_APPLYWS_S;  // guide-row stages per consumer
#ifndef FLR_APPLYWS_M
#define FLR_APPLYWS_M 2
#endif
#ifndef FLR_APPLYWS_S2
#define FLR_APPLYWS_S2 2
#endif
#ifndef FLR_SMEM_RESERVE
#define FLR_SMEM_RESERVE 4096  // bytes kept free for barriers and static shared memory
#endif
constexpr int kApplyWsM = FLR_APPLYWS_M;   // model stages per consumer

// DEEP: one model stage and three 2-row guide stages per consumer (the guides are mostly L2
// hits -- the fit of the same call left them there: C2 43.0 vs 43.5 us per frame); the
// default (two model stages, two guide stages) is faster when the guides stream from HBM
// (C4 37.1 vs 37.75, 32-frame calls 43.3 vs 44.4 us per frame)
template <int Q, bool MOD = false, bool HG = false, bool DEEP = false>
struct ApplyWsCfg {
    using SD = StreamDims<Q>;
    // floats per output row: Q guide planes (fp32, or fp16 when HG) (+ 3 albedo and 3
    // direct-light planes)
    static constexpr int GF = HG ? kSeg / 2 : kSeg;  // floats per guide plane row
    static constexpr int ROW1 = Q * GF + (MOD ? 6 : 0) * kSeg;
    static constexpr int MODF = 2 * kApplyNCol * SD::MS;  // floats per model stage
    static constexpr int MSTG = DEEP ? 1 : kApplyWsM;     // model stages
    // a row stage holds RB output rows (one TMA box {128, RB, planes} per tensor): two rows
    // per box double what the producer warp can issue per SM (see FitWsCfg); RB = 2 with 2
    // stages when that fits in 227 KB, else single rows with up to kApplyWsS stages
    static constexpr bool TWO = (size_t)kApplyWsNC * ((2 * 2 * ROW1 + MSTG * MODF + 31) / 32 * 32) * 4 + FLR_SMEM_RESERVE <=
                                232448;
    static constexpr int RB = TWO ? 2 : 1;
    static constexpr int ROWF = RB * ROW1;  // floats per row stage
    static constexpr int fit_stages(int s)
    {
        return (s <= 2 || (size_t)kApplyWsNC * ((s * ROWF + MSTG * MODF + 31) / 32 * 32) * 4 + FLR_SMEM_RESERVE <= 232448)
                   ? s : fit_stages(s - 1);
    }
    static constexpr int NC = kApplyWsNC, S = TWO ? fit_stages(DEEP ? 3 : FLR_APPLYWS_S2) : fit_stages(kApplyWsS), SM = MSTG,
                         THREADS = (NC + 1) * 32;
    static constexpr int WARPF = (S * ROWF + SM * MODF + 31) / 32 * 32;  // 128-byte aligned regions
    static constexpr size_t BAR_OFF = (size_t)NC * WARPF * sizeof(float);
    static constexpr int NBAR = 2 * (S + SM);  // full + empty per stage
    static constexpr size_t SMEM = BAR_OFF + (size_t)NC * NBAR * sizeof(uint64_t);
    static_assert(WARPF % 32 == 0 && ROWF % 32 == 0 && MODF % 4 == 0, "16-byte aligned stages");
    // the modulated variant (6 more planes per row) does not fit for the largest Q: those
    // shapes remodulate in a separate elementwise kernel (apply_mod_supported)
    static constexpr bool FITS = SMEM <= 232448;
    static_assert(FITS || MOD, "apply pipeline exceeds 227 KB of shared memory");
    // offsets (floats) in a row stage: guide plane j, remodulation plane c (albedo 0-2,
    // direct 3-5), row r of the stage
    __host__ __device__ static constexpr int g_off(int j, int r) { return (j * RB + r) * GF; }
    __host__ __device__ static constexpr int m_off(int c, int r) { return RB * Q * GF + (c * RB + r) * kSeg; }
};

// One APPLY item (frame f, geometry g) for one consumer warp: its models from the warp's
// model ring (km: model stages consumed), its guide rows from the row ring (kr), the
// output rows streamed out.  RG: the ring geometry (S, SM, ROWF, MODF, RB, g_off, m_off).
template <int Q, bool MOD, bool HG, class RG>
__device__ __forceinline__ void apply_consume_item(const ApplyArgs& a, const ApplyGeom& g, int f, const float* rows_st,
                                                   const float* mod_st, uint64_t* rfull, uint64_t* rempty,
                                                   uint64_t* mfull, uint64_t* mempty, int& kr, int& km, int lane)
{
    using C = RG;
    using SD = StreamDims<Q>;
    constexpr int S = C::S, SM = C::SM, MS = SD::MS;
    constexpr int MP = MS / 2;  // model float pairs
    const float invD = 1.0f / (float)a.D;
    const size_t plane = (size_t)a.W * a.H;
    const int xq = g.xs + lane * 4;  // the lane's quad
    const bool active = xq < a.W;
    const float fxq = ((float)xq + 0.5f) * invD - 0.5f;
    const int ib = (int)floorf(fxq);
    const int c0 = min(max(ib, 0), a.Bx - 1) - g.ic0;
    const int c1 = min(max(ib + 1, 0), a.Bx - 1) - g.ic0;
    f2 t2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
        t2[h] = pk2(((float)(xq + 2 * h) + 0.5f) * invD - 0.5f - (float)ib,
                    ((float)(xq + 2 * h + 1) + 0.5f) * invD - 0.5f - (float)ib);
    // the lane's two model columns, top (block row j0) and bottom (j1) -> registers:
    // A_y = top + t_y (bottom - top) is then 2 x MS/2 packed FMAs per row
    f2 top0[MP], dlt0[MP], top1[MP], dlt1[MP];
    {
        const int ms = km % SM;
#ifndef FLR_APPLYWS_NOWAIT
        mbar_wait(&mfull[ms], (km / SM) & 1);
#else  // timing experiment (tools/t_rate.cu): rings filled once and re-read -- the consumers' arithmetic alone
        if (km < SM) mbar_wait(&mfull[ms], (km / SM) & 1);
#endif
        const float* mod = mod_st + ms * C::MODF;
#pragma unroll
        for (int v = 0; v < MS / 4; ++v) {
            const float4 p0 = reinterpret_cast<const float4*>(mod + c0 * MS)[v];
            const float4 q0 = reinterpret_cast<const float4*>(mod + (kApplyNCol + c0) * MS)[v];
            const float4 p1 = reinterpret_cast<const float4*>(mod + c1 * MS)[v];
            const float4 q1 = reinterpret_cast<const float4*>(mod + (kApplyNCol + c1) * MS)[v];
            top0[2 * v] = pk2(p0.x, p0.y), top0[2 * v + 1] = pk2(p0.z, p0.w);
            top1[2 * v] = pk2(p1.x, p1.y), top1[2 * v + 1] = pk2(p1.z, p1.w);
            dlt0[2 * v] = sub2(pk2(q0.x, q0.y), top0[2 * v]), dlt0[2 * v + 1] = sub2(pk2(q0.z, q0.w), top0[2 * v + 1]);
            dlt1[2 * v] = sub2(pk2(q1.x, q1.y), top1[2 * v]), dlt1[2 * v + 1] = sub2(pk2(q1.z, q1.w), top1[2 * v + 1]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&mempty[ms]);  // models are in registers: free the stage
        ++km;
    }
    float* O = a.out + (size_t)f * 3 * plane;
#pragma unroll 1
    for (int ys = g.y0; ys < g.y1; ys += C::RB, ++kr) {
        const int rs = kr % S;
#ifndef FLR_APPLYWS_NOWAIT
        mbar_wait(&rfull[rs], (kr / S) & 1);
#else
        if (kr < S) mbar_wait(&rfull[rs], (kr / S) & 1);
#endif
        const float* st = rows_st + rs * C::ROWF;
        float o[C::RB][3][4];
#pragma unroll
        for (int r = 0; r < C::RB; ++r) {
            const int y = ys + r;
            const float fy = ((float)y + 0.5f) * invD - 0.5f;
            const f2 ty2 = bc2(fy - floorf(fy));
            float gq[Q][4];
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                float4 v;
                if (HG) {  // 4 fp16 guides -> fp32 (exact)
                    const uint2 hv = reinterpret_cast<const uint2*>(st + C::g_off(j, r))[lane];
                    const float2 lo = __half22float2(*reinterpret_cast<const __half2*>(&hv.x));
                    const float2 hi = __half22float2(*reinterpret_cast<const __half2*>(&hv.y));
                    v = make_float4(lo.x, lo.y, hi.x, hi.y);
                } else {
                    v = reinterpret_cast<const float4*>(st + C::g_off(j, r))[lane];
                }
                gq[j][0] = v.x; gq[j][1] = v.y; gq[j][2] = v.z; gq[j][3] = v.w;
            }
            float m0[MS], m1[MS];
#pragma unroll
            for (int v = 0; v < MP; ++v) {
                upk2(fma2(ty2, dlt0[v], top0[v]), m0[2 * v], m0[2 * v + 1]);
                upk2(fma2(ty2, dlt1[v], top1[v]), m1[2 * v], m1[2 * v + 1]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // pixel pairs (2h, 2h+1)
                f2 gp[Q];
#pragma unroll
                for (int j = 0; j < Q; ++j) gp[j] = pk2(gq[j][2 * h], gq[j][2 * h + 1]);
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    f2 p0 = bc2(m0[cc]), p1 = bc2(m1[cc]);
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        p0 = fma2(gp[j], bc2(m0[(1 + j) * 3 + cc]), p0);
                        p1 = fma2(gp[j], bc2(m1[(1 + j) * 3 + cc]), p1);
                    }
                    upk2(fma2(t2[h], sub2(p1, p0), p0), o[r][cc][2 * h], o[r][cc][2 * h + 1]);
                }
            }
            if (MOD) {  // remodulation and direct light: out = albedo * I + direct (R21)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    const float4 al = reinterpret_cast<const float4*>(st + C::m_off(cc, r))[lane];
                    float4 dl = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (a.has_direct) dl = reinterpret_cast<const float4*>(st + C::m_off(3 + cc, r))[lane];
                    o[r][cc][0] = fmaf(al.x, o[r][cc][0], dl.x);
                    o[r][cc][1] = fmaf(al.y, o[r][cc][1], dl.y);
                    o[r][cc][2] = fmaf(al.z, o[r][cc][2], dl.z);
                    o[r][cc][3] = fmaf(al.w, o[r][cc][3], dl.w);
                }
            }
        }
        __syncwarp();  // guide stage consumed by every lane
        if (lane == 0) mbar_arrive(&rempty[rs]);
        if (active) {
#pragma unroll
            for (int r = 0; r < C::RB; ++r) {
                if (ys + r >= g.y1) break;  // odd row count at an image edge
                float* Orow = O + (size_t)(ys + r) * a.W + xq;
#pragma unroll
                for (int cc = 0; cc < 3; ++cc)
                    asm volatile(FLR_OUT_ST " [%0], {%1,%2,%3,%4};" ::"l"(Orow + cc * plane),
                                 "f"(o[r][cc][0]), "f"(o[r][cc][1]), "f"(o[r][cc][2]), "f"(o[r][cc][3])
                                 : "memory");
            }
        }
    }
}

template <int Q, bool MOD = false, bool HG = false, bool DEEP = false>
__global__ void __launch_bounds__(ApplyWsCfg<Q, MOD, HG, DEEP>::THREADS, 1) k_apply_ws(const __grid_constant__ ApplyArgs a, int n)
{
    using C = ApplyWsCfg<Q, MOD, HG, DEEP>;
    if (threadIdx.x == 0) FLR_TL(2, 0);
    constexpr int NC = C::NC, S = C::S, SM = C::SM;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + C::BAR_OFF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NC * C::NBAR; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int per_frame = a.nband * a.nsub * a.nseg, nitems = n * per_frame, GW = gridDim.x * NC;
    // Only the producer touches data of earlier grids (the models, by bulk copy), so only it
    // waits (griddepcontrol.wait), and only after it has queued the first guide rows: the
    // guides are inputs of the call, complete before the fit grid got past its own wait
    // (every grid of the chain triggers its dependents only after its wait).
    // Dependents (normally the next call's moment grid) launch only once the models' grid has
    // completed (the producer's lane 0 triggers after its wait): a following moment grid that
    // streams before its own wait (FLR_FLAG_INPUTS_READY) then cannot overwrite the moment
    // field K2 is still reading.

    auto geom = [&](int it, int& f) {
        f = it / per_frame;
        int rem = it - f * per_frame;
        if (a.reverse) rem = per_frame - 1 - rem;
        return apply_geom(a, rem / a.nseg, rem - (rem / a.nseg) * a.nseg);
    };

    if (warp == NC) {
        // ---------------- producer: lane c feeds consumer c ----------------
        if (lane >= NC) return;
        const int c = lane;
        float* base = reinterpret_cast<float*>(smem_raw) + (size_t)c * C::WARPF;
        float* rows_st = base;
        float* mod_st = base + S * C::ROWF;
        uint64_t* rfull = bars + c * C::NBAR;
        uint64_t* rempty = rfull + S;
        uint64_t* mfull = rempty + S;
        uint64_t* mempty = mfull + SM;
                const uint64_t pg = policy_evict_first(), pm = policy_evict_normal();
        // two cursors over the consumer's items: the guide rows (it, y) and the models (itm),
        // which run up to SM items ahead -- a model stage is free as soon as the consumer has
        // its models in registers, so the next item's models are in flight while this one's
        // rows stream (models issued only once the rows of an item were queued left every
        // item start waiting one L2 round trip for its models)
        int it = blockIdx.x * NC + c, itm, f = 0, fm = 0, y = 0, kr = 0, km = 0;
        ApplyGeom g, gm;
        auto valid = [&](int& i, ApplyGeom& gg, int& ff) {  // skip empty sub-bands (rows outside the image)
            for (; i < nitems; i += GW) {
                gg = geom(i, ff);
                if (gg.y0 < gg.y1) break;
            }
        };
        valid(it, g, f);
        y = g.y0;
        itm = it, gm = g, fm = f;
        // guide rows of the first item, ahead of the models (and of the wait): the guides are
        // inputs of the call
        for (; kr < S && it < nitems; ++kr) {
            ws_proxy_fence();
            apply_issue_row<Q, MOD, HG, C::RB>(a, g, f, y, rows_st + kr * C::ROWF, &rfull[kr], pg);
            if ((y += C::RB) >= g.y1) {
                it += GW;
                valid(it, g, f);
                y = g.y0;
            }
        }
        pdl_wait();  // the models come from the previous grid
        if (lane == 0) pdl_trigger();
        if (lane == 0) FLR_TL(2, 1);

        constexpr unsigned mask = (1u << NC) - 1;
        while (__any_sync(mask, it < nitems || itm < nitems)) {
#ifdef FLR_APPLYWS_NOWAIT
            if (kr >= S && km >= SM) it = itm = nitems;
#endif
            if (itm < nitems) {
                const int s = km % SM;
                if (km < SM || mbar_test_wait(&mempty[s], ((km / SM) - 1) & 1)) {
                    ws_proxy_fence();
                    apply_issue_models<Q>(a, gm, fm, mod_st + s * C::MODF, &mfull[s], pm);
                    ++km;
                    itm += GW;
                    valid(itm, gm, fm);
                }
            }
            if (it < nitems) {
                const int s = kr % S;
                if (kr < S || mbar_test_wait(&rempty[s], ((kr / S) - 1) & 1)) {
                    ws_proxy_fence();
                    apply_issue_row<Q, MOD, HG, C::RB>(a, g, f, y, rows_st + s * C::ROWF, &rfull[s], pg);
                    ++kr;
                    if ((y += C::RB) >= g.y1) {
                        it += GW;
                        valid(it, g, f);
                        y = g.y0;
                    }
                }
            }
        }
        return;
    }

    // ---------------- consumer warp ----------------
    const int w = warp;
    float* base = reinterpret_cast<float*>(smem_raw) + (size_t)w * C::WARPF;
    const float* rows_st = base;
    const float* mod_st = base + S * C::ROWF;
    uint64_t* rfull = bars + w * C::NBAR;
    uint64_t* rempty = rfull + S;
    uint64_t* mfull = rempty + S;
    uint64_t* mempty = mfull + SM;
    int kr = 0, km = 0;
    for (int it = blockIdx.x * NC + w; it < nitems; it += GW) {
        int f;
        const ApplyGeom g = geom(it, f);
        if (g.y0 >= g.y1) continue;
        apply_consume_item<Q, MOD, HG, C>(a, g, f, rows_st, mod_st, rfull, rempty, mfull, mempty, kr, km, lane);
    }
    if (threadIdx.x == 0) FLR_TL(2, 2);
}

}  // namespace flr
