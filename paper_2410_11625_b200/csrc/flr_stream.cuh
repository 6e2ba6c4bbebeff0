// flr_stream.cuh -- warp-granular streaming of full-resolution planes through a
// per-warp shared-memory ring filled by the TMA engine.
//
// Every stream warp owns a ring of S stages.  A stage holds one pixel row of a
// 128-pixel segment of every plane an item needs, fetched by ONE 3-D TMA tensor
// load per tensor (box 128 x 1 x planes; out-of-image pixels arrive as zeros)
// that completes on the stage's mbarrier.  Lane 0 of the warp keeps the producer
// cursor and refills a stage as soon as the warp has read it, so S rows stay in
// flight per warp.  Two item kinds:
//   FIT: one block row x 128 fit pixels -> fp64
//         moments of 128/D blocks: fp32 accumulation about the per-block shift c
//         (design rule H1) with packed FFMA2 pairs, exact fp64 un-shift.
//   APPLY: 8 output rows x 128 output pixels,
//         I = x~ A_blend, with the two bracketing rows of block models delivered
//         as one extra (bulk-copy) stage.
#pragma once
#include <cuda.h>

#include "flr_common.cuh"
#include "flr_pipe.cuh"

namespace flr {

constexpr int kSeg = 128;       // pixels per segment row (32 lanes x 4)
constexpr int kApplyNCol = 18;  // model columns an APPLY item can touch (128/8 + 2)

template <int Q>
struct StreamDims {
    static constexpr int NPF = Q + 3;                 // planes of a FIT row
    static constexpr int MS = Dims<Q>::MSTRIDE;       // floats per padded model
    static constexpr int MODF = 2 * kApplyNCol * MS;  // floats of an APPLY item's models
    static constexpr int STG_FIT = NPF * kSeg;  // (Q+3) * 512 B: a multiple of 128 B
    static constexpr int STG_APPLY = ((Q * kSeg > MODF ? Q * kSeg : MODF) + 31) / 32 * 32;
};

struct Ring {
    float* stage;      // [S][STG]
    uint64_t* full;    // [S]
    int S, STG;
    unsigned cons = 0;    // stages consumed (uniform across the warp)
    unsigned prod = 0;    // stages produced (lane 0 only)
    int cslot = 0;        // consumer slot = cons % S, kept incrementally (no integer modulo)
    unsigned cphase = 0;  // consumer parity = (cons / S) & 1
    int pslot = 0;        // producer slot = prod % S (lane 0 only)
};

// lane 0: issue stages until S are in flight or the sequence ends
template <class Seq>
__device__ __forceinline__ void ring_fill(Ring& r, Seq& q)
{
    while (r.prod < r.cons + r.S && q.next(r.stage + r.pslot * r.STG, &r.full[r.pslot])) {
        ++r.prod;
        if (++r.pslot == r.S) r.pslot = 0;
    }
}

// wait until the warp's next stage is filled.  If lane 0's cursor stopped at an item
// whose dependency was not ready yet (Seq::next returned false), lane 0 keeps retrying
// here, where the warp has nothing else to do.
template <class Seq>
__device__ __forceinline__ const float* ring_wait(Ring& r, Seq& q, int lane)
{
    if (lane == 0) {
        while (r.prod <= r.cons) {
            ring_fill(r, q);
            if (r.prod <= r.cons) __nanosleep(256);
        }
    }
    __syncwarp();
#ifdef FLR_DBG_TIMES
    const long long t0 = clock64();
    mbar_wait(&r.full[r.cslot], r.cphase);
    extern __device__ unsigned long long g_flr_wait_cycles[4096];
    if (lane == 0) g_flr_wait_cycles[(blockIdx.x * 32 + (threadIdx.x >> 5)) & 4095] += clock64() - t0;
#else
    mbar_wait(&r.full[r.cslot], r.cphase);
#endif
    return r.stage + r.cslot * r.STG;
}

// all lanes done reading the current stage: release it and let lane 0 refill
template <class Seq>
__device__ __forceinline__ void ring_release(Ring& r, Seq& q, int lane)
{
    __syncwarp();
    ++r.cons;
    if (++r.cslot == r.S) {
        r.cslot = 0;
        r.cphase ^= 1u;
    }
    if (lane == 0) {
#ifndef FLR_DBG_NOFENCE
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
        ring_fill(r, q);
    }
}

// ============================================================================
// FIT item: frame f, block row by, segment sg (fit pixels [128 sg, 128 sg + 128)).
// ============================================================================
struct FitArgs {
    CUtensorMap tg;  // guides   [n*Q][H][W], box {128, 1, Q}
    CUtensorMap ty;  // radiance [n*3][H][W], box {128, 1, 3}
    double* mom;     // [n][KM][By][Bxp]
    int W, H, Bx, Bxp, By, nseg;
    CUtensorMap ta;  // albedo [n*3][H][W], box {128, 1, 3} (modulated fit only)
    float afloor;    // albedo floor of the demodulation (modulated fit only)
    int early;       // inputs ready (FLR_FLAG_INPUTS_READY): stream before the grid-dependency
                     // wait, which then only gates this grid's dependents (see k_fit_ws)
};

// HG: the guide planes are IEEE binary16 (half the stage bytes of the guides)
// SW: segment width in pixels (the TMA box width of every plane); RB: pixel rows per box
// (the tensor maps' box height).  Stage layout: [Q planes][RB rows][SW] guides, then
// [3 (+3) planes][RB rows][SW] radiance (+ albedo); rows past the image arrive as zeros.
template <int Q, int D, bool MOD = false, bool HG = false, int SW = kSeg, int RB = 1>
__device__ __forceinline__ void fit_issue_row(const FitArgs& a, int f, int by, int sg, int rr, float* dst,
                                              uint64_t* bar, uint64_t pol_g, uint64_t pol_y)
{
    constexpr int GF = HG ? SW / 2 : SW;  // floats of stage per guide plane row
    mbar_arrive_expect_tx(bar, RB * (Q * GF + (3 + (MOD ? 3 : 0)) * SW) * 4);
    const int x = sg * SW, y = by * D + rr;
    tma_load_3d(dst, &a.tg, x, y, f * Q, bar, pol_g);
    tma_load_3d(dst + RB * Q * GF, &a.ty, x, y, f * 3, bar, pol_y);
    if (MOD) tma_load_3d(dst + RB * (Q * GF + 3 * SW), &a.ta, x, y, f * 3, bar, pol_y);
}

// ============================================================================
// APPLY item: frame f, band j (output rows [jD - D/2, jD + D/2) inside the image),
// segment sg (output pixels [128 sg, 128 sg + 128)).  Every row of band j lies between
// the block centres (b + 1/2) D - 1/2 of block rows j-1 and j (clamped, R4), and for
// D % 8 == 0 every 4-pixel quad lies between one pair of block-centre columns.
// ============================================================================
struct ApplyArgs {
    CUtensorMap tg;       // output-resolution guides [n*Q][H][W], box {128, 1, Q}
    const float* models;  // [n][By][Bx][MS]
    float* out;           // [n][3][H][W]
    int W, H, D, Bx, By, nseg, nband;
    int nsub;  // sub-bands per band (D % nsub == 0): more, smaller APPLY items for one frame
    int reverse;  // walk each frame's items bottom-up (the rows the fit read last come first)
    CUtensorMap ta, td;  // albedo, direct [n*3][H][W], box {128, 1, 3} (modulated apply only)
    int has_direct;      // modulated apply: 0 = no direct-light planes (treated as zero)
};

__host__ __device__ inline int apply_nband(int H, int D, int By)
{
    const int nb = (H + D / 2 + D - 1) / D;  // bands j with j*D - D/2 < H
    return nb < By + 1 ? nb : By + 1;
}

struct ApplyGeom {
    int y0, y1;   // rows [y0, y1)
    int xs;       // first pixel of the segment
    int j0, j1;   // bracketing block rows (clamped)
    int ic0, nc;  // first staged model column, number staged
};

// item geometry of sub-band u = j * nsub + s of band j: rows [jD - D/2 + s D/nsub, ...)
// clipped to the band and the image (possibly empty)
__device__ __forceinline__ ApplyGeom apply_geom(const ApplyArgs& a, int u, int sg)
{
    ApplyGeom g;
    const float invD = 1.0f / (float)a.D;
    const int j = a.nsub == 1 ? u : u / a.nsub, s = u - j * a.nsub, rs = a.D / a.nsub;
    const int yb = j * a.D - a.D / 2 + s * rs;
    g.y0 = max(yb, 0);
    g.y1 = min(yb + rs, a.H);
    g.xs = sg * kSeg;
    g.j0 = min(max(j - 1, 0), a.By - 1);
    g.j1 = min(j, a.By - 1);
    g.ic0 = min(max((int)floorf(((float)g.xs + 0.5f) * invD - 0.5f), 0), a.Bx - 1);
    g.nc = min(kApplyNCol, a.Bx - g.ic0);
    return g;
}

// model stage: the two rows of block models [j][ic0 .. ic0+nc) (lane 0)
template <int Q>
__device__ __forceinline__ void apply_issue_models(const ApplyArgs& a, const ApplyGeom& g, int f, float* dst,
                                                   uint64_t* bar, uint64_t pol_m)
{
    using SD = StreamDims<Q>;
    const unsigned mb = (unsigned)(g.nc * SD::MS * 4);
    mbar_arrive_expect_tx(bar, 2 * mb);
    const float* M = a.models + (size_t)f * a.By * a.Bx * SD::MS;
    bulk_g2s(dst, M + ((size_t)g.j0 * a.Bx + g.ic0) * SD::MS, mb, bar, pol_m);
    bulk_g2s(dst + kApplyNCol * SD::MS, M + ((size_t)g.j1 * a.Bx + g.ic0) * SD::MS, mb, bar, pol_m);
}

// guide rows y .. y + RB - 1 of an APPLY item (one box per tensor; the tensor maps' box
// height is RB).  Stage layout: [Q][RB][128] guides, then [3][RB][128] albedo and
// [3][RB][128] direct light (modulated apply only)
template <int Q, bool MOD = false, bool HG = false, int RB = 1>
__device__ __forceinline__ void apply_issue_row(const ApplyArgs& a, const ApplyGeom& g, int f, int y, float* dst,
                                                uint64_t* bar, uint64_t pol_g)
{
    constexpr int GF = HG ? kSeg / 2 : kSeg;  // floats of stage per guide plane row
    mbar_arrive_expect_tx(bar, RB * (Q * GF + (MOD ? (a.has_direct ? 6 : 3) : 0) * kSeg) * 4);
    tma_load_3d(dst, &a.tg, g.xs, y, f * Q, bar, pol_g);
    if (MOD) {  // remodulation planes: albedo, then the direct light
        tma_load_3d(dst + RB * Q * GF, &a.ta, g.xs, y, f * 3, bar, pol_g);
        if (a.has_direct) tma_load_3d(dst + RB * (Q * GF + 3 * kSeg), &a.td, g.xs, y, f * 3, bar, pol_g);
    }
}

// stream warp.  `mod` = per-warp [2][kApplyNCol][MS] raw models, `lerp` = [kApplyNCol][MS].
template <int Q, class Seq>
__device__ __forceinline__ void apply_consume(Ring& r, Seq& sq, const ApplyArgs& a, int f, int ty, int sg, int lane,
                                              float* mod, float* lerp)
{
    using SD = StreamDims<Q>;
    constexpr int MS = SD::MS, P = Q + 1;
    const ApplyGeom g = apply_geom(a, ty, sg);
    const float invD = 1.0f / (float)a.D;
    {  // models: copy out of the ring so the stage can be refilled at once
        const float* st = ring_wait(r, sq, lane);
        const float4* s4 = reinterpret_cast<const float4*>(st);
        float4* d4 = reinterpret_cast<float4*>(mod);
        for (int i = lane; i < 2 * kApplyNCol * MS / 4; i += 32) d4[i] = s4[i];
        ring_release(r, sq, lane);
    }
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
    const size_t plane = (size_t)a.W * a.H;
    float* O = a.out + (size_t)f * 3 * plane;
#pragma unroll 1
    for (int y = g.y0; y < g.y1; ++y) {
        const float fy = ((float)y + 0.5f) * invD - 0.5f;
        const float tyy = fy - floorf(fy);
        // y-blend the staged model columns once per row for the whole warp
        for (int i = lane; i < g.nc * (MS / 4); i += 32) {
            const float4 p = reinterpret_cast<const float4*>(mod)[i];
            const float4 q = reinterpret_cast<const float4*>(mod + kApplyNCol * MS)[i];
            reinterpret_cast<float4*>(lerp)[i] =
                make_float4(fmaf(tyy, q.x - p.x, p.x), fmaf(tyy, q.y - p.y, p.y), fmaf(tyy, q.z - p.z, p.z),
                            fmaf(tyy, q.w - p.w, p.w));
        }
        __syncwarp();
        const float* st = ring_wait(r, sq, lane);
        float gq[Q][4];
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            const float4 v = reinterpret_cast<const float4*>(st + j * kSeg)[lane];
            gq[j][0] = v.x; gq[j][1] = v.y; gq[j][2] = v.z; gq[j][3] = v.w;
        }
        ring_release(r, sq, lane);
        float m0[4 * (MS / 4)], m1[4 * (MS / 4)];
#pragma unroll
        for (int v = 0; v < MS / 4; ++v) {
            const float4 p = reinterpret_cast<const float4*>(lerp + c0 * MS)[v];
            const float4 q = reinterpret_cast<const float4*>(lerp + c1 * MS)[v];
            m0[4 * v] = p.x; m0[4 * v + 1] = p.y; m0[4 * v + 2] = p.z; m0[4 * v + 3] = p.w;
            m1[4 * v] = q.x; m1[4 * v + 1] = q.y; m1[4 * v + 2] = q.z; m1[4 * v + 3] = q.w;
        }
        __syncwarp();  // `lerp` is rewritten for the next row
        float o[3][4];
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
                upk2(fma2(t2[h], sub2(p1, p0), p0), o[cc][2 * h], o[cc][2 * h + 1]);
            }
        }
        if (active) {
            float* Orow = O + (size_t)y * a.W + xq;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
                asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(Orow + cc * plane), "f"(o[cc][0]),
                             "f"(o[cc][1]), "f"(o[cc][2]), "f"(o[cc][3])
                             : "memory");
        }
        (void)P;
    }
}

}  // namespace flr
