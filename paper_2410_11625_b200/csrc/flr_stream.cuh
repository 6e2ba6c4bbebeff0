// flr_stream.cuh -- the item geometry and TMA issue helpers of the streaming kernels
// (k_fit_ws, k_apply_ws, k_flr_wave): full-resolution planes move through shared-memory
// rings filled by the TMA engine, one 3-D tensor box {128 px, rows, planes} per tensor per
// stage (out-of-image pixels arrive as zeros).  Two item kinds:
//   FIT: one block row x 128 fit pixels -> fp64
//         moments of 128/D blocks: fp32 accumulation about the per-block shift c
//         (design rule H1) with packed FFMA2 pairs, exact fp64 un-shift.
//   APPLY: a sub-band of output rows x 128 output pixels,
//         I = x~ A_blend, with the two bracketing rows of block models delivered by
//         bulk copy into a model stage.
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
    int keep_y0;     // guide rows y >= keep_y0 are read evict_normal (the call's bottom-up apply
                     // re-reads them from L2), the rows above evict_first; H: none
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

}  // namespace flr
