// flr_fused.cuh -- the whole FLR hot path (fit + solve + apply) as ONE
// persistent, warp-specialised kernel per call: a row wavefront over every frame.
//
// One CTA per SM (cooperative launch: all CTAs co-resident), 12 warps:
//   warps 0..7  stream warps: FIT items (block row x 128 fit pixels -> fp64 block
//               moments) and APPLY items (band of D_out output rows x 128 pixels ->
//               radiance), each warp with its own TMA-fed row ring (flr_stream.cuh);
//   warps 8..11 solver group: SOLVE items (32 x 4 blocks: Gaussian blur of the
//               moment field + the appendix's normalised, regularised solve, fp64).
// 12 warps cap every thread at 168 registers, so the solver keeps only the S block of
// its blurred moments in registers and parks n, u, Y, XY (and then B^) in shared memory.
// The stream warps walk one merged sequence per frame: super-row s holds the FIT
// items of block row s and the APPLY items of band s - LAG, so an APPLY runs about
// LAG block rows after the FIT that produced its moments -- while those guide rows
// are still in L2 (the 56 B/px minimum-traffic design).
// Dependencies are global counters (acquire/release at gpu scope):
//   fit_done[f][by]   += 1 per FIT item of row by           (complete at nseg_fit)
//   solve_done[f][m]  += 1 per SOLVE tile of row-tile m      (complete at ncx)
// SOLVE(m) waits for fit rows [4m-R, 4m+3+R]; APPLY(band j) waits for the solve row
// tiles holding block rows j-1 and j.  Every wait is on an item placed earlier in
// the sequence, so the schedule cannot deadlock while all CTAs are resident.
#pragma once
#include "flr_persist.cuh"
#include "flr_tiles.cuh"

namespace flr {

constexpr int kFusedStreamWarps = 8;
constexpr int kFusedSolveWarps = 4;
constexpr int kFusedThreads = 32 * (kFusedStreamWarps + kFusedSolveWarps);
constexpr int kFusedG = 8;  // moment components per halo box of the solver

struct FusedArgs {
    FitArgs fit;          // fit-resolution guides/radiance maps, moment field
    ApplyArgs app;        // output-resolution guide map, models, output
    CUtensorMap tmom;     // moment field, box {halo_x(R), 4 + 2R, kTileG}
    Taps taps;
    int* fit_done;        // [n][By]
    int* solve_done;      // [n][nrt]
    int n, lag, nrt, ncx;
    double eps_add, eps_mul;
};

// solver tile geometry: single halo buffer of G components, v-pass buffer, spill area
template <int Q, int R>
struct FusedTile {
    static constexpr int RE = (R + 1) & ~1;
    static constexpr int HX = kTileTX + 2 * RE, HY = kTileTY + 2 * R, G = kFusedG;
    static constexpr int NT = kTileTX * kTileTY;
    static constexpr int NO = 4 * Q + 4;  // components kept in shared memory: n, u, Y, XY
    static constexpr int HALO = G * HY * HX, VB = G * kTileTY * HX, SPILL = NO * NT;
    static constexpr size_t BYTES = (size_t)(HALO + VB + SPILL) * sizeof(double);
    // spill slot of a non-S component k
    __host__ __device__ static constexpr int o_idx(int k)
    {
        using Dm = Dims<Q>;
        return k < Dm::C_S ? k : (k < Dm::C_XY ? Q + 1 + (k - Dm::C_Y) : Q + 4 + (k - Dm::C_XY));
    }
    __host__ __device__ static constexpr bool in_reg(int k) { return k >= Dims<Q>::C_S && k < Dims<Q>::C_Y; }
};

template <int Q, int R>
struct FusedCfg {
    static constexpr int S = 2;
    using SD = StreamDims<Q>;
    static constexpr int STG = SD::STG_FIT > SD::STG_APPLY ? SD::STG_FIT : SD::STG_APPLY;
    static constexpr int WARP_FLOATS = (S * STG + 3 * kApplyNCol * SD::MS + 31) / 32 * 32;
    static constexpr size_t STREAM_BYTES = (size_t)kFusedStreamWarps * WARP_FLOATS * 4;
    static constexpr size_t SOLVE_BYTES = FusedTile<Q, R>::BYTES;
    static constexpr size_t BAR_OFF = STREAM_BYTES + SOLVE_BYTES;
    static constexpr size_t SMEM = BAR_OFF + (kFusedStreamWarps * S + 1) * sizeof(uint64_t);
    static_assert(SMEM <= 232448, "fused kernel exceeds 227 KB of shared memory");
};

// One 32 x 4 tile of blocks by the 128-thread solver group: for each group of G
// moment components, one TMA halo box (single buffer: the next box is issued as soon
// as the v-pass has consumed this one), vertical then horizontal fp64 pass (P:334,
// separable Gaussian), then the appendix solve per thread (flr_solve.cuh).
template <int Q, int R, class Sync>
__device__ __forceinline__ void fused_blur_solve(const CUtensorMap* tm, int f, int bx0, int by0, int Bx, int By,
                                                 float* __restrict__ models, int mstride, double eps_add,
                                                 double eps_mul, const Taps& t, double* sm, uint64_t* bar,
                                                 unsigned& use, int tid, Sync grp_sync)
{
    using Dm = Dims<Q>;
    using FT = FusedTile<Q, R>;
    constexpr int KM = Dm::KM, GG = FT::G, NG = (KM + GG - 1) / GG;
    constexpr int TX = kTileTX, TY = kTileTY, NT = FT::NT;
    constexpr int RE = FT::RE, HX = FT::HX, HY = FT::HY;
    constexpr unsigned BOX_BYTES = FT::HALO * sizeof(double);
    double* halo = sm;
    double* vb = sm + FT::HALO;
    double* spill = vb + FT::VB + tid;  // component slot o at spill[o * NT]
    const int tx = tid % TX, ty = tid / TX;
    auto issue = [&](int grp) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(bar, BOX_BYTES);
        tma_load_3d(halo, tm, bx0 - RE, by0 - R, f * KM + grp * GG, bar, policy_evict_normal());
    };
    if (tid == 0) issue(0);
    double sreg[Dm::NS];
#pragma unroll
    for (int grp = 0; grp < NG; ++grp) {
        mbar_wait(bar, use & 1);
        ++use;
        for (int col = tid; col < GG * HX; col += 2 * NT) {
            const int col2 = col + NT;
            const bool two = col2 < GG * HX;
            const int gi = col / HX, cc = col - gi * HX;
            const int gi2 = two ? col2 / HX : gi, cc2 = two ? col2 - gi2 * HX : cc;
            const double* src = halo + gi * HY * HX + cc;
            const double* src2 = halo + gi2 * HY * HX + cc2;
            double v[HY], w[HY];
#pragma unroll
            for (int r = 0; r < HY; ++r) {
                v[r] = src[r * HX];
                w[r] = src2[r * HX];
            }
#pragma unroll
            for (int r = 0; r < TY; ++r) {
                double a = t.g[R] * v[r + R], b = t.g[R] * w[r + R];
#pragma unroll
                for (int d = 1; d <= R; ++d) {
                    a = fma(t.g[R + d], v[r + R - d] + v[r + R + d], a);
                    b = fma(t.g[R + d], w[r + R - d] + w[r + R + d], b);
                }
                vb[(gi * TY + r) * HX + cc] = a;
                if (two) vb[(gi2 * TY + r) * HX + cc2] = b;
            }
        }
        grp_sync.sync();  // halo consumed, vb complete
        if (tid == 0 && grp + 1 < NG) issue(grp + 1);
#pragma unroll
        for (int gi = 0; gi < GG; ++gi) {
            const int k = grp * GG + gi;
            if (k < KM) {
                const double* src = vb + (gi * TY + ty) * HX + tx + RE;
                double acc = t.g[R] * src[0];
#pragma unroll
                for (int d = 1; d <= R; ++d) acc = fma(t.g[R + d], src[-d] + src[d], acc);
                if (FT::in_reg(k)) sreg[k - Dm::C_S] = acc;
                else spill[FT::o_idx(k) * NT] = acc;
            }
        }
        grp_sync.sync();  // vb free for the next group
    }
    const int bx = bx0 + tx, by = by0 + ty;
    if (bx >= Bx || by >= By) return;
    SmemB B{spill + FT::o_idx(Dm::C_XY) * NT, NT};  // B^ overwrites the XY slots it is made from
    solve_block_b<Q>([&](int k) { return FT::in_reg(k) ? sreg[k - Dm::C_S] : spill[FT::o_idx(k) * NT]; }, eps_add,
                     eps_mul, models + ((size_t)(f * By + by) * Bx + bx) * mstride, B);
}

// ---- merged stream sequence -------------------------------------------------
struct StreamItem {
    int kind;  // 0 FIT, 1 APPLY, -1 none
    int f, row, sg;
};

__device__ __forceinline__ int fused_before(const FusedArgs& a, int s)
{
    // items of super-rows [0, s): FIT rows min(s, By), APPLY bands clamp(s - LAG, 0, nband)
    const int fr = min(s, a.fit.By);
    const int ab = min(max(s - a.lag, 0), a.app.nband);
    return fr * a.fit.nseg + ab * a.app.nseg;
}

__device__ __forceinline__ StreamItem fused_decode(const FusedArgs& a, int it)
{
    StreamItem r;
    const int nsuper = max(a.fit.By, a.lag + a.app.nband);
    const int per_frame = fused_before(a, nsuper);
    if (it >= per_frame * a.n) {
        r.kind = -1;
        return r;
    }
    r.f = it / per_frame;
    const int i = it - r.f * per_frame;
    int lo = 0, hi = nsuper;  // largest s with before(s) <= i
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (fused_before(a, mid) <= i) lo = mid;
        else hi = mid;
    }
    const int j = i - fused_before(a, lo);
    const int nf = lo < a.fit.By ? a.fit.nseg : 0;
    if (j < nf) {
        r.kind = 0;
        r.row = lo;
        r.sg = j;
    } else {
        r.kind = 1;
        r.row = lo - a.lag;
        r.sg = j - nf;
    }
    return r;
}

// APPLY(band j) may start once the solve row tiles of block rows j-1 and j are done
__device__ __forceinline__ bool apply_ready(const FusedArgs& a, int f, int j)
{
    const int m0 = min(max(j - 1, 0), a.app.By - 1) / kTileTY, m1 = min(j, a.app.By - 1) / kTileTY;
    return ld_acquire(&a.solve_done[f * a.nrt + m0]) >= a.ncx && ld_acquire(&a.solve_done[f * a.nrt + m1]) >= a.ncx;
}

// producer cursor of a stream warp over its items (lane 0 only)
template <int Q, int D>
struct FusedSeq {
    const FusedArgs* a;
    int it, step, row;  // row: FIT 0..rows-1; APPLY -1 = model stage, then y
    StreamItem cur;
    ApplyGeom g;
    uint64_t pol_keep, pol_once;
    __device__ void load()
    {
        cur = fused_decode(*a, it);
        row = cur.kind == 1 ? -1 : 0;
        if (cur.kind == 1) g = apply_geom(a->app, cur.row, cur.sg);
    }
    __device__ bool next(float* dst, uint64_t* bar)
    {
        if (cur.kind < 0) return false;
        if (cur.kind == 0) {
            // guides stay in L2 for the APPLY ~LAG rows later; radiance is read once
            fit_issue_row<Q, D>(a->fit, cur.f, cur.row, cur.sg, row, dst, bar, pol_keep, pol_once);
            if (++row == min(D, a->fit.H - cur.row * D)) {
                it += step;
                load();
            }
            return true;
        }
        if (row < 0) {
            if (!apply_ready(*a, cur.f, cur.row)) return false;  // retried from ring_wait
            asm volatile("fence.proxy.async.global;" ::: "memory");  // models written by other SMs
            apply_issue_models<Q>(a->app, g, cur.f, dst, bar, pol_once);
            row = g.y0;
            if (row >= g.y1) {
                it += step;
                load();
            }
            return true;
        }
        apply_issue_row<Q>(a->app, g, cur.f, row, dst, bar, pol_once);
        if (++row == g.y1) {
            it += step;
            load();
        }
        return true;
    }
};

template <int Q, int D, int R>
__global__ void __launch_bounds__(kFusedThreads, 1) k_flr_fused(const __grid_constant__ FusedArgs a)
{
    using C = FusedCfg<Q, R>;
    using SD = StreamDims<Q>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + C::BAR_OFF);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kFusedStreamWarps * C::S + 1; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp < kFusedStreamWarps) {
        // ---------------- stream warp: FIT / APPLY items ----------------
        Ring r;
        r.stage = reinterpret_cast<float*>(smem_raw) + (size_t)warp * C::WARP_FLOATS;
        r.full = bars + warp * C::S;
        r.S = C::S;
        r.STG = C::STG;
        float* mod = r.stage + C::S * C::STG;
        float* lerp = mod + 2 * kApplyNCol * SD::MS;
        const int step = gridDim.x * kFusedStreamWarps;
        FusedSeq<Q, D> seq;
        seq.a = &a;
        seq.it = blockIdx.x * kFusedStreamWarps + warp;
        seq.step = step;
        seq.pol_keep = policy_evict_last();
        seq.pol_once = policy_evict_first();
        seq.load();
        if (lane == 0) ring_fill(r, seq);
        for (int it = blockIdx.x * kFusedStreamWarps + warp;; it += step) {
            const StreamItem item = fused_decode(a, it);
            if (item.kind < 0) break;
            if (item.kind == 0) {
                fit_consume<Q, D>(r, seq, a.fit, item.f, item.row, item.sg, lane);
                __threadfence();
                __syncwarp();
                if (lane == 0) red_release_add(&a.fit_done[item.f * a.fit.By + item.row], 1);
            } else {
                apply_consume<Q>(r, seq, a.app, item.f, item.row, item.sg, lane, mod, lerp);
            }
        }
    } else {
        // ---------------- solver group: SOLVE tiles ----------------
        const int tid = threadIdx.x - kFusedStreamWarps * 32;
        const NamedSync gs{1, kFusedThreads - kFusedStreamWarps * 32};
        double* sm = reinterpret_cast<double*>(smem_raw + C::STREAM_BYTES);
        uint64_t* sbar = bars + kFusedStreamWarps * C::S;
        unsigned use = 0;
        const int per_frame = a.nrt * a.ncx, nitems = a.n * per_frame;
        const int By = a.fit.By, nseg = a.fit.nseg;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const int f = it / per_frame, rem = it - f * per_frame, m = rem / a.ncx, cx = rem - m * a.ncx;
            if (tid == 0) {  // moments of fit rows [4m - R, 4m + 3 + R]
                const int r0 = max(m * kTileTY - R, 0), r1 = min(m * kTileTY + kTileTY - 1 + R, By - 1);
                for (int rr = r0; rr <= r1; ++rr)
                    while (ld_acquire(&a.fit_done[f * By + rr]) < nseg) __nanosleep(128);
                asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> TMA reads
            }
            gs.sync();
#ifndef FLR_DBG_FAKE_SOLVE
            fused_blur_solve<Q, R>(&a.tmom, f, cx * kTileTX, m * kTileTY, a.fit.Bx, By,
                                   const_cast<float*>(a.app.models), SD::MS, a.eps_add, a.eps_mul, a.taps, sm, sbar,
                                   use, tid, gs);
#endif
            __threadfence();
            gs.sync();
            if (tid == 0) red_release_add(&a.solve_done[f * a.nrt + m], 1);
        }
    }
}

}  // namespace flr
