// flr_inst.cu -- kernel launchers for ONE guide count Q = FLR_Q (compiled 15 times).
#ifndef FLR_Q
#error "compile with -DFLR_Q=<1..15>"
#endif
#include "flr_launch.h"
#include "flr_staged.cuh"
#include "flr_tiles.cuh"
#include "flr_k2.cuh"
#include "flr_fitws.cuh"
#include "flr_applyws.cuh"
#if FLR_Q == 4 || FLR_Q == 8
#include "flr_wave.cuh"
#endif
#include <algorithm>
#include <cstring>

namespace flr {

#ifdef FLR_STUB
// dev build: this Q is compiled out (see build.py FLR_QS); calls report FLR_ERR_UNSUPPORTED
template <int Q>
void launch_fit(int, int, int, int, int, int, const float*, const float*, float*, double*, double*, float*,
                int, double, double, const Taps&, LaunchCtx& ctx, const float*, float, bool)
{
    ctx.unsupported = true;
}
template <int Q>
void launch_apply(int, int, int, int, int, int, const float*, int, const float*, float*, LaunchCtx& ctx,
                  const float*, const float*, bool)
{
    ctx.unsupported = true;
}
template <int Q>
bool launch_wave(const WaveLaunch&, LaunchCtx&)
{
    return false;
}
#else
template <class K>
static void set_smem(K kernel, size_t bytes)
{
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// launch with programmatic stream serialization (PDL): the grid may start while the
// previous grid in the stream drains; kernels call pdl_wait() before touching its output
template <class... KArgs, class... Args>
static void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

static int num_sms()
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

#ifndef FLR_APPLY_SUB_ROWS
#define FLR_APPLY_SUB_ROWS 8
#endif
// fewest output rows of an APPLY item (items = sub-bands of a block row of models): whole
// 8-row bands at D = 8 halve the per-item model copies and producer operations (C2 44.15 vs
// 44.5 us per frame with 4-row items; the per-SM apply rate 61 vs 51 GB/s at 37 SMs)
constexpr int kApplySubRows = FLR_APPLY_SUB_ROWS;

// K1: the warp-specialised TMA kernel when the planes allow it, else the tiled kernel
template <int Q, int D>
static void launch_k1(int n, int W, int H, int Bx, int By, const float* G, const float* Y, double* mom,
                      cudaStream_t s, const float* A, float afloor, bool hg, bool early, bool acc64, bool keep)
{
    FitArgs a;
    std::memset(&a, 0, sizeof(a));
    a.mom = mom;
    a.W = W, a.H = H, a.Bx = Bx, a.Bxp = mom_pitch(Bx), a.By = By, a.nseg = cdiv(W, kFS);
    a.afloor = afloor;
    a.early = early;
    // keep: the apply of this call re-reads these guides; the bottom kGuideL2Rows bytes of them
    // (one frame) stay in L2 for the bottom-up apply.  C2 (66 MB of guides): all rows
    // evict_normal 42.9 vs 43.55 us per frame (apply -2.8 us; the fit streams next to more
    // dirty lines: +2.2 us), the bottom 3/4 (= 50 MB) 42.1; lo-res (C4) and batched guides
    // stream with evict_first
    const size_t row_bytes = (size_t)Q * W * (hg ? 2 : 4);
    a.keep_y0 = keep && n == 1 ? H - (int)std::min<size_t>((size_t)H, kGuideL2Rows / row_bytes) : H;
    const int items = n * By * a.nseg;
    if (hg) {  // fp16 guide planes: the warp-specialised kernel with a half-width guide stage
        using C = FitWsCfg<Q, false, true>;
        if (!make_tmap_planes_f16(&a.tg, G, W, H, n * Q, kFS, Q, C::RB) ||
            !make_tmap_planes(&a.ty, Y, W, H, n * 3, kFS, 3, C::RB))
            return;
        set_smem(k_fit_ws<Q, D, false, true>, C::SMEM);
        launch_pdl(k_fit_ws<Q, D, false, true>, dim3(min(num_sms(), cdiv(items, C::NC))), dim3(C::THREADS), C::SMEM, s,
                   a, n);
        return;
    }
    if (A) {  // modulated fit: the warp-specialised kernel with the albedo planes in its ring
        using C = FitWsCfg<Q, true>;
        if (!make_tmap_planes(&a.tg, G, W, H, n * Q, kFS, Q, C::RB) ||
            !make_tmap_planes(&a.ty, Y, W, H, n * 3, kFS, 3, C::RB) || !make_tmap_planes(&a.ta, A, W, H, n * 3, kFS, 3, C::RB))
            return;
        set_smem(k_fit_ws<Q, D, true>, C::SMEM);
        launch_pdl(k_fit_ws<Q, D, true>, dim3(min(num_sms(), cdiv(items, C::NC))), dim3(C::THREADS), C::SMEM, s, a, n);
        return;
    }
    using CF = FitWsCfg<Q>;
    if (vec_ok(G, W) && vec_ok(Y, W) && make_tmap_planes(&a.tg, G, W, H, n * Q, kFS, Q, CF::RB) &&
        make_tmap_planes(&a.ty, Y, W, H, n * 3, kFS, 3, CF::RB)) {  // default: one producer warp feeds 7 consumers
        using C = CF;
        const dim3 grid(min(num_sms(), cdiv(items, C::NC)));
        if (acc64) {  // Tikhonov mode: fp64 accumulation (FitAcc64)
            set_smem(k_fit_ws<Q, D, false, false, true>, C::SMEM);
            launch_pdl(k_fit_ws<Q, D, false, false, true>, grid, dim3(C::THREADS), C::SMEM, s, a, n);
            return;
        }
        set_smem(k_fit_ws<Q, D>, C::SMEM);
        launch_pdl(k_fit_ws<Q, D>, grid, dim3(C::THREADS), C::SMEM, s, a, n);
        return;
    }
    // unaligned planes or W % 4 != 0: the tiled kernel (scalar tails)
    const size_t sm = fit_smem_bytes<Q, D>();
    dim3 grid(cdiv(W, 128), By, n), block(FitGeom<D>::THREADS);
    const int Bxp = mom_pitch(Bx);
    if (vec_ok(G, W) && vec_ok(Y, W)) {
        set_smem(k_fit_moments<Q, D, true>, sm);
        k_fit_moments<Q, D, true><<<grid, block, sm, s>>>(W, H, Bx, Bxp, By, G, Y, mom);
    } else {
        set_smem(k_fit_moments<Q, D, false>, sm);
        k_fit_moments<Q, D, false><<<grid, block, sm, s>>>(W, H, Bx, Bxp, By, G, Y, mom);
    }
}

template <int Q>
void launch_fit(int n, int W, int H, int D, int Bx, int By, const float* G, const float* Y,
                float* raw, double* mom, double* hb, float* models, int mstride, double ea,
                double em, const Taps& taps, LaunchCtx& ctx, const float* A, float afloor, bool hg)
{
    const cudaStream_t s = ctx.s;
    ctx.l2_guides = ctx.keep_guides && !hg && (size_t)n * Q * W * H * 4 <= kGuideL2Keep;
    // K1: block moments (fp64, un-shifted) -> mom
    if (D >= 4) {
        ctx.before(hg ? "k_fit_ws_f16" : A ? "k_fit_ws_mod" : !vec_ok(G, W) || !vec_ok(Y, W) ? "k_fit_moments"
                   : em < 0.0 ? "k_fit_ws_f64acc" : "k_fit_ws");
        const bool acc64 = em < 0.0 && !hg && !A;  // Tikhonov mode (flr_solve.cuh sentinels)
        const bool keep = ctx.keep_guides;
        if (D == 4) launch_k1<Q, 4>(n, W, H, Bx, By, G, Y, mom, s, A, afloor, hg, ctx.early, acc64, keep);
        else if (D == 8) launch_k1<Q, 8>(n, W, H, Bx, By, G, Y, mom, s, A, afloor, hg, ctx.early, acc64, keep);
        else launch_k1<Q, 16>(n, W, H, Bx, By, G, Y, mom, s, A, afloor, hg, ctx.early, acc64, keep);
    } else {
        ctx.before("k_moments_small");
        k_moments_small<Q><<<dim3(cdiv(Bx, 128), By, n), 128, 0, s>>>(W, H, Bx, By, D, G, Y, raw);
        ctx.before("k_unshift");
        const int nb = Bx * By;
        k_unshift<Q><<<dim3(cdiv(nb, 128), n), 128, 0, s>>>(Bx, mom_pitch(Bx), By, raw, mom);
    }
    // K2: blur + solve -> models
    CUtensorMap tm;
    const int Bxp = mom_pitch(Bx), R = taps.R;
    // default (Q <= 8, R <= 8): one 32 x 8 tile kernel, the moment field read once (+ halo)
    // by TMA, no blurred-field round trip through L2 (flr_k2.cuh).  The tile kernel keeps
    // all KM blurred components of a block in registers, so larger Q take the row variant.
    if constexpr (Q <= 8) {
        // (the tile stages MSTRIDE floats per block and zero-pads past the raw model, so the
        // centred Tikhonov layout takes the row variant)
        if (R >= 1 && R <= kTileMaxR && mstride <= Dims<Q>::MSTRIDE && !tikhonov_centered(em)) {
            const dim3 grid(cdiv(Bx, kK2TX), cdiv(By, kK2TY), n);
            bool ok = false;
#define FLR_KT(RR)                                                                                          \
    case RR: {                                                                                              \
        using KG = K2WsGeom<Q, RR>;                                                                         \
        if (!make_tmap_3d(&tm, mom, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, Bx, By, Bxp, n * Dims<Q>::KM, KG::HX, \
                          KG::NVB, KG::G))                                                                   \
            break;                                                                                          \
        ctx.before("k_blur_solve_tile");                                                                    \
        set_smem(k_blur_solve_tile<Q, RR>, KG::SMEM);                                                       \
        launch_pdl(k_blur_solve_tile<Q, RR>, grid, dim3(kK2WsThreads), KG::SMEM, s, tm, Bx, By, models, mstride, \
                   ea, em, taps);                                                                  \
        ok = true;                                                                                          \
        break;                                                                                              \
    }
            switch (R) { FLR_KT(1) FLR_KT(2) FLR_KT(3) FLR_KT(4) FLR_KT(5) FLR_KT(6) FLR_KT(7) FLR_KT(8) }
#undef FLR_KT
            if (ok) return;
        }
    }
    if (R >= 1 && R <= kTileMaxR && blur_rows_smem(Bx, R) <= 227 * 1024 && (size_t)n * Dims<Q>::KM <= 65535) {
        // row-strip blur -> blurred field (hb) -> per-block solve
        ctx.before("k_blur_rows");
        const size_t sm = blur_rows_smem(Bx, R);
        const dim3 grid(cdiv(By, kRowsCH), n * Dims<Q>::KM);
#define FLR_KB(RR)                                                                                          \
    case RR:                                                                                                \
        set_smem(k_blur_rows<RR>, sm);                                                                      \
        launch_pdl(k_blur_rows<RR>, grid, dim3(kRowsThreads), sm, s, (const double*)mom, Bx, Bxp, By, hb, taps); \
        break;
        switch (R) { FLR_KB(1) FLR_KB(2) FLR_KB(3) FLR_KB(4) FLR_KB(5) FLR_KB(6) FLR_KB(7) FLR_KB(8) }
#undef FLR_KB
        if (mstride == Dims<Q>::MSTRIDE && aligned(models, 16) && !tikhonov_centered(em)) {
            ctx.before("k_solve_rows");
            set_smem(k_solve_rows<Q>, solve_rows_smem<Q>());
            launch_pdl(k_solve_rows<Q>, dim3(cdiv(Bx, kSolveRowN), By, n), dim3(kSolveRowN), solve_rows_smem<Q>(), s,
                       Bx, Bxp, By, (const double*)hb, models, ea, em);
        } else {
            ctx.before("k_solve");
            launch_pdl(k_solve<Q>, dim3(cdiv(Bx, 128), By, n), dim3(128), 0, s, Bx, Bxp, By, (const double*)hb,
                       models, mstride, ea, em);
        }
        return;
    }
    // wide windows (R > 8) or very wide rows: plain two-pass blur
    ctx.before("k_hblur");
    const size_t rows = (size_t)n * Dims<Q>::KM * By;
    const unsigned gy = rows < 65535 ? (unsigned)rows : 65535u;
    const unsigned gz = (unsigned)((rows + gy - 1) / gy);
    k_hblur<<<dim3(cdiv(Bx, 64), gy, gz), 64, 0, s>>>(Bx, Bxp, rows, mom, hb, taps);
    ctx.before("k_vblur_solve");
    dim3 block(32, 4), grid(cdiv(Bx, 32), cdiv(By, 4), n);
    k_vblur_solve<Q><<<grid, block, 0, s>>>(Bx, Bxp, By, hb, models, mstride, ea, em, taps);
}

template <int Q>
void launch_apply(int n, int W, int H, int D, int Bx, int By, const float* models, int mstride,
                  const float* G, float* out, LaunchCtx& ctx, const float* A, const float* Dl, bool hg)
{
    const cudaStream_t s = ctx.s;
    if (hg) {  // fp16 guide planes (caller checked half_guides_apply_ok)
        ApplyArgs a;
        std::memset(&a, 0, sizeof(a));
        if (mstride != Dims<Q>::MSTRIDE || !make_tmap_planes_f16(&a.tg, G, W, H, n * Q, kSeg, Q, ApplyWsCfg<Q, false, true>::RB)) {
            ctx.unsupported = true;
            return;
        }
        a.models = models, a.out = out;
        a.W = W, a.H = H, a.D = D, a.Bx = Bx, a.By = By, a.nseg = cdiv(W, kSeg), a.nband = apply_nband(H, D, By);
        a.nsub = 1;
        while (D % (2 * a.nsub) == 0 && D / (2 * a.nsub) >= kApplySubRows)
            a.nsub *= 2;
        a.reverse = 1;
        using C = ApplyWsCfg<Q, false, true>;
        const int items = n * a.nseg * a.nband * a.nsub;
        const int grid = min(num_sms(), cdiv(items, C::NC));
        ctx.before("k_apply_ws_f16");
        set_smem(k_apply_ws<Q, false, true>, C::SMEM);
        launch_pdl(k_apply_ws<Q, false, true>, dim3(grid), dim3(C::THREADS), C::SMEM, s, a, n);
        return;
    }
    if constexpr (!ApplyWsCfg<Q, true>::FITS) {
        if (A) {
            ctx.unsupported = true;
            return;
        }
    } else if (A) {  // modulated apply (caller checked apply_mod_fused): warp-specialised kernel only
        ApplyArgs a;
        std::memset(&a, 0, sizeof(a));
        constexpr int RB = ApplyWsCfg<Q, true>::RB;
        if (mstride != Dims<Q>::MSTRIDE || !make_tmap_planes(&a.tg, G, W, H, n * Q, kSeg, Q, RB) ||
            !make_tmap_planes(&a.ta, A, W, H, n * 3, kSeg, 3, RB) ||
            (Dl && !make_tmap_planes(&a.td, Dl, W, H, n * 3, kSeg, 3, RB))) {
            ctx.unsupported = true;
            return;
        }
        a.has_direct = Dl != nullptr;
        a.models = models, a.out = out;
        a.W = W, a.H = H, a.D = D, a.Bx = Bx, a.By = By, a.nseg = cdiv(W, kSeg), a.nband = apply_nband(H, D, By);
        a.nsub = 1;
        while (D % (2 * a.nsub) == 0 && D / (2 * a.nsub) >= kApplySubRows)
            a.nsub *= 2;
        a.reverse = 1;
        using C = ApplyWsCfg<Q, true>;
        const int items = n * a.nseg * a.nband * a.nsub;
        const int grid = min(num_sms(), cdiv(items, C::NC));
        ctx.before("k_apply_ws_mod");
        set_smem(k_apply_ws<Q, true>, C::SMEM);
        launch_pdl(k_apply_ws<Q, true>, dim3(grid), dim3(C::THREADS), C::SMEM, s, a, n);
        return;
    }
    if (D % 8 == 0 && mstride == Dims<Q>::MSTRIDE && aligned(models, 16)) {
        const int off = (D / 2) % 8;
        ApplyArgs a;
        int nsub = 1;  // sub-bands of >= kApplySubRows rows (finer items balance the warps of one frame)
        while (D % (2 * nsub) == 0 && D / (2 * nsub) >= kApplySubRows)
            nsub *= 2;
        if (vec_ok(G, W) && vec_ok(out, W) &&
            make_tmap_planes(&a.tg, G, W, H, n * Q, kSeg, Q, ApplyWsCfg<Q>::RB)) {  // TMA path
            a.models = models, a.out = out;
            a.W = W, a.H = H, a.D = D, a.Bx = Bx, a.By = By, a.nseg = cdiv(W, kSeg), a.nband = apply_nband(H, D, By);
            a.nsub = nsub;
            a.reverse = 1;  // bottom-up: the fit's last rows are the likeliest still in L2
            const int items = n * a.nseg * a.nband * a.nsub;
            // warp-specialised (one producer warp feeds 7 consumer warps, 2-row stages); faster
            // than per-warp self-feeding rings for one frame and for batches alike
            auto go = [&](auto deep) {
                constexpr bool DEEP = decltype(deep)::value;
                using C = ApplyWsCfg<Q, false, false, DEEP>;
                const int grid = min(num_sms(), cdiv(items, C::NC));
                ctx.before("k_apply_ws");
                set_smem(k_apply_ws<Q, false, false, DEEP>, C::SMEM);
                launch_pdl(k_apply_ws<Q, false, false, DEEP>, dim3(grid), dim3(C::THREADS), C::SMEM, s, a, n);
            };
            // (the deep ring only where its stages hold as many rows as the default's: one map)
            if constexpr (ApplyWsCfg<Q, false, false, true>::RB == ApplyWsCfg<Q>::RB) {
                if (ctx.l2_guides) {
                    go(std::true_type{});
                    return;
                }
            }
            go(std::false_type{});
            return;
        }
        dim3 grid(cdiv(cdiv(W + off, 8), kApplyUnits), cdiv(H + off, kApplyRows), n),
            block(kApplyUnits * kApplyRows);
        ctx.before("k_apply_tile");
        if (vec_ok(G, W) && vec_ok(out, W))
            k_apply_tile<Q, true><<<grid, block, 0, s>>>(W, H, D, Bx, By, models, G, out);
        else
            k_apply_tile<Q, false><<<grid, block, 0, s>>>(W, H, D, Bx, By, models, G, out);
    } else {
        dim3 grid(cdiv(W, 128), H, n), block(128);
        ctx.before("k_apply_px");
        k_apply_px<Q><<<grid, block, 0, s>>>(W, H, D, Bx, By, models, mstride, G, out);
    }
}
template <int Q>
bool launch_wave(const WaveLaunch& L, LaunchCtx& ctx)
{
#if FLR_Q == 4 || FLR_Q == 8
    const int Dout = L.D * L.U, R = L.taps.R;
    const int Wo = L.W * L.U, Ho = L.H * L.U;
    if (!(L.D == 4 || L.D == 8) || Dout % 8 || !(R == 3 || R == 5)) return false;
    if (!vec_ok(L.G, L.W) || !vec_ok(L.Y, L.W) || !vec_ok(L.Gout, Wo) || !vec_ok(L.out, Wo) || !aligned(L.models, 16))
        return false;
    if ((size_t)L.n * L.By * cdiv(L.W, kFS) >= (1u << 30)) return false;
    WaveArgs w;
    std::memset(&w, 0, sizeof(w));
    const int Bxp = mom_pitch(L.Bx);
    if (!make_tmap_planes(&w.fit.tg, L.G, L.W, L.H, L.n * Q, kFS, Q, 2) ||
        !make_tmap_planes(&w.fit.ty, L.Y, L.W, L.H, L.n * 3, kFS, 3, 2) ||
        !make_tmap_planes(&w.app.tg, L.Gout, Wo, Ho, L.n * Q, kSeg, Q, 2))
        return false;
    auto tmom = [&](auto KGv) {
        using KG = decltype(KGv);
        return make_tmap_3d(&w.tmom, L.mom, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, L.Bx, L.By, Bxp, L.n * Dims<Q>::KM, KG::HX,
                            KG::NVB, KG::G);
    };
    if (!(R == 3 ? tmom(K2Geom<Q, 3>{}) : tmom(K2Geom<Q, 5>{}))) return false;
    w.fit.mom = L.mom;
    w.fit.W = L.W, w.fit.H = L.H, w.fit.Bx = L.Bx, w.fit.Bxp = Bxp, w.fit.By = L.By, w.fit.nseg = cdiv(L.W, kFS);
    w.app.models = L.models, w.app.out = L.out;
    w.app.W = Wo, w.app.H = Ho, w.app.D = Dout, w.app.Bx = L.Bx, w.app.By = L.By;
    w.app.nseg = cdiv(Wo, kSeg), w.app.nband = apply_nband(Ho, Dout, L.By);
    w.app.nsub = 1;
    while (Dout % (2 * w.app.nsub) == 0 && Dout / (2 * w.app.nsub) >= 4)
        w.app.nsub *= 2;
    w.taps = L.taps;
    w.eps_add = L.eps_add, w.eps_mul = L.eps_mul;
    w.n = L.n;
    w.nfit = L.n * L.By * w.fit.nseg, w.nfc = cdiv(w.nfit, kWaveNC);
    w.napp = L.n * w.app.nband * w.app.nsub * w.app.nseg;
    w.ntr = cdiv(L.By, kK2TY), w.ntc = cdiv(L.Bx, kK2TX);
    w.flags = L.flags;
    // the queue heads and row counters start at zero.  The kernel is launched WITHOUT
    // programmatic dependent launch: a PDL launch may overlap the preceding kernel across
    // this memset (in a graph the memset then races the running kernel)
    cudaMemsetAsync(L.flags, 0, sizeof(int) * (size_t)wave_flags_ints(L.n, L.By), ctx.s);
#define FLR_WAVE_L(DD, RR)                                                                        \
    if (L.D == DD && R == RR) {                                                                   \
        using C = WaveCfg<Q, RR>;                                                                 \
        set_smem(k_flr_wave<Q, DD, RR>, C::SMEM);                                                 \
        ctx.before("k_flr_wave");                                                                 \
        k_flr_wave<Q, DD, RR><<<dim3(num_sms()), dim3(C::THREADS), C::SMEM, ctx.s>>>(w);           \
        return true;                                                                              \
    }
    FLR_WAVE_L(4, 3) FLR_WAVE_L(4, 5) FLR_WAVE_L(8, 3) FLR_WAVE_L(8, 5)
#undef FLR_WAVE_L
    return false;
#else
    (void)L;
    (void)ctx;
    return false;
#endif
}

#endif  // FLR_STUB

template void launch_fit<FLR_Q>(int, int, int, int, int, int, const float*, const float*, float*,
                                double*, double*, float*, int, double, double, const Taps&,
                                LaunchCtx&, const float*, float, bool);
template void launch_apply<FLR_Q>(int, int, int, int, int, int, const float*, int, const float*,
                                  float*, LaunchCtx&, const float*, const float*, bool);
template <int Q>
bool apply_mod_supported()
{
#ifdef FLR_STUB
    return false;
#else
    return ApplyWsCfg<Q, true>::FITS;
#endif
}
template bool apply_mod_supported<FLR_Q>();
template bool launch_wave<FLR_Q>(const WaveLaunch&, LaunchCtx&);

}  // namespace flr
