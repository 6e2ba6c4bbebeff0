// flr_inst.cu -- kernel launchers for ONE guide count Q = FLR_Q (compiled 15 times).
#ifndef FLR_Q
#error "compile with -DFLR_Q=<1..15>"
#endif
#include "flr_launch.h"
#include "flr_staged.cuh"
#include "flr_tiles.cuh"
#include "flr_persist.cuh"
#include "flr_k2.cuh"
#include "flr_fitws.cuh"
#include "flr_applyws.cuh"
#if FLR_Q == 4 || FLR_Q == 8
#include "flr_fused.cuh"
#endif
#include <algorithm>
#include <cstdlib>
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
bool launch_fused(const FusedLaunch&, LaunchCtx&)
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
    static const bool off = std::getenv("FLR_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

static int num_sms()
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// returns true when the TMA-ring kernel ran with `done` row counters (K2 may then wait per row)
template <int Q, int D>
static bool launch_k1(int n, int W, int H, int Bx, int By, const float* G, const float* Y, double* mom,
                      int* done, cudaStream_t s, const float* A, float afloor, bool hg, bool early)
{
    if (hg) {  // fp16 guide planes: the warp-specialised kernel with a half-width guide stage
        FitArgs a;
        std::memset(&a, 0, sizeof(a));
        if (!make_tmap_planes_f16(&a.tg, G, W, H, n * Q, kFS, Q) || !make_tmap_planes(&a.ty, Y, W, H, n * 3, kFS, 3))
            return false;
        a.mom = mom;
        a.W = W, a.H = H, a.Bx = Bx, a.Bxp = mom_pitch(Bx), a.By = By, a.nseg = cdiv(W, kFS);
        a.early = early;
        using C = FitWsCfg<Q, false, true>;
        const int grid = min(num_sms(), cdiv(n * By * a.nseg, C::NC));
        set_smem(k_fit_ws<Q, D, false, true>, C::SMEM);
        launch_pdl(k_fit_ws<Q, D, false, true>, dim3(grid), dim3(C::THREADS), C::SMEM, s, a, n);
        return false;
    }
    if (A) {  // modulated fit: the warp-specialised kernel with the albedo planes in its ring
        FitArgs a;
        if (!make_tmap_planes(&a.tg, G, W, H, n * Q, kFS, Q) || !make_tmap_planes(&a.ty, Y, W, H, n * 3, kFS, 3) ||
            !make_tmap_planes(&a.ta, A, W, H, n * 3, kFS, 3))
            return false;
        a.mom = mom;
        a.W = W, a.H = H, a.Bx = Bx, a.Bxp = mom_pitch(Bx), a.By = By, a.nseg = cdiv(W, kFS);
        a.done = nullptr;
        a.gpol = 0;
        a.afloor = afloor;
        a.early = early;
        using C = FitWsCfg<Q, true>;
        const int grid = min(num_sms(), cdiv(n * By * a.nseg, C::NC));
        set_smem(k_fit_ws<Q, D, true>, C::SMEM);
        launch_pdl(k_fit_ws<Q, D, true>, dim3(grid), dim3(C::THREADS), C::SMEM, s, a, n);
        return false;
    }
    static const bool use_ldg = std::getenv("FLR_FIT_LDG") != nullptr;
    if (use_ldg && vec_ok(G, W) && vec_ok(Y, W)) {  // LDG-prefetch persistent kernel (memory-latency bound)
        FitLdgArgs la{G, Y, mom, W, H, Bx, mom_pitch(Bx), By, cdiv(W, kSeg)};
        const int items = n * By * la.nseg;
        const int grid = min(num_sms(), cdiv(items, kFitLdgWarps));
        launch_pdl(k_fit_ldg<Q, D>, dim3(grid), dim3(kFitLdgWarps * 32), 0, s, la, n);
        return false;
    }
    FitArgs a;
    static const bool ring_env = std::getenv("FLR_FIT_RING") != nullptr;
    const int sw = ring_env ? kSeg : kFS;  // TMA box width = segment width of the kernel
    if (vec_ok(G, W) && vec_ok(Y, W) && make_tmap_planes(&a.tg, G, W, H, n * Q, sw, Q) &&
        make_tmap_planes(&a.ty, Y, W, H, n * 3, sw, 3)) {  // TMA-fed persistent path
        a.mom = mom;
        a.W = W, a.H = H, a.Bx = Bx, a.Bxp = mom_pitch(Bx), a.By = By, a.nseg = cdiv(W, sw);
        a.done = done;
        a.early = early && !std::getenv("FLR_FIT_RING");
        static const int gpol = std::getenv("FLR_FIT_GPOL") ? std::atoi(std::getenv("FLR_FIT_GPOL")) : 0;
        a.gpol = gpol;

        const int items = n * By * a.nseg;
        static const bool ring = std::getenv("FLR_FIT_RING") != nullptr;
        if (ring) {  // per-warp self-feeding rings (lane 0 of each warp issues its own TMA)
            using C = FitCfg<Q>;
            const int grid = min(num_sms(), cdiv(items, C::NSW));
            set_smem(k_fit_stream<Q, D>, C::SMEM);
            launch_pdl(k_fit_stream<Q, D>, dim3(grid), dim3(C::THREADS), C::SMEM, s, a, n);
        } else {  // default: warp-specialised (one producer warp feeds 7 consumer warps)
            using C = FitWsCfg<Q>;
            const int grid = min(num_sms(), cdiv(items, C::NC));
            set_smem(k_fit_ws<Q, D>, C::SMEM);
            launch_pdl(k_fit_ws<Q, D>, dim3(grid), dim3(C::THREADS), C::SMEM, s, a, n);
        }
        return done != nullptr;
    }
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
    return false;
}

template <int Q>
void launch_fit(int n, int W, int H, int D, int Bx, int By, const float* G, const float* Y,
                float* raw, double* mom, double* hb, float* models, int mstride, double ea,
                double em, const Taps& taps, LaunchCtx& ctx, const float* A, float afloor, bool hg)
{
    const cudaStream_t s = ctx.s;
    // wavefront flags: fit_done [n][By] | k2_done [n][ceil(By / kK2TY)]
    int* fit_done = ctx.wave_flags;
    int* k2_done = fit_done ? fit_done + (size_t)n * By : nullptr;
    if (fit_done) cudaMemsetAsync(fit_done, 0, sizeof(int) * (size_t)n * (By + cdiv(By, kK2TY)), s);
    ctx.wave_k2 = nullptr;
    bool fit_signals = false;
    const int fit_nseg = cdiv(W, std::getenv("FLR_FIT_RING") ? kSeg : kFS);  // FIT items per block row
    // K1: block moments (fp64, un-shifted) -> mom
    if (D >= 4) {
        ctx.before(hg ? "k_fit_ws_f16" : A ? "k_fit_ws_mod" : !vec_ok(G, W) || !vec_ok(Y, W) ? "k_fit_moments" : std::getenv("FLR_FIT_LDG") ? "k_fit_ldg" : std::getenv("FLR_FIT_RING") ? "k_fit_stream" : "k_fit_ws");
        if (D == 4) fit_signals = launch_k1<Q, 4>(n, W, H, Bx, By, G, Y, mom, fit_done, s, A, afloor, hg, ctx.early && !fit_done);
        else if (D == 8) fit_signals = launch_k1<Q, 8>(n, W, H, Bx, By, G, Y, mom, fit_done, s, A, afloor, hg, ctx.early && !fit_done);
        else fit_signals = launch_k1<Q, 16>(n, W, H, Bx, By, G, Y, mom, fit_done, s, A, afloor, hg, ctx.early && !fit_done);
    } else {
        ctx.before("k_moments_small");
        k_moments_small<Q><<<dim3(cdiv(Bx, 128), By, n), 128, 0, s>>>(W, H, Bx, By, D, G, Y, raw);
        ctx.before("k_unshift");
        const int nb = Bx * By;
        k_unshift<Q><<<dim3(cdiv(nb, 128), n), 128, 0, s>>>(Bx, mom_pitch(Bx), By, raw, mom);
    }
    // K2: blur (component-parallel, fp64) -> hb, then solve (thread per block) -> models
    CUtensorMap tm;
    const int Bxp = mom_pitch(Bx), R = taps.R;
    constexpr int NGRP = (Dims<Q>::KM + kBlurG - 1) / kBlurG;
    // K2 variants: default k_blur_solve_tile (32 x 8 tiles, TMA ring, flr_k2.cuh);
    // FLR_ROWS_SOLVE: row-strip blur -> blurred field -> row solve (two kernels);
    // FLR_TILE_SOLVE: the 32 x 4 tile kernel with in-register h-pass (flr_tiles.cuh)
    static const bool tile = std::getenv("FLR_TILE_SOLVE") != nullptr;
    static const bool rows = std::getenv("FLR_ROWS_SOLVE") != nullptr;
    (void)NGRP;
    bool k2tile = false;
    // the tile kernel keeps all KM blurred components of a block in registers: up to Q = 8
    // (KM = 72); larger Q take the row variant (components in shared memory)
    if constexpr (Q <= 8) {  // (not instantiated for larger Q: keeps the build time down)
    if (!tile && !rows && R >= 1 && R <= kTileMaxR && mstride == Dims<Q>::MSTRIDE) {
        // default: one tile kernel, moment field read once (+ halo) by TMA, no blurred-field
        // round trip through L2
        const dim3 grid(cdiv(Bx, kK2TX), cdiv(By, kK2TY), n);
        static const int k2pol = std::getenv("FLR_K2_POL") ? std::atoi(std::getenv("FLR_K2_POL")) : 1;
#define FLR_KT(RR)                                                                                          \
    case RR: {                                                                                              \
        using KG = K2Geom<Q, RR>;                                                                           \
        if (!make_tmap_3d(&tm, mom, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, Bx, By, Bxp, n * Dims<Q>::KM, KG::HX, \
                          KG::NV, KG::G))                                                                   \
            break;                                                                                          \
        ctx.before("k_blur_solve_tile");                                                                    \
        set_smem(k_blur_solve_tile<Q, RR>, KG::SMEM);                                                       \
        launch_pdl(k_blur_solve_tile<Q, RR>, grid, dim3(kK2Threads), KG::SMEM, s, tm, Bx, By, models, ea, em, \
                   taps, (const int*)(fit_signals ? fit_done : nullptr), fit_nseg, k2_done, k2pol);           \
        k2tile = true;                                                                                      \
        break;                                                                                              \
    }
        switch (R) { FLR_KT(1) FLR_KT(2) FLR_KT(3) FLR_KT(4) FLR_KT(5) FLR_KT(6) FLR_KT(7) FLR_KT(8) }
#undef FLR_KT
    }
    }
    if (k2tile) {
        if (k2_done) ctx.wave_k2 = k2_done, ctx.wave_nrt = cdiv(By, kK2TY), ctx.wave_target = cdiv(Bx, kK2TX);
    } else if (!tile && R >= 1 && R <= kTileMaxR && blur_rows_smem(Bx, R) <= 227 * 1024 &&
        (size_t)n * Dims<Q>::KM <= 65535) {
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
        if (mstride == Dims<Q>::MSTRIDE && !std::getenv("FLR_REG_SOLVE")) {
            ctx.before("k_solve_rows");
            set_smem(k_solve_rows<Q>, solve_rows_smem<Q>());
            launch_pdl(k_solve_rows<Q>, dim3(cdiv(Bx, kSolveRowN), By, n), dim3(kSolveRowN), solve_rows_smem<Q>(), s,
                       Bx, Bxp, By, (const double*)hb, models, ea, em);
        } else {
            ctx.before("k_solve");
            launch_pdl(k_solve<Q>, dim3(cdiv(Bx, 128), By, n), dim3(128), 0, s, Bx, Bxp, By, (const double*)hb,
                       models, mstride, ea, em);
        }
    } else if (Q <= 8 && R >= 1 && R <= kTileMaxR &&
        make_tmap_3d(&tm, mom, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, Bx, By, Bxp, n * Dims<Q>::KM, halo_x(R),
                     kTileTY + 2 * R, tile_g(R))) {
        ctx.before("k_blur_solve");
        const size_t sm = blur_solve_smem_bytes(taps.R);
        const dim3 grid(cdiv(Bx, kTileTX), cdiv(By, kTileTY), n), block(kTileTX * kTileTY);
#define FLR_K2(RR)                                                                                  \
    case RR:                                                                                        \
        set_smem(k_blur_solve<Q, RR>, sm);                                                          \
        launch_pdl(k_blur_solve<Q, RR>, grid, block, sm, s, tm, Bx, By, models, mstride, ea, em, taps); \
        break;
        if constexpr (Q <= 8) {
            switch (taps.R) { FLR_K2(1) FLR_K2(2) FLR_K2(3) FLR_K2(4) FLR_K2(5) FLR_K2(6) FLR_K2(7) FLR_K2(8) }
        }
#undef FLR_K2
    } else {
        ctx.before("k_hblur");
        const size_t rows = (size_t)n * Dims<Q>::KM * By;
        const unsigned gy = rows < 65535 ? (unsigned)rows : 65535u;
        const unsigned gz = (unsigned)((rows + gy - 1) / gy);
        k_hblur<<<dim3(cdiv(Bx, 64), gy, gz), 64, 0, s>>>(Bx, Bxp, rows, mom, hb, taps);
        ctx.before("k_vblur_solve");
        dim3 block(32, 4), grid(cdiv(Bx, 32), cdiv(By, 4), n);
        k_vblur_solve<Q><<<grid, block, 0, s>>>(Bx, Bxp, By, hb, models, mstride, ea, em, taps);
    }
}

template <int Q>
void launch_apply(int n, int W, int H, int D, int Bx, int By, const float* models, int mstride,
                  const float* G, float* out, LaunchCtx& ctx, const float* A, const float* Dl, bool hg)
{
    const cudaStream_t s = ctx.s;
    if (hg) {  // fp16 guide planes (caller checked half_guides_apply_ok)
        ApplyArgs a;
        std::memset(&a, 0, sizeof(a));
        if (mstride != Dims<Q>::MSTRIDE || !make_tmap_planes_f16(&a.tg, G, W, H, n * Q, kSeg, Q)) {
            ctx.unsupported = true;
            return;
        }
        a.models = models, a.out = out;
        a.W = W, a.H = H, a.D = D, a.Bx = Bx, a.By = By, a.nseg = cdiv(W, kSeg), a.nband = apply_nband(H, D, By);
        a.nsub = 1;
        while (D % (2 * a.nsub) == 0 && D / (2 * a.nsub) >= 4)
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
        if (mstride != Dims<Q>::MSTRIDE || !make_tmap_planes(&a.tg, G, W, H, n * Q, kSeg, Q) ||
            !make_tmap_planes(&a.ta, A, W, H, n * 3, kSeg, 3) ||
            (Dl && !make_tmap_planes(&a.td, Dl, W, H, n * 3, kSeg, 3))) {
            ctx.unsupported = true;
            return;
        }
        a.has_direct = Dl != nullptr;
        a.models = models, a.out = out;
        a.W = W, a.H = H, a.D = D, a.Bx = Bx, a.By = By, a.nseg = cdiv(W, kSeg), a.nband = apply_nband(H, D, By);
        a.nsub = 1;
        while (D % (2 * a.nsub) == 0 && D / (2 * a.nsub) >= 4)
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
        if (vec_ok(G, W) && vec_ok(out, W) && make_tmap_planes(&a.tg, G, W, H, n * Q, kSeg, Q)) {  // TMA path
            a.models = models, a.out = out;
            a.W = W, a.H = H, a.D = D, a.Bx = Bx, a.By = By, a.nseg = cdiv(W, kSeg), a.nband = apply_nband(H, D, By);
            using C = ApplyCfg<Q>;
            // sub-bands of >= 4 rows: finer items balance the warps (a single 1080p frame
            // otherwise leaves most warps with 1 item and some with 2; measured 28 -> 25 us)
            a.nsub = 1;
            while (D % (2 * a.nsub) == 0 && D / (2 * a.nsub) >= 4)
                a.nsub *= 2;
            if (const char* e = std::getenv("FLR_APPLY_NSUB")) a.nsub = std::max(1, std::atoi(e));
            if (D % a.nsub) a.nsub = 1;
            static const int rev = std::getenv("FLR_APPLY_REV") ? std::atoi(std::getenv("FLR_APPLY_REV")) : 1;
            a.reverse = rev;
            a.ready = ctx.wave_k2, a.ready_target = ctx.wave_target, a.nrt = ctx.wave_nrt, a.ready_ty = kK2TY;
            ctx.wave_k2 = nullptr;
            const int items = n * a.nseg * a.nband * a.nsub;
            // many items (batches): the 11-warp self-feeding rings keep more rows in flight;
            // few items (one frame): the warp-specialised kernel's faster items win
            // (measured 1080p: 1 frame 22.6 vs 26.6 us, 8 frames 17.8 vs 16.2 us per frame)
            static const char* env = std::getenv("FLR_APPLY_RING");
            const bool ring = env ? env[0] == '1' : items >= 4 * num_sms() * ApplyCfg<Q>::NSW;
            if (ring || a.ready) {  // per-warp self-feeding rings (supports the row wavefront)
                using C = ApplyCfg<Q>;
                const int grid = min(num_sms(), cdiv(items, C::NSW));
                ctx.before("k_apply_stream");
                set_smem(k_apply_stream<Q>, C::SMEM);
                launch_pdl(k_apply_stream<Q>, dim3(grid), dim3(C::THREADS), C::SMEM, s, a, n);
            } else {  // default: warp-specialised (one producer warp feeds 7 consumer warps)
                using C = ApplyWsCfg<Q>;
                const int grid = min(num_sms(), cdiv(items, C::NC));
                ctx.before("k_apply_ws");
                set_smem(k_apply_ws<Q>, C::SMEM);
                launch_pdl(k_apply_ws<Q>, dim3(grid), dim3(C::THREADS), C::SMEM, s, a, n);
            }
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
bool launch_fused(const FusedLaunch& L, LaunchCtx& ctx)
{
#if FLR_Q == 4 || FLR_Q == 8
    const int Dout = L.D * L.U, R = L.taps.R;
    const int Wo = L.W * L.U, Ho = L.H * L.U;
    if (!(L.D == 4 || L.D == 8) || Dout % 8 || !(R == 3 || R == 5)) return false;
    if (!vec_ok(L.G, L.W) || !vec_ok(L.Y, L.W) || !vec_ok(L.Gout, Wo) || !vec_ok(L.out, Wo)) return false;
    FusedArgs a;
    std::memset(&a, 0, sizeof(a));
    const int Bxp = mom_pitch(L.Bx);
    if (!make_tmap_planes(&a.fit.tg, L.G, L.W, L.H, L.n * Q, kSeg, Q) ||
        !make_tmap_planes(&a.fit.ty, L.Y, L.W, L.H, L.n * 3, kSeg, 3) ||
        !make_tmap_planes(&a.app.tg, L.Gout, Wo, Ho, L.n * Q, kSeg, Q) ||
        !make_tmap_3d(&a.tmom, L.mom, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, L.Bx, L.By, Bxp, L.n * Dims<Q>::KM,
                      halo_x(R), kTileTY + 2 * R, kFusedG))
        return false;
    a.fit.mom = L.mom;
    a.fit.W = L.W, a.fit.H = L.H, a.fit.Bx = L.Bx, a.fit.Bxp = Bxp, a.fit.By = L.By, a.fit.nseg = cdiv(L.W, kSeg);
    a.app.models = L.models, a.app.out = L.out;
    a.app.W = Wo, a.app.H = Ho, a.app.D = Dout, a.app.Bx = L.Bx, a.app.By = L.By;
    a.app.nseg = cdiv(Wo, kSeg), a.app.nband = apply_nband(Ho, Dout, L.By), a.app.nsub = 1;
    a.taps = L.taps;
    a.nrt = cdiv(L.By, kTileTY), a.ncx = cdiv(L.Bx, kTileTX);
    a.fit_done = L.flags;
    a.solve_done = L.flags + L.n * L.By;
    a.n = L.n;
    int lag = 32 + R;  // block rows between a FIT and the APPLY that reuses its guides (tunable)
    if (const char* e = std::getenv("FLR_FUSED_LAG")) lag = std::max(R + kTileTY + 1, std::atoi(e));
    a.lag = lag;
    a.eps_add = L.eps_add, a.eps_mul = L.eps_mul;
    cudaMemsetAsync(L.flags, 0, sizeof(int) * (size_t)L.n * (L.By + a.nrt), ctx.s);

    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3(num_sms());
    cfg.blockDim = dim3(kFusedThreads);
    cfg.stream = ctx.s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#define FLR_FUSED(DD, RR)                                                                        \
    if (L.D == DD && R == RR) {                                                                  \
        using C = FusedCfg<Q, RR>;                                                               \
        cfg.dynamicSmemBytes = C::SMEM;                                                          \
        set_smem(k_flr_fused<Q, DD, RR>, C::SMEM);                                               \
        ctx.before("k_flr_fused");                                                               \
        cudaLaunchKernelEx(&cfg, k_flr_fused<Q, DD, RR>, a);                                     \
        return true;                                                                             \
    }
    FLR_FUSED(4, 3) FLR_FUSED(4, 5) FLR_FUSED(8, 3) FLR_FUSED(8, 5)
#undef FLR_FUSED
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
template bool launch_fused<FLR_Q>(const FusedLaunch&, LaunchCtx&);
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

}  // namespace flr
