// flr_inst.cu -- kernel launchers for ONE guide count Q = FLR_Q (compiled 15 times).
#ifndef FLR_Q
#error "compile with -DFLR_Q=<1..15>"
#endif
#include "flr_launch.h"
#include "flr_staged.cuh"
#include "flr_tiles.cuh"
#include "flr_persist.cuh"

namespace flr {

#ifdef FLR_STUB
// dev build: this Q is compiled out (see build.py FLR_QS); calls report FLR_ERR_UNSUPPORTED
template <int Q>
void launch_fit(int, int, int, int, int, int, const float*, const float*, float*, double*, double*, float*,
                int, double, double, const Taps&, LaunchCtx& ctx)
{
    ctx.unsupported = true;
}
template <int Q>
void launch_apply(int, int, int, int, int, int, const float*, int, const float*, float*, LaunchCtx& ctx)
{
    ctx.unsupported = true;
}
#else
template <class K>
static void set_smem(K kernel, size_t bytes)
{
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static int num_sms()
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

template <int Q, int D>
static void launch_k1(int n, int W, int H, int Bx, int By, const float* G, const float* Y, double* mom,
                      cudaStream_t s)
{
    FitArgs a;
    if (vec_ok(G, W) && vec_ok(Y, W) && make_tmap_planes(&a.tg, G, W, H, n * Q, kSeg, Q) &&
        make_tmap_planes(&a.ty, Y, W, H, n * 3, kSeg, 3)) {  // TMA-fed persistent path
        a.mom = mom;
        a.W = W, a.H = H, a.Bx = Bx, a.Bxp = mom_pitch(Bx), a.By = By, a.nseg = cdiv(W, kSeg);
        using C = FitCfg<Q>;
        const int items = n * By * a.nseg;
        const int grid = min(num_sms(), cdiv(items, C::NSW));
        set_smem(k_fit_stream<Q, D>, C::SMEM);
        k_fit_stream<Q, D><<<grid, C::THREADS, C::SMEM, s>>>(a, n);
        return;
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
}

template <int Q>
void launch_fit(int n, int W, int H, int D, int Bx, int By, const float* G, const float* Y,
                float* raw, double* mom, double* hb, float* models, int mstride, double ea,
                double em, const Taps& taps, LaunchCtx& ctx)
{
    const cudaStream_t s = ctx.s;
    // K1: block moments (fp64, un-shifted) -> mom
    if (D >= 4) {
        ctx.before(vec_ok(G, W) && vec_ok(Y, W) ? "k_fit_stream" : "k_fit_moments");
        if (D == 4) launch_k1<Q, 4>(n, W, H, Bx, By, G, Y, mom, s);
        else if (D == 8) launch_k1<Q, 8>(n, W, H, Bx, By, G, Y, mom, s);
        else launch_k1<Q, 16>(n, W, H, Bx, By, G, Y, mom, s);
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
    if (R >= 1 && R <= kTileMaxR &&
        make_tmap_3d(&tm, mom, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, Bx, By, Bxp, n * Dims<Q>::KM, halo_x(R),
                     kTileTY + 2 * R, kTileG)) {
        ctx.before("k_blur_solve");
        const size_t sm = blur_solve_smem_bytes(taps.R);
        const dim3 grid(cdiv(Bx, kTileTX), cdiv(By, kTileTY), n), block(kTileTX * kTileTY);
#define FLR_K2(RR)                                                                                  \
    case RR:                                                                                        \
        set_smem(k_blur_solve<Q, RR>, sm);                                                          \
        k_blur_solve<Q, RR><<<grid, block, sm, s>>>(tm, Bx, By, models, mstride, ea, em, taps);      \
        break;
        switch (taps.R) { FLR_K2(1) FLR_K2(2) FLR_K2(3) FLR_K2(4) FLR_K2(5) FLR_K2(6) FLR_K2(7) FLR_K2(8) }
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
                  const float* G, float* out, LaunchCtx& ctx)
{
    const cudaStream_t s = ctx.s;
    if (D % 8 == 0 && mstride == Dims<Q>::MSTRIDE && aligned(models, 16)) {
        const int off = (D / 2) % 8;
        ApplyArgs a;
        if (vec_ok(G, W) && vec_ok(out, W) && make_tmap_planes(&a.tg, G, W, H, n * Q, kSeg, Q)) {  // TMA path
            a.models = models, a.out = out;
            a.W = W, a.H = H, a.D = D, a.Bx = Bx, a.By = By, a.nseg = cdiv(W + off, kSeg), a.ntile = cdiv(H + off, 8);
            using C = ApplyCfg<Q>;
            const int items = n * a.nseg * a.ntile;
            const int grid = min(num_sms(), cdiv(items, C::NSW));
            ctx.before("k_apply_stream");
            set_smem(k_apply_stream<Q>, C::SMEM);
            k_apply_stream<Q><<<grid, C::THREADS, C::SMEM, s>>>(a, n);
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

#endif  // FLR_STUB

template void launch_fit<FLR_Q>(int, int, int, int, int, int, const float*, const float*, float*,
                                double*, double*, float*, int, double, double, const Taps&,
                                LaunchCtx&);
template void launch_apply<FLR_Q>(int, int, int, int, int, int, const float*, int, const float*,
                                  float*, LaunchCtx&);

}  // namespace flr
