// flr_api.cu -- the C ABI of libflr.so (declared in include/flr.h): argument
// validation, workspace carving, Gaussian taps, and kernel launches on the
// caller's stream.  No allocation, no synchronisation, no host<->device copies.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/flr.h"
#include "flr_common.cuh"
#include "flr_launch.h"
#include "flr_solve.cuh"
#include "flr_staged.cuh"

using namespace flr;

namespace {

thread_local int32_t g_last_launches = 0;
thread_local const char* g_last_names[kMaxLaunchNames] = {};

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

bool valid_block(int b) { return b == 1 || b == 2 || b == 4 || b == 8 || b == 16; }

flr_status check_params(const flr_params* p)
{
    if (!p) return FLR_ERR_INVALID_VALUE;
    if (!valid_block(p->block) || p->upsample < 1 || p->upsample > 64) return FLR_ERR_INVALID_VALUE;
    if (!(p->sigma > 0.0) || !std::isfinite(p->sigma)) return FLR_ERR_INVALID_VALUE;
    if (!(p->eps_add >= 0.0) || !std::isfinite(p->eps_add)) return FLR_ERR_INVALID_VALUE;
    if (!(p->eps_mul >= 0.0) || !(p->eps_mul < 1.0)) return FLR_ERR_INVALID_VALUE;
    if (p->radius < 0) return FLR_ERR_INVALID_VALUE;
    if (p->solver != FLR_SOLVER_APPENDIX && p->solver != FLR_SOLVER_TIKHONOV) return FLR_ERR_INVALID_VALUE;
    if (p->flags & ~FLR_FLAG_INPUTS_READY) return FLR_ERR_INVALID_VALUE;
    if (p->variant != FLR_VARIANT_AUTO && p->variant != FLR_VARIANT_STAGED && p->variant != FLR_VARIANT_FUSED)
        return FLR_ERR_UNSUPPORTED;
    return FLR_OK;
}

// eps_mul as the kernels take it: a negative value selects the Tikhonov solve
// (solve_block_tikhonov in flr_solve.cuh); users cannot pass one (check_params)
inline double solver_eps_mul(const flr_params* p) { return p->solver == FLR_SOLVER_TIKHONOV ? kTikhonovRaw : p->eps_mul; }
// floats per block of the centred Tikhonov models ([b0 | slopes | mu], k_apply_centered)
inline int centered_stride(int Q) { return 4 * (Q + 1); }

// R1: default radius ceil(2 sigma / D_out) blocks (Fig. 3's 41-tap kernel at std 10)
int effective_radius(const flr_params* p)
{
    if (p->radius > 0) return p->radius;
    const double r = std::ceil(2.0 * p->sigma / ((double)p->block * p->upsample) - 1e-12);
    return (int)(r < 0 ? 0 : r);
}

struct Layout {
    size_t raw, mom, hb, models, flags, total;
};

// workspace: raw fp32 moments | fp64 un-shifted moments | fp64 x-blurred | padded models
Layout layout(int n, int Q, int Bx, int By)
{
    const size_t nb = (size_t)n * Bx * By;
    Layout L;
    size_t off = 0;
    L.raw = off;
    off += align256(nb * kraw_of(Q) * sizeof(float));
    const size_t nbp = (size_t)n * mom_pitch(Bx) * By;  // pitched moment rows (TMA)
    L.mom = off;
    off += align256(nbp * km_of(Q) * sizeof(double));
    L.hb = off;
    off += align256(nbp * km_of(Q) * sizeof(double));
    L.models = off;
    off += align256(nb * (mstride_of(Q) > centered_stride(Q) ? mstride_of(Q) : centered_stride(Q)) * sizeof(float));
    L.flags = off;  // task-queue heads + row counters of the wave schedule (zeroed per call)
    off += align256(sizeof(int) * (size_t)wave_flags_ints(n, By));
    L.total = off;
    return L;
}

// unnormalised Gaussian taps g_i = exp(-i^2 / (2 s^2)), s in blocks (R2)
Taps make_taps(double s, int R)
{
    Taps t;
    std::memset(&t, 0, sizeof(t));
    t.R = R;
    for (int i = -R; i <= R; ++i) t.g[R + i] = std::exp(-(double)(i * i) / (2.0 * s * s));
    return t;
}

#define FLR_DISPATCH_Q(Q, CALL)                                                   \
    switch (Q) {                                                                  \
    case 1: { constexpr int QQ = 1; CALL; } break;                                \
    case 2: { constexpr int QQ = 2; CALL; } break;                                \
    case 3: { constexpr int QQ = 3; CALL; } break;                                \
    case 4: { constexpr int QQ = 4; CALL; } break;                                \
    case 5: { constexpr int QQ = 5; CALL; } break;                                \
    case 6: { constexpr int QQ = 6; CALL; } break;                                \
    case 7: { constexpr int QQ = 7; CALL; } break;                                \
    case 8: { constexpr int QQ = 8; CALL; } break;                                \
    case 9: { constexpr int QQ = 9; CALL; } break;                                \
    case 10: { constexpr int QQ = 10; CALL; } break;                              \
    case 11: { constexpr int QQ = 11; CALL; } break;                              \
    case 12: { constexpr int QQ = 12; CALL; } break;                              \
    case 13: { constexpr int QQ = 13; CALL; } break;                              \
    case 14: { constexpr int QQ = 14; CALL; } break;                              \
    case 15: { constexpr int QQ = 15; CALL; } break;                              \
    default: return FLR_ERR_INVALID_VALUE;                                        \
    }

flr_status check_fit_args(int n, int Q, int W, int H, const void* G, const void* Y,
                          const flr_params* p)
{
    flr_status st = check_params(p);
    if (st) return st;
    if (Q < 1 || Q > kMaxQ) return FLR_ERR_INVALID_VALUE;
    if (n < 1 || W < 1 || H < 1 || n > 65535) return FLR_ERR_SHAPE;
    if (!G || !Y) return FLR_ERR_INVALID_VALUE;
    if (!aligned(G, 4) || !aligned(Y, 4)) return FLR_ERR_ALIGNMENT;
    if (effective_radius(p) > kMaxR) return FLR_ERR_UNSUPPORTED;
    return FLR_OK;
}

LaunchCtx make_ctx(flr_stream_t stream, flr_event_trace* trace)
{
    LaunchCtx c;
    c.s = (cudaStream_t)stream;
    if (trace) {
        trace->recorded = 0;
        if (trace->events && trace->capacity > 0) {
            c.events = trace->events;
            c.capacity = trace->capacity;
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            if (cudaStreamIsCapturing(c.s, &cs) == cudaSuccess) c.capturing = cs != cudaStreamCaptureStatusNone;
        }
    }
    return c;
}

flr_status finish(LaunchCtx& ctx, flr_event_trace* trace)
{
    ctx.end();
    if (trace) trace->recorded = ctx.recorded;
    if (ctx.unsupported) return FLR_ERR_UNSUPPORTED;
    if (cudaGetLastError() != cudaSuccess) return FLR_ERR_CUDA;
    g_last_launches = ctx.launches;
    for (int i = 0; i < kMaxLaunchNames; ++i) g_last_names[i] = ctx.names[i];
    return FLR_OK;
}

flr_status check_ws(int n, int Q, int W, int H, const flr_params* p, void* ws, size_t bytes);

// fit into `models` with `mstride` floats per block; arguments already validated
flr_status do_fit(int n, int Q, int W, int H, const float* G, const float* Y, const flr_params* p,
                  float* models, int mstride, void* ws, LaunchCtx& ctx, bool hg = false,
                  bool inputs_from_call = false, double eps_mul_override = 0.0)
{
    const int D = p->block;
    const int Bx = cdiv(W, D), By = cdiv(H, D);
    const Layout L = layout(n, Q, Bx, By);
    char* base = (char*)ws;
    const double sblk = p->sigma / ((double)D * p->upsample);
    const Taps taps = make_taps(sblk, effective_radius(p));
    // FLR_FLAG_INPUTS_READY: the moment grid may stream before its grid-dependency wait --
    // unless its radiance was produced inside this call (the unfused demodulation)
    ctx.early = (p->flags & FLR_FLAG_INPUTS_READY) && !inputs_from_call;
    FLR_DISPATCH_Q(Q, (launch_fit<QQ>(n, W, H, D, Bx, By, G, Y, (float*)(base + L.raw),
                                      (double*)(base + L.mom), (double*)(base + L.hb), models,
                                      mstride, p->eps_add, eps_mul_override < 0.0 ? eps_mul_override : solver_eps_mul(p),
                                      taps, ctx, nullptr, 0.f, hg)));
    return FLR_OK;
}

// generic (unfused) albedo protocol, any shape: y = r / max(a, floor) into `y`, and
// out = a * out + d in place (R20, R21)
__global__ void k_demod(size_t total, const float* __restrict__ r, const float* __restrict__ a, float afloor,
                        float* __restrict__ y)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
        y[i] = r[i] * __frcp_rn(fmaxf(a[i], afloor));
}
__global__ void k_remod(size_t total, float* __restrict__ out, const float* __restrict__ a,
                        const float* __restrict__ d)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
        out[i] = fmaf(a[i], out[i], d ? d[i] : 0.0f);
}
inline unsigned ew_grid(size_t total)
{
    const size_t b = (total + 255) / 256;
    return (unsigned)(b < 148 * 16 ? b : 148 * 16);
}

flr_status check_ws(int n, int Q, int W, int H, const flr_params* p, void* ws, size_t bytes)
{
    size_t need = 0;
    flr_status st = flr_workspace_size(n, Q, W, H, p, &need);
    if (st) return st;
    if (!ws) return FLR_ERR_INVALID_VALUE;
    if (!aligned(ws, 256)) return FLR_ERR_ALIGNMENT;
    if (bytes < need) return FLR_ERR_WORKSPACE;
    return FLR_OK;
}

}  // namespace

extern "C" {

void flr_default_params(flr_params* p)
{
    if (!p) return;
    p->block = 8;
    p->upsample = 1;
    p->radius = 0;
    p->variant = FLR_VARIANT_AUTO;
    p->sigma = 10.0;
    p->eps_add = 1e-5;
    p->eps_mul = 1e-4;
    p->solver = FLR_SOLVER_APPENDIX;
    p->flags = 0;
}

const char* flr_status_string(flr_status s)
{
    switch (s) {
    case FLR_OK: return "FLR_OK";
    case FLR_ERR_INVALID_VALUE: return "FLR_ERR_INVALID_VALUE";
    case FLR_ERR_SHAPE: return "FLR_ERR_SHAPE";
    case FLR_ERR_ALIGNMENT: return "FLR_ERR_ALIGNMENT";
    case FLR_ERR_WORKSPACE: return "FLR_ERR_WORKSPACE";
    case FLR_ERR_UNSUPPORTED: return "FLR_ERR_UNSUPPORTED";
    case FLR_ERR_CUDA: return "FLR_ERR_CUDA";
    }
    return "FLR_ERR_UNKNOWN";
}

int32_t flr_effective_radius(const flr_params* p)
{
    if (check_params(p) != FLR_OK) return -1;
    return effective_radius(p);
}

int32_t flr_last_launch_count(void) { return g_last_launches; }

const char* flr_last_launch_name(int32_t i)
{
    if (i < 0 || i >= g_last_launches || i >= kMaxLaunchNames || !g_last_names[i]) return "";
    return g_last_names[i];
}

flr_status flr_workspace_size(int32_t n, int32_t Q, int32_t W_fit, int32_t H_fit,
                              const flr_params* p, size_t* bytes)
{
    flr_status st = check_params(p);
    if (st) return st;
    if (!bytes) return FLR_ERR_INVALID_VALUE;
    if (Q < 1 || Q > kMaxQ) return FLR_ERR_INVALID_VALUE;
    if (n < 1 || W_fit < 1 || H_fit < 1 || n > 65535) return FLR_ERR_SHAPE;
    *bytes = layout(n, Q, cdiv(W_fit, p->block), cdiv(H_fit, p->block)).total;
    return FLR_OK;
}

flr_status flr_fit(int32_t n, int32_t Q, int32_t W_fit, int32_t H_fit, const float* guides_fit,
                   const float* radiance_fit, const flr_params* p, float* models, void* workspace,
                   size_t workspace_bytes, flr_stream_t stream)
{
    flr_status st = check_fit_args(n, Q, W_fit, H_fit, guides_fit, radiance_fit, p);
    if (st) return st;
    if (!models) return FLR_ERR_INVALID_VALUE;
    if (!aligned(models, 4)) return FLR_ERR_ALIGNMENT;
    if ((st = check_ws(n, Q, W_fit, H_fit, p, workspace, workspace_bytes))) return st;
    LaunchCtx ctx = make_ctx(stream, nullptr);
    if ((st = do_fit(n, Q, W_fit, H_fit, guides_fit, radiance_fit, p, models, 3 * (Q + 1), workspace,
                     ctx)))
        return st;
    return finish(ctx, nullptr);
}

flr_status flr_apply(int32_t n, int32_t Q, int32_t W_out, int32_t H_out, int32_t block_out,
                     int32_t Bx, int32_t By, const float* models, const float* guides_out, float* out,
                     flr_stream_t stream)
{
    if (Q < 1 || Q > kMaxQ || block_out < 1) return FLR_ERR_INVALID_VALUE;
    if (n < 1 || W_out < 1 || H_out < 1 || n > 65535) return FLR_ERR_SHAPE;
    if (!models || !guides_out || !out) return FLR_ERR_INVALID_VALUE;
    if (Bx != cdiv(W_out, block_out) || By != cdiv(H_out, block_out)) return FLR_ERR_SHAPE;
    if (!aligned(models, 4) || !aligned(guides_out, 4) || !aligned(out, 4)) return FLR_ERR_ALIGNMENT;
    LaunchCtx ctx = make_ctx(stream, nullptr);
    FLR_DISPATCH_Q(Q, (launch_apply<QQ>(n, W_out, H_out, block_out, Bx, By, models, 3 * (QQ + 1),
                                        guides_out, out, ctx)));
    return finish(ctx, nullptr);
}

}  // extern "C"

namespace {
// fit on (guides_lo, radiance_lo) + apply with guides_hi; hg: both guide sets are fp16
flr_status denoise_upsample_impl(int32_t n, int32_t Q, int32_t W_lo, int32_t H_lo, const void* guides_lo_,
                                 const float* radiance_lo, int32_t W_hi, int32_t H_hi, const void* guides_hi_,
                                 const flr_params* p, float* out, void* workspace, size_t workspace_bytes,
                                 flr_stream_t stream, flr_event_trace* trace, bool hg)
{
    const float* guides_lo = (const float*)guides_lo_;
    const float* guides_hi = (const float*)guides_hi_;
    flr_status st = check_fit_args(n, Q, W_lo, H_lo, guides_lo, radiance_lo, p);
    if (st) return st;
    if (!guides_hi || !out) return FLR_ERR_INVALID_VALUE;
    if ((int64_t)W_hi != (int64_t)W_lo * p->upsample || (int64_t)H_hi != (int64_t)H_lo * p->upsample)
        return FLR_ERR_SHAPE;
    if (!aligned(guides_hi, 4) || !aligned(out, 4)) return FLR_ERR_ALIGNMENT;
    if ((st = check_ws(n, Q, W_lo, H_lo, p, workspace, workspace_bytes))) return st;
    const int D = p->block;
    const int Bx = cdiv(W_lo, D), By = cdiv(H_lo, D);
    const Layout L = layout(n, Q, Bx, By);
    float* models = (float*)((char*)workspace + L.models);
    const int ms = mstride_of(Q);
    LaunchCtx ctx = make_ctx(stream, trace);
    // FUSED: the one-kernel wave schedule (flr_wave.cuh).  AUTO stays on the staged kernels:
    // on B200 the wave schedule is correct (bitwise equal) but slower
    if (p->variant == FLR_VARIANT_FUSED && !hg && p->solver != FLR_SOLVER_TIKHONOV) {
        WaveLaunch W;
        W.n = n, W.W = W_lo, W.H = H_lo, W.D = D, W.U = p->upsample, W.Bx = Bx, W.By = By;
        W.G = guides_lo, W.Y = radiance_lo, W.Gout = guides_hi, W.out = out;
        W.mom = (double*)((char*)workspace + L.mom);
        W.models = models;
        W.flags = (int*)((char*)workspace + L.flags);
        W.eps_add = p->eps_add, W.eps_mul = solver_eps_mul(p);
        W.taps = make_taps(p->sigma / ((double)D * p->upsample), effective_radius(p));
        bool done = false;
        FLR_DISPATCH_Q(Q, (done = launch_wave<QQ>(W, ctx)));
        if (done) return finish(ctx, trace);
    }
    if (p->variant == FLR_VARIANT_FUSED) return FLR_ERR_UNSUPPORTED;
    const int Dout = D * p->upsample;
    if (p->solver == FLR_SOLVER_TIKHONOV && !hg) {
        // Tikhonov models centred at the window mean, evaluated per block and blended
        // (k_apply_centered): the raw-basis fp32 apply loses precision at eps ~1e-6
        flr_params pc = *p;
        const int cs = centered_stride(Q);
        LaunchCtx* c = &ctx;
        if ((st = do_fit(n, Q, W_lo, H_lo, guides_lo, radiance_lo, &pc, models, cs, workspace, *c, false, false,
                         kTikhonovCentered)))
            return st;
        c->before("k_apply_centered");
        FLR_DISPATCH_Q(Q, (k_apply_centered<QQ><<<dim3(cdiv(W_hi, 128), H_hi, n), 128, 0, c->s>>>(
                               W_hi, H_hi, Dout, Bx, By, models, cs, guides_hi, out)));
        return finish(ctx, trace);
    }
    if (hg && (!half_guides_fit_ok(D, W_lo, guides_lo, radiance_lo) ||
               !half_guides_apply_ok(Dout, W_hi, models, guides_hi, out)))
        return FLR_ERR_UNSUPPORTED;
    // denoise (U = 1, one guide set): the apply re-reads the fit's guides, which the fit then
    // leaves in L2 when they fit there (launch_fit)
    ctx.keep_guides = guides_lo == guides_hi;  // (fp16 guides too: C2 38.6 -> 38.5 us per frame)
    const size_t frame_guides = (size_t)Q * W_lo * H_lo * sizeof(float);
    if (ctx.keep_guides && !hg && n > 1 && frame_guides <= kGuideL2Keep) {
        // a batch of frames that each fit in L2: frame by frame (fit -> K2 -> apply, one
        // workspace slice), so every frame's apply finds its guides in L2 and the moment field
        // stays L2-resident (32-frame calls 42.3 -> 41.2, 8-frame calls 43.25 -> 41.4 us per
        // frame).  Frames after the first stream their inputs while the previous frame's apply
        // drains: they are inputs of this call, complete once the first frame's fit has passed
        // its grid wait (FLR_FLAG_INPUTS_READY semantics, which the first frame takes from p).
        flr_params pf = *p;
        const size_t px = (size_t)W_lo * H_lo, nb = (size_t)Bx * By;
        for (int f = 0; f < n; ++f) {
            if (f == 1) pf.flags |= FLR_FLAG_INPUTS_READY;
            if ((st = do_fit(1, Q, W_lo, H_lo, guides_lo + f * Q * px, radiance_lo + f * 3 * px, &pf, models + f * nb * ms,
                             ms, workspace, ctx, false)))
                return st;
            FLR_DISPATCH_Q(Q, (launch_apply<QQ>(1, W_hi, H_hi, Dout, Bx, By, models + f * nb * ms, ms,
                                                guides_hi + f * Q * px, out + f * 3 * px, ctx, nullptr, nullptr, false)));
        }
        return finish(ctx, trace);
    }
    if ((st = do_fit(n, Q, W_lo, H_lo, guides_lo, radiance_lo, p, models, ms, workspace, ctx, hg)))
        return st;
    FLR_DISPATCH_Q(Q, (launch_apply<QQ>(n, W_hi, H_hi, Dout, Bx, By, models, ms, guides_hi, out, ctx, nullptr,
                                        nullptr, hg)));
    return finish(ctx, trace);
}
}  // namespace

extern "C" {

flr_status flr_denoise_upsample_traced(int32_t n, int32_t Q, int32_t W_lo, int32_t H_lo,
                                       const float* guides_lo, const float* radiance_lo, int32_t W_hi,
                                       int32_t H_hi, const float* guides_hi, const flr_params* p,
                                       float* out, void* workspace, size_t workspace_bytes,
                                       flr_stream_t stream, flr_event_trace* trace)
{
    return denoise_upsample_impl(n, Q, W_lo, H_lo, guides_lo, radiance_lo, W_hi, H_hi, guides_hi, p, out,
                                 workspace, workspace_bytes, stream, trace, false);
}

flr_status flr_denoise_upsample_f16_traced(int32_t n, int32_t Q, int32_t W_lo, int32_t H_lo,
                                           const uint16_t* guides_lo, const float* radiance_lo, int32_t W_hi,
                                           int32_t H_hi, const uint16_t* guides_hi, const flr_params* p, float* out,
                                           void* workspace, size_t workspace_bytes, flr_stream_t stream,
                                           flr_event_trace* trace)
{
    if (p && p->variant == FLR_VARIANT_FUSED) return FLR_ERR_UNSUPPORTED;
    return denoise_upsample_impl(n, Q, W_lo, H_lo, guides_lo, radiance_lo, W_hi, H_hi, guides_hi, p, out,
                                 workspace, workspace_bytes, stream, trace, true);
}

flr_status flr_denoise_upsample_f16(int32_t n, int32_t Q, int32_t W_lo, int32_t H_lo, const uint16_t* guides_lo,
                                    const float* radiance_lo, int32_t W_hi, int32_t H_hi,
                                    const uint16_t* guides_hi, const flr_params* p, float* out, void* workspace,
                                    size_t workspace_bytes, flr_stream_t stream)
{
    return flr_denoise_upsample_f16_traced(n, Q, W_lo, H_lo, guides_lo, radiance_lo, W_hi, H_hi, guides_hi, p, out,
                                           workspace, workspace_bytes, stream, nullptr);
}

flr_status flr_denoise_f16_traced(int32_t n, int32_t Q, int32_t W, int32_t H, const uint16_t* guides,
                                  const float* radiance, const flr_params* p, float* out, void* workspace,
                                  size_t workspace_bytes, flr_stream_t stream, flr_event_trace* trace)
{
    if (p && (p->upsample != 1 || p->variant == FLR_VARIANT_FUSED))
        return p->upsample != 1 ? FLR_ERR_INVALID_VALUE : FLR_ERR_UNSUPPORTED;
    return denoise_upsample_impl(n, Q, W, H, guides, radiance, W, H, guides, p, out, workspace, workspace_bytes,
                                 stream, trace, true);
}

flr_status flr_denoise_f16(int32_t n, int32_t Q, int32_t W, int32_t H, const uint16_t* guides,
                           const float* radiance, const flr_params* p, float* out, void* workspace,
                           size_t workspace_bytes, flr_stream_t stream)
{
    return flr_denoise_f16_traced(n, Q, W, H, guides, radiance, p, out, workspace, workspace_bytes, stream,
                                  nullptr);
}

flr_status flr_fit_f16(int32_t n, int32_t Q, int32_t W_fit, int32_t H_fit, const uint16_t* guides_fit,
                       const float* radiance_fit, const flr_params* p, float* models, void* workspace,
                       size_t workspace_bytes, flr_stream_t stream)
{
    flr_status st = check_fit_args(n, Q, W_fit, H_fit, guides_fit, radiance_fit, p);
    if (st) return st;
    if (!models) return FLR_ERR_INVALID_VALUE;
    if (!aligned(models, 4)) return FLR_ERR_ALIGNMENT;
    if ((st = check_ws(n, Q, W_fit, H_fit, p, workspace, workspace_bytes))) return st;
    if (!half_guides_fit_ok(p->block, W_fit, guides_fit, radiance_fit)) return FLR_ERR_UNSUPPORTED;
    LaunchCtx ctx = make_ctx(stream, nullptr);
    if ((st = do_fit(n, Q, W_fit, H_fit, (const float*)guides_fit, radiance_fit, p, models, 3 * (Q + 1), workspace,
                     ctx, true)))
        return st;
    return finish(ctx, nullptr);
}


flr_status flr_denoise_upsample(int32_t n, int32_t Q, int32_t W_lo, int32_t H_lo,
                                const float* guides_lo, const float* radiance_lo, int32_t W_hi,
                                int32_t H_hi, const float* guides_hi, const flr_params* p, float* out,
                                void* workspace, size_t workspace_bytes, flr_stream_t stream)
{
    return flr_denoise_upsample_traced(n, Q, W_lo, H_lo, guides_lo, radiance_lo, W_hi, H_hi, guides_hi,
                                       p, out, workspace, workspace_bytes, stream, nullptr);
}

flr_status flr_denoise_traced(int32_t n, int32_t Q, int32_t W, int32_t H, const float* guides,
                              const float* radiance, const flr_params* p, float* out, void* workspace,
                              size_t workspace_bytes, flr_stream_t stream, flr_event_trace* trace)
{
    if (p && p->upsample != 1) return FLR_ERR_INVALID_VALUE;
    return flr_denoise_upsample_traced(n, Q, W, H, guides, radiance, W, H, guides, p, out, workspace,
                                       workspace_bytes, stream, trace);
}

flr_status flr_denoise_modulated_traced(int32_t n, int32_t Q, int32_t W, int32_t H, const float* guides,
                                        const float* radiance_mod, const float* albedo, const float* direct,
                                        float albedo_floor, const flr_params* p, float* out, void* workspace,
                                        size_t workspace_bytes, flr_stream_t stream, flr_event_trace* trace)
{
    flr_status st = check_fit_args(n, Q, W, H, guides, radiance_mod, p);
    if (st) return st;
    if (p->upsample != 1) return FLR_ERR_INVALID_VALUE;
    if (!albedo || !out || !(albedo_floor > 0.0f) || !std::isfinite(albedo_floor)) return FLR_ERR_INVALID_VALUE;
    if (!aligned(albedo, 4) || !aligned(out, 4) || (direct && !aligned(direct, 4))) return FLR_ERR_ALIGNMENT;
    if ((st = check_ws(n, Q, W, H, p, workspace, workspace_bytes))) return st;
    const int D = p->block;
    const int Bx = cdiv(W, D), By = cdiv(H, D);
    const Layout L = layout(n, Q, Bx, By);
    float* models = (float*)((char*)workspace + L.models);
    const int ms = mstride_of(Q);
    const size_t total = (size_t)n * 3 * W * H;
    LaunchCtx ctx = make_ctx(stream, trace);
    if (fit_mod_fused(D, W, guides, radiance_mod, albedo)) {  // demodulation in the moment kernel's loads
        const double sblk = p->sigma / (double)D;
        const Taps taps = make_taps(sblk, effective_radius(p));
        char* base = (char*)workspace;
        ctx.early = (p->flags & FLR_FLAG_INPUTS_READY) != 0;
        ctx.keep_guides = true;  // the remodulating apply re-reads these guides (58.5 -> 57.5 us per C2 frame)
        FLR_DISPATCH_Q(Q, (launch_fit<QQ>(n, W, H, D, Bx, By, guides, radiance_mod, (float*)(base + L.raw),
                                          (double*)(base + L.mom), (double*)(base + L.hb), models, ms,
                                          p->eps_add, solver_eps_mul(p), taps, ctx, albedo, albedo_floor)));
    } else {  // demodulate into `out` (same shape), then the plain fit reads it
        ctx.before("k_demod");
        k_demod<<<ew_grid(total), 256, 0, (cudaStream_t)stream>>>(total, radiance_mod, albedo, albedo_floor, out);
        if ((st = do_fit(n, Q, W, H, guides, out, p, models, ms, workspace, ctx, false, true))) return st;
    }
    bool mod_ok = false;
    FLR_DISPATCH_Q(Q, (mod_ok = apply_mod_supported<QQ>()));
    if (mod_ok && apply_mod_fused(D, W, models, guides, out, albedo, direct)) {  // remodulation in the apply's stores
        FLR_DISPATCH_Q(Q, (launch_apply<QQ>(n, W, H, D, Bx, By, models, ms, guides, out, ctx, albedo, direct)));
    } else {
        FLR_DISPATCH_Q(Q, (launch_apply<QQ>(n, W, H, D, Bx, By, models, ms, guides, out, ctx)));
        ctx.before("k_remod");
        k_remod<<<ew_grid(total), 256, 0, (cudaStream_t)stream>>>(total, out, albedo, direct);
    }
    return finish(ctx, trace);
}

flr_status flr_denoise_modulated(int32_t n, int32_t Q, int32_t W, int32_t H, const float* guides,
                                 const float* radiance_mod, const float* albedo, const float* direct,
                                 float albedo_floor, const flr_params* p, float* out, void* workspace,
                                 size_t workspace_bytes, flr_stream_t stream)
{
    return flr_denoise_modulated_traced(n, Q, W, H, guides, radiance_mod, albedo, direct, albedo_floor, p, out,
                                        workspace, workspace_bytes, stream, nullptr);
}

flr_status flr_denoise(int32_t n, int32_t Q, int32_t W, int32_t H, const float* guides,
                       const float* radiance, const flr_params* p, float* out, void* workspace,
                       size_t workspace_bytes, flr_stream_t stream)
{
    return flr_denoise_traced(n, Q, W, H, guides, radiance, p, out, workspace, workspace_bytes, stream,
                              nullptr);
}

}  // extern "C"
