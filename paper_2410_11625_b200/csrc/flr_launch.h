// flr_launch.h -- host-side launcher declarations, one explicit instantiation per Q
// (flr_inst.cu is compiled once per Q = 1..15 so the build parallelises).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "flr_common.cuh"

namespace flr {

inline int cdiv(int a, int b) { return (a + b - 1) / b; }
inline bool aligned(const void* ptr, size_t a) { return ((uintptr_t)ptr % a) == 0; }
inline bool vec_ok(const void* ptr, int W) { return aligned(ptr, 16) && (W % 4) == 0; }

// 3-D TMA tensor map over `planes` planes of W x H elements (row stride `pitch` elements):
// box {bx, by, bz}.  Requires pitch * esize % 16 == 0 and a 16-byte aligned base.
// Out-of-range box elements read as 0.
inline bool make_tmap_3d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int esize, int W, int H,
                         int pitch, int planes, int bx, int by, int bz)
{
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)pitch * esize, (cuuint64_t)pitch * H * esize};
    const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
    const cuuint32_t estr[3] = {1, 1, 1};
    return encode(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// fp32 planes [planes][H][W], box {bx, by, bz}
inline bool make_tmap_planes(CUtensorMap* m, const float* base, int W, int H, int planes, int bx, int bz, int by = 1)
{
    return make_tmap_3d(m, base, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, W, H, W, planes, bx, by, bz);
}
// moment-field row pitch (elements): even, so rows are 16-byte aligned for TMA
inline int mom_pitch(int Bx) { return (Bx + 1) & ~1; }

// Per-call launch context: the caller's stream, a launch counter, and an optional
// caller-owned event trace (events[i] is recorded right before launch i and one
// more after the last launch; see flr_event_trace in include/flr.h).
// largest guide volume of one call the fit leaves in L2 (evict_normal) for the apply; batched
// denoise calls whose frames fit run frame by frame (flr_api.cu)
constexpr size_t kGuideL2Keep = (size_t)80 << 20;
// guide bytes of one frame the fit leaves in L2 for the bottom-up apply (its last rows)
#ifndef FLR_GUIDE_L2_MB
#define FLR_GUIDE_L2_MB 50
#endif
constexpr size_t kGuideL2Rows = (size_t)FLR_GUIDE_L2_MB << 20;
constexpr int kMaxLaunchNames = 256;  // launch names kept per call (flr_last_launch_name)

struct LaunchCtx {
    cudaStream_t s = nullptr;
    int launches = 0;
    void** events = nullptr;
    int capacity = 0;
    int recorded = 0;
    bool capturing = false;   // stream capture: events become graph event-record nodes
    bool unsupported = false; // set by launchers compiled out of a dev build (FLR_STUB)
    bool early = false;       // FLR_FLAG_INPUTS_READY: the moment grid streams before its grid wait
    bool keep_guides = false; // the call's apply re-reads the fit's guide planes (denoise, U = 1)
    bool l2_guides = false;   // ... and the fit left them in L2 (evict_normal): the deep apply ring
    void record()
    {
        if (events && recorded < capacity) {
            cudaEvent_t e = (cudaEvent_t)events[recorded++];
            if (capturing) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
            else cudaEventRecord(e, s);
        }
    }
    const char* names[kMaxLaunchNames] = {};
    void before(const char* name)
    {
        record();
        if (launches < kMaxLaunchNames) names[launches] = name;
        ++launches;
    }
    void end() { record(); }
};

// K1 -> K2 (blur + solve) into `models` (mstride floats per block)
// A (optional): albedo [n][3][H][W]; the fit then uses Y / max(A, afloor) as its radiance
// (demodulation fused into the moment kernel; only when fit_mod_fused() holds)
template <int Q>
void launch_fit(int n, int W, int H, int D, int Bx, int By, const float* G, const float* Y,
                float* raw, double* mom, double* hb, float* models, int mstride, double ea,
                double em, const Taps& taps, LaunchCtx& ctx, const float* A = nullptr, float afloor = 0.f,
                bool hg = false);

// K4 with the fastest kernel the shape allows
// A (optional): albedo [n][3][H][W]; out = A * I + Dl (Dl optional direct light), fused into
// the apply kernel's stores (only when apply_mod_fused() holds)
template <int Q>
void launch_apply(int n, int W, int H, int D, int Bx, int By, const float* models, int mstride,
                  const float* G, float* out, LaunchCtx& ctx, const float* A = nullptr,
                  const float* Dl = nullptr, bool hg = false);

// hg (half guides): G points to IEEE binary16 planes; only the warp-specialised TMA kernels
// read them, so the shape must satisfy half_guides_ok() (the API checks before launching)
inline bool half_guides_fit_ok(int D, int W, const void* G, const void* Y)
{
    return (D == 4 || D == 8 || D == 16) && aligned(G, 16) && W % 8 == 0 && vec_ok(Y, W);
}
inline bool half_guides_apply_ok(int D, int W, const void* models, const void* G, const void* out)
{
    return D % 8 == 0 && aligned(models, 16) && aligned(G, 16) && W % 8 == 0 && vec_ok(out, W);
}
// fp16 planes [planes][H][W], box {bx, by, bz}
inline bool make_tmap_planes_f16(CUtensorMap* m, const void* base, int W, int H, int planes, int bx, int bz,
                                 int by = 1)
{
    return make_tmap_3d(m, base, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, W, H, W, planes, bx, by, bz);
}

// shapes for which the modulated (albedo) protocol runs fused into the TMA kernels
inline bool fit_mod_fused(int D, int W, const void* G, const void* Y, const void* A)
{
    return (D == 4 || D == 8 || D == 16) && vec_ok(G, W) && vec_ok(Y, W) && vec_ok(A, W);
}
template <int Q>
bool apply_mod_supported();  // the fused modulated apply kernel fits in shared memory for this Q
inline bool apply_mod_fused(int D, int W, const void* models, const void* G, const void* out, const void* A,
                            const void* Dl)
{
    return D % 8 == 0 && aligned(models, 16) && vec_ok(G, W) && vec_ok(out, W) && vec_ok(A, W) &&
           (!Dl || vec_ok(Dl, W));
}

// the one-kernel wavefront schedule (flr_wave.cuh).  Returns false, launching nothing,
// when the shape is not compiled in (Q in {4, 8}, block in {4, 8}, R in {3, 5}, output
// block a multiple of 8, 16-byte aligned planes with W % 4 == 0): the caller then runs
// the staged kernels.
struct WaveLaunch {
    int n, W, H, D, U, Bx, By;    // fit resolution, block size, upsample
    const float *G, *Y, *Gout;    // fit guides, fit radiance, output-resolution guides
    float* out;
    double* mom;                  // [n][KM][By][Bxp]
    float* models;                // padded [n][By][Bx][MSTRIDE]
    int* flags;                   // wave_flags_ints(n, By) ints of workspace
    double eps_add, eps_mul;
    Taps taps;
};
#ifdef FLR_WAVE_TRACE
inline int wave_flags_ints(int n, int By) { return 4 + n * (By + 3 * ((By + 7) / 8) + 2) + 4 * 96 * 160 + 2; }
#else
inline int wave_flags_ints(int n, int By) { return 4 + n * (By + 3 * ((By + 7) / 8) + 2); }
#endif
template <int Q>
bool launch_wave(const WaveLaunch& L, LaunchCtx& ctx);

#define FLR_DECLARE_Q(Q)                                                                          \
    extern template void launch_fit<Q>(int, int, int, int, int, int, const float*, const float*,  \
                                       float*, double*, double*, float*, int, double, double,     \
                                       const Taps&, LaunchCtx&, const float*, float, bool);       \
    extern template void launch_apply<Q>(int, int, int, int, int, int, const float*, int,         \
                                         const float*, float*, LaunchCtx&, const float*,          \
                                         const float*, bool);                                     \
    extern template bool apply_mod_supported<Q>();                                              \
    extern template bool launch_wave<Q>(const WaveLaunch&, LaunchCtx&);
FLR_DECLARE_Q(1) FLR_DECLARE_Q(2) FLR_DECLARE_Q(3) FLR_DECLARE_Q(4) FLR_DECLARE_Q(5)
FLR_DECLARE_Q(6) FLR_DECLARE_Q(7) FLR_DECLARE_Q(8) FLR_DECLARE_Q(9) FLR_DECLARE_Q(10)
FLR_DECLARE_Q(11) FLR_DECLARE_Q(12) FLR_DECLARE_Q(13) FLR_DECLARE_Q(14) FLR_DECLARE_Q(15)
#undef FLR_DECLARE_Q

}  // namespace flr
