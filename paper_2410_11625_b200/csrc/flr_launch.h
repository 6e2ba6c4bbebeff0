// flr_launch.h -- host-side launcher declarations, one explicit instantiation per Q
// (flr_inst.cu is compiled once per Q = 1..15 so the build parallelises).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "flr_common.cuh"

namespace flr {

inline int cdiv(int a, int b) { return (a + b - 1) / b; }
inline bool aligned(const void* ptr, size_t a) { return ((uintptr_t)ptr % a) == 0; }
inline bool vec_ok(const void* ptr, int W) { return aligned(ptr, 16) && (W % 4) == 0; }

// Per-call launch context: the caller's stream, a launch counter, and an optional
// caller-owned event trace (events[i] is recorded right before launch i and one
// more after the last launch; see flr_event_trace in include/flr.h).
struct LaunchCtx {
    cudaStream_t s = nullptr;
    int launches = 0;
    void** events = nullptr;
    int capacity = 0;
    int recorded = 0;
    bool capturing = false;   // stream capture: events become graph event-record nodes
    bool unsupported = false; // set by launchers compiled out of a dev build (FLR_STUB)
    void record()
    {
        if (events && recorded < capacity) {
            cudaEvent_t e = (cudaEvent_t)events[recorded++];
            if (capturing) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
            else cudaEventRecord(e, s);
        }
    }
    const char* names[16] = {};
    void before(const char* name)
    {
        record();
        if (launches < 16) names[launches] = name;
        ++launches;
    }
    void end() { record(); }
};

// K1 -> K2a -> K2b -> K3 into `models` (mstride floats per block)
template <int Q>
void launch_fit(int n, int W, int H, int D, int Bx, int By, const float* G, const float* Y,
                float* raw, double* mom, double* hb, float* models, int mstride, double ea,
                double em, const Taps& taps, LaunchCtx& ctx);

// K4 with the fastest kernel the shape allows
template <int Q>
void launch_apply(int n, int W, int H, int D, int Bx, int By, const float* models, int mstride,
                  const float* G, float* out, LaunchCtx& ctx);

#define FLR_DECLARE_Q(Q)                                                                          \
    extern template void launch_fit<Q>(int, int, int, int, int, int, const float*, const float*,  \
                                       float*, double*, double*, float*, int, double, double,     \
                                       const Taps&, LaunchCtx&);                          \
    extern template void launch_apply<Q>(int, int, int, int, int, int, const float*, int,         \
                                         const float*, float*, LaunchCtx&);
FLR_DECLARE_Q(1) FLR_DECLARE_Q(2) FLR_DECLARE_Q(3) FLR_DECLARE_Q(4) FLR_DECLARE_Q(5)
FLR_DECLARE_Q(6) FLR_DECLARE_Q(7) FLR_DECLARE_Q(8) FLR_DECLARE_Q(9) FLR_DECLARE_Q(10)
FLR_DECLARE_Q(11) FLR_DECLARE_Q(12) FLR_DECLARE_Q(13) FLR_DECLARE_Q(14) FLR_DECLARE_Q(15)
#undef FLR_DECLARE_Q

}  // namespace flr
