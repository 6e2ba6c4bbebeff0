// flr_pipe.cuh -- sm_100a asynchronous-copy plumbing: mbarriers, 1-D bulk copies
// (cp.async.bulk, the TMA engine's non-tensor mode) with L2 cache-policy hints, and
// acquire/release flags for the persistent schedule.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#ifdef FLR_WATCHDOG
#include <cstdio>
#endif

namespace flr {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// ---- mbarrier ---------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity)
{
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, unsigned parity)  // non-blocking
{
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
#ifdef FLR_WATCHDOG
// debug builds: a wait that has not completed after ~2^32 cycles reports itself and traps
__device__ __forceinline__ void mbar_wait_dbg(uint64_t* bar, unsigned parity, int line)
{
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, parity)) {
        if (clock64() - t0 > (1ll << 32)) {
            printf("FLR watchdog: mbar_wait line %d block %d thread %d bar_off %u parity %u\n", line, blockIdx.x,
                   threadIdx.x, (unsigned)__cvta_generic_to_shared(bar), parity);
            __trap();
        }
    }
}
#define mbar_wait(b, p) mbar_wait_dbg((b), (p), __LINE__)
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity)
{
    while (!mbar_try_wait(bar, parity)) {
    }
}
#endif

// Producer side of a warp-specialised ring, before a TMA write into a stage the consumers
// have read: a generic -> async proxy fence (conservative; measured free, FLR_WS_NO_PROXY_FENCE
// drops it for experiments).
__device__ __forceinline__ void ws_proxy_fence()
{
#ifndef FLR_WS_NO_PROXY_FENCE
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
}

__device__ __forceinline__ int smid()
{
    int v;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
    return v;
}

__device__ __forceinline__ long long gtimer()
{
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Optional CTA timeline (tools/t_timeline.cu, -DFLR_TIMELINE): globaltimer stamps per CTA
// of the three default kernels, [kernel][cta][slot] with slot 0 = entry, 1 = past the
// grid-dependency wait, 2 = exit.  Compiled out of the library.
#ifdef FLR_TIMELINE
__device__ long long g_flr_tl[3 * 1024 * 4];  // single-TU tools only (no -rdc)
#define FLR_TL(k, slot)                                                                           \
    (((slot) == 2 ? (void)(g_flr_tl[((k) * 1024 + blockIdx.x + blockIdx.y * gridDim.x) * 4 + 3] = smid()) \
                  : (void)0),                                                                          \
     g_flr_tl[((k) * 1024 + blockIdx.x + blockIdx.y * gridDim.x) * 4 + (slot)] = gtimer())
#else
#define FLR_TL(k, slot) ((void)0)
#endif

// ---- L2 cache policies --------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last_frac(float f)
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(p) : "f"(f));
    return p;
}
// policy codes (kernel arguments): 0 evict_first, 1 evict_normal, 2 evict_last,
// 3 / 4 evict_last for 3/4 / 1/2 of the lines (the rest evict_first)
__device__ __forceinline__ uint64_t policy_by_code(int code)
{
    switch (code) {
    case 1: return policy_evict_normal();
    case 2: return policy_evict_last();
    case 3: return policy_evict_last_frac(0.75f);
    case 4: return policy_evict_last_frac(0.5f);
    default: return policy_evict_first();
    }
}
// fp64 store with an L2 cache-policy hint
__device__ __forceinline__ void st_hint_f64(double* p, double v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// ---- bulk copy global -> shared (bytes % 16 == 0, both addresses 16-byte aligned) ----
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ---- global flags (acquire / release at gpu scope) ----------------------------
__device__ __forceinline__ int ld_acquire(const int* p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p)
{
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v)
{
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ int atom_cas_acq_rel(int* p, int cmp, int v)
{
    int old;
    asm volatile("atom.acq_rel.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_release_max(int* p, int v)
{
    asm volatile("red.release.gpu.global.max.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(int* p, int v)
{
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace flr

namespace flr {

// named barrier `id` (1..15) over `count` threads (a multiple of 32) of the CTA
__device__ __forceinline__ void named_bar_sync(int id, int count)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- programmatic dependent launch (no-ops when launched without the PDL attribute) ----
// wait: block until the preceding grid in the stream has completed and flushed its writes
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// trigger: let the next grid in the stream start launching its CTAs now
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- TMA tensor load (3-D tile; coordinates may be negative: out-of-range elements are zero) ----
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar,
                                            uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ---- packed fp32 pairs (sm_100a FFMA2/FADD2): a scalar operand broadcasts to both halves ----
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float a, float b)
{
    f2 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(f2 v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ float lo2(f2 v)
{
    float a, b;
    upk2(v, a, b);
    return a;
}
__device__ __forceinline__ float hi2(f2 v)
{
    float a, b;
    upk2(v, a, b);
    return b;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c)
{
    f2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b)
{
    f2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b)
{
    f2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 bc2(float a) { return pk2(a, a); }

}  // namespace flr
