// flr_persist.cuh -- persistent, TMA-fed streaming kernels (one CTA per SM):
//   k_fit_stream  : K1 block moments (FIT items) for the staged schedule
//   k_apply_stream: K4 blended apply (APPLY items) for the staged schedule
// Every warp is a stream warp with its own bulk-copy ring (flr_stream.cuh).  Items
// are assigned round-robin to warp slots (blockIdx.x*NSW + w); each warp's lane 0
// walks the same sequence ahead of the consumer to keep S rows in flight.
#pragma once
#include "flr_stream.cuh"

namespace flr {

// L2 policy of the fit pass's guide reads.  A 1080p frame's guides (66 MB) do not survive
// in L2 until the apply pass anyway (measured: apply re-reads them all from DRAM), so by
// default they are streamed (evict_first) and the L2 keeps the moment field for K2;
// FLR_FIT_GUIDES_LAST builds try to keep them resident instead.
__device__ __forceinline__ uint64_t std_policy_guides_fit()
{
#ifdef FLR_FIT_GUIDES_LAST
    return policy_evict_last();
#else
    return policy_evict_first();
#endif
}

// ring geometry of a streaming kernel: S stages of STG floats + EXTRA floats per warp
template <int STG_, int EXTRA_, int S_, int MAXW>
struct RingCfg {
    static constexpr int S = S_, STG = STG_, EXTRA = EXTRA_;
    static_assert(STG % 32 == 0, "TMA destinations need 128-byte aligned stages");
    static constexpr int WARP_FLOATS = (S * STG + EXTRA + 31) / 32 * 32;  // 128-byte multiple
    static constexpr int NSW0 = (208 * 1024) / (WARP_FLOATS * 4 + S * 8);
    static constexpr int NSW = NSW0 > MAXW ? MAXW : (NSW0 < 1 ? 1 : NSW0);  // stream warps per CTA
    static constexpr size_t SMEM = (size_t)NSW * WARP_FLOATS * 4 + (size_t)NSW * S * sizeof(uint64_t);
    static constexpr int THREADS = NSW * 32;
};
#ifndef FLR_FIT_S
#define FLR_FIT_S 4
#endif
#ifndef FLR_FIT_MAXW
#define FLR_FIT_MAXW 8
#endif
template <int Q>
using FitCfg = RingCfg<StreamDims<Q>::STG_FIT, 0, FLR_FIT_S, FLR_FIT_MAXW>;
template <int Q>
using ApplyCfg = RingCfg<StreamDims<Q>::STG_APPLY, 3 * kApplyNCol * StreamDims<Q>::MS, 3, 12>;

template <class C>
struct RingSmem {
    float* base;
    __device__ explicit RingSmem(unsigned char* p) : base(reinterpret_cast<float*>(p)) {}
    __device__ float* stages(int w) const { return base + (size_t)w * C::WARP_FLOATS; }
    __device__ float* extra(int w) const { return stages(w) + C::S * C::STG; }
    __device__ uint64_t* bars() const { return reinterpret_cast<uint64_t*>(base + (size_t)C::NSW * C::WARP_FLOATS); }
    __device__ Ring ring(int w) const
    {
        Ring r;
        r.stage = stages(w);
        r.full = bars() + (size_t)w * C::S;
        r.S = C::S;
        r.STG = C::STG;
        return r;
    }
    __device__ void init_barriers() const
    {
        for (int i = threadIdx.x; i < C::NSW * C::S; i += blockDim.x) mbar_init(bars() + i, 1);
        fence_mbar_init();
    }
};

// producer cursor over a warp's FIT items: one stage per pixel row (item decoded once)
template <int Q, int D>
struct FitSeq {
    const FitArgs* a;
    int it, nitems, per_frame, step;
    int f, by, sg, row, rows;
    uint64_t pg, py;
    __device__ void decode()
    {
        row = 0;
        if (it >= nitems) return;
        f = it / per_frame;
        const int rem = it - f * per_frame;
        by = rem / a->nseg;
        sg = rem - by * a->nseg;
        rows = min(D, a->H - by * D);
    }
    __device__ bool next(float* dst, uint64_t* bar)
    {
        if (it >= nitems) return false;
        fit_issue_row<Q, D>(*a, f, by, sg, row, dst, bar, pg, py);
        if (++row == rows) {
            it += step;
            decode();
        }
        return true;
    }
};

// producer cursor over a warp's APPLY items: a model stage, then one stage per output row
template <int Q>
struct ApplySeq {
    const ApplyArgs* a;
    int it, nitems, per_frame, step;
    int f, row;
    ApplyGeom g;
    uint64_t pg, pm;
    __device__ void decode()
    {
        row = -1;
        if (it >= nitems) return;
        f = it / per_frame;
        const int rem = it - f * per_frame;
        g = apply_geom(*a, rem / a->nseg, rem % a->nseg);
    }
    __device__ bool next(float* dst, uint64_t* bar)
    {
        if (it >= nitems) return false;
        if (row < 0) {
            if (a->ready) {  // wavefront: the K2 tile rows (ready_ty block rows each) holding rows j0, j1
                const int m0 = g.j0 / a->ready_ty, m1 = g.j1 / a->ready_ty;
                const int v0 = ld_relaxed(&a->ready[f * a->nrt + m0]), v1 = ld_relaxed(&a->ready[f * a->nrt + m1]);
                if (v0 < a->ready_target || v1 < a->ready_target) return false;  // retried from ring_wait
                fence_acquire();
                asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> bulk copy
            }
            apply_issue_models<Q>(*a, g, f, dst, bar, pm);
            row = g.y0;
        } else {
            apply_issue_row<Q>(*a, g, f, row, dst, bar, pg);
            ++row;
        }
        if (row >= g.y1) {
            it += step;
            decode();
        }
        return true;
    }
};

template <int Q, int D>
__global__ void __launch_bounds__(FitCfg<Q>::THREADS, 1) k_fit_stream(const __grid_constant__ FitArgs a, int n)
{
    using C = FitCfg<Q>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const RingSmem<C> sm(smem_raw);
    sm.init_barriers();
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per_frame = a.By * a.nseg, nitems = n * per_frame;
    const int GW = gridDim.x * C::NSW, first = blockIdx.x * C::NSW + w;
    Ring r = sm.ring(w);
    FitSeq<Q, D> seq;
    seq.a = &a, seq.it = first, seq.nitems = nitems, seq.per_frame = per_frame, seq.step = GW;
    seq.pg = std_policy_guides_fit(), seq.py = policy_evict_first();
    seq.decode();
    pdl_wait();  // caller data may come from the previous grid: wait before the first read
    pdl_trigger();  // dependents launch only once we are past our own wait
    if (lane == 0) ring_fill(r, seq);
#ifdef FLR_DBG_TIMES
    const long long tk0 = clock64();
    int nit = 0;
#endif
    for (int it = first; it < nitems; it += GW) {
        const int f = it / per_frame, rem = it % per_frame;
        fit_consume<Q, D>(r, seq, a, f, rem / a.nseg, rem % a.nseg, lane);
        if (a.done) {  // publish the item's moments to the K2 wavefront (release is cumulative
            __syncwarp();  // over the lanes' stores ordered before it by the warp barrier)
            if (lane == 0) red_release_add(&a.done[f * a.By + rem / a.nseg], 1);
        }
#ifdef FLR_DBG_TIMES
        ++nit;
#endif
    }
#ifdef FLR_DBG_TIMES
    extern __device__ unsigned long long g_flr_total_cycles[4096];
    extern __device__ int g_flr_items[4096];
    if (lane == 0) {
        g_flr_total_cycles[(blockIdx.x * 32 + w) & 4095] = clock64() - tk0;
        g_flr_items[(blockIdx.x * 32 + w) & 4095] = nit;
    }
#endif
}

#ifndef FLR_FITLDG_WARPS
#define FLR_FITLDG_WARPS 8
#endif
constexpr int kFitLdgWarps = FLR_FITLDG_WARPS;

// K1 without shared memory: persistent, one warp per FIT item, LDG prefetch of the next row
template <int Q, int D>
__global__ void __launch_bounds__(kFitLdgWarps * 32, 1) k_fit_ldg(const __grid_constant__ FitLdgArgs a, int n)
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per_frame = a.By * a.nseg, nitems = n * per_frame;
    const int GW = gridDim.x * kFitLdgWarps;
    pdl_wait();
    pdl_trigger();  // dependents launch only once we are past our own wait
    for (int it = blockIdx.x * kFitLdgWarps + w; it < nitems; it += GW) {
        const int f = it / per_frame, rem = it - f * per_frame, by = rem / a.nseg;
        fit_ldg_item<Q, D>(a, f, by, rem - by * a.nseg, lane);
    }
}

template <int Q>
__global__ void __launch_bounds__(ApplyCfg<Q>::THREADS, 1) k_apply_stream(const __grid_constant__ ApplyArgs a, int n)
{
    using C = ApplyCfg<Q>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const RingSmem<C> sm(smem_raw);
    sm.init_barriers();
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per_frame = a.nband * a.nsub * a.nseg, nitems = n * per_frame;
    const int GW = gridDim.x * C::NSW, first = blockIdx.x * C::NSW + w;
    Ring r = sm.ring(w);
    ApplySeq<Q> seq;
    seq.a = &a, seq.it = first, seq.nitems = nitems, seq.per_frame = per_frame, seq.step = GW;
    seq.pg = policy_evict_first(), seq.pm = policy_evict_normal();  // last use of the guides
    seq.decode();
    if (!a.ready) pdl_wait();  // models come from the previous grid (or per tile row, see ApplySeq)
    pdl_trigger();
    if (lane == 0) ring_fill(r, seq);
    for (int it = first; it < nitems; it += GW) {
        const int f = it / per_frame, rem = it % per_frame;
        float* mod = sm.extra(w);
        apply_consume<Q>(r, seq, a, f, rem / a.nseg, rem % a.nseg, lane, mod, mod + 2 * kApplyNCol * StreamDims<Q>::MS);
    }
}

}  // namespace flr
