// flr_persist.cuh -- k_apply_stream: K4 blended apply (APPLY items) for batched calls,
// a persistent, TMA-fed streaming kernel (one CTA per SM).  Every warp is a stream
// warp with its own bulk-copy ring (flr_stream.cuh).  Items are assigned round-robin
// to warp slots (blockIdx.x*NSW + w); each warp's lane 0 walks the same sequence
// ahead of the consumer to keep S rows in flight.
#pragma once
#include "flr_stream.cuh"

namespace flr {

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
    pdl_wait();  // the models come from the previous grid
    pdl_trigger();
    if (lane == 0) ring_fill(r, seq);
    for (int it = first; it < nitems; it += GW) {
        const int f = it / per_frame, rem = it % per_frame;
        float* mod = sm.extra(w);
        apply_consume<Q>(r, seq, a, f, rem / a.nseg, rem % a.nseg, lane, mod, mod + 2 * kApplyNCol * StreamDims<Q>::MS);
    }
}

}  // namespace flr
