// flr_wave.cuh -- the whole FLR pass (moments -> blur + solve -> apply) as ONE
// persistent kernel per call, scheduled as a row wavefront across all SMs.
//
// Why: the staged schedule (three grids) leaves HBM idle while the fp64 blur + solve grid
// runs (~25 % of a 1080p step), pays each grid's ramp and tail, and re-reads the guides
// from DRAM in the apply because they were read ~30 us earlier.  Here every CTA (one per
// SM, 8 warps) loops over TASKS claimed from three global queues:
//   FIT   chunk  : 7 FIT items (block row x 128 px, one per consumer warp; flr_fitws.cuh)
//   K2    tile   : one 32 x 8 tile of blocks, blur + solve by all 256 threads (flr_k2.cuh)
//   APPLY chunk  : 7 APPLY items (4 output rows x 128 px, one per consumer warp)
// A task is claimed only when its inputs are complete (per-row FIT counters, per-tile-row
// K2 counters in the workspace; acquire/release), so no CTA ever waits on an unclaimed
// task and the schedule cannot deadlock, whatever the residency.  The scheduler prefers
// the most downstream ready task (APPLY > K2 > FIT): K2 tiles run as soon as their block
// rows are fitted, under the rest of the fit's streaming, and the apply follows the fit by
// a few block rows, so the guides it re-reads are still in L2.  In a batched call the
// queues span all frames, so frame i+1's fit streams under frame i's blur + solve.
//
// Warp roles inside a CTA: warp 7 = scheduler + TMA producer (lane c feeds consumer warp c
// through a ring of 2-row stages + a 2-stage model ring, as in k_fit_ws / k_apply_ws;
// consecutive stream tasks are issued back to back, so the rings stay full across task
// boundaries); warps 0-6 = consumers.  Tasks reach the consumers through a 4-slot
// descriptor queue in shared memory.  A K2 task drains the rings (its shared memory
// overlaps them) and is then run by all 8 warps.
#pragma once
#include "flr_applyws.cuh"
#include "flr_fitws.cuh"
#include "flr_k2.cuh"

namespace flr {

constexpr int kWaveNC = 7;  // consumer warps (+ 1 scheduler / producer warp)
constexpr int kWaveTQ = 4;  // task-descriptor queue slots
enum WaveTask : int { kTaskFit = 0, kTaskApply = 1, kTaskK2 = 2, kTaskDone = 3, kTaskNone = 4 };

#ifdef FLR_WAVE_TRACE
// timeline diagnostics: per CTA up to 96 records {type, index, t_claim_begin, t_claimed} after
// the flags (globaltimer ns; tools/wave_timeline.py reads them)
#define WTRACE_REC(i, ty, ix, t0, t1)                                                              \
    do {                                                                                          \
        if ((i) < 96) {                                                                           \
            long long* r_ = reinterpret_cast<long long*>(w.flags + 4 + w.n * (w.fit.By + 3 * w.ntr + 2)) + \
                            (blockIdx.x * 96 + (i)) * 2;                                          \
            r_[0] = ((long long)(ty) << 32) | (unsigned)(ix);                                     \
            r_[1] = ((t1) << 16) | (((t1) - (t0)) & 0xffff);                                      \
        }                                                                                         \
    } while (0)
#define WTRACE_BASE (f == 0 ? reinterpret_cast<long long*>(w.flags + 4 + w.n * (w.fit.By + 3 * w.ntr + 2)) : nullptr)
#else
#define WTRACE_REC(i, ty, ix, t0, t1) ((void)0)
#define WTRACE_BASE nullptr
#endif

template <int Q, int R>
struct WaveCfg {
    using SD = StreamDims<Q>;
    using FC = FitWsCfg<Q>;
    using KG = K2Geom<Q, R>;
    static_assert(FC::RB == 2 && FC::S == 2, "the wave ring is the fit kernel's 2 x 2-row ring");
    static constexpr int NC = kWaveNC, THREADS = (NC + 1) * 32;
    static constexpr int RB = 2, S = 2, SM = 2;
    static constexpr int GF = kSeg;                         // floats per guide plane row
    static constexpr int ROWF = FC::STG;                    // row-stage stride (a FIT stage: Q + 3 planes x 2 rows)
    static constexpr int MODF = 2 * kApplyNCol * SD::MS;    // model stage (two rows of 18 models)
    static constexpr int WARPF = (S * ROWF + SM * MODF + 31) / 32 * 32;
    static constexpr size_t RING_BYTES = (size_t)NC * WARPF * sizeof(float);
    static constexpr size_t K2_BYTES = (KG::BAR_OFF + 127) / 128 * 128;
    static constexpr size_t UNION = RING_BYTES > K2_BYTES ? RING_BYTES : K2_BYTES;
    static constexpr int NBAR_C = 2 * (S + SM);             // per consumer: full / empty, row + model
    static constexpr int NBAR = NC * NBAR_C + KG::S + 2 * kWaveTQ;
    static constexpr size_t BAR_OFF = UNION;
    static constexpr size_t TQ_OFF = (BAR_OFF + (size_t)NBAR * sizeof(uint64_t) + 15) / 16 * 16;
    static constexpr size_t SMEM = TQ_OFF + kWaveTQ * sizeof(int4);
    static_assert(SMEM <= 232448, "wave kernel exceeds 227 KB of shared memory");
    // apply_consume_item's view of the ring (guide plane j, row r of a stage)
    __host__ __device__ static constexpr int g_off(int j, int r) { return (j * RB + r) * GF; }
    __host__ __device__ static constexpr int m_off(int c, int r) { return RB * Q * GF + (c * RB + r) * kSeg; }
};

struct WaveArgs {
    FitArgs fit;      // fit-resolution planes (box height 2), moment field
    ApplyArgs app;    // output-resolution guides (box height 2), padded models, output
    CUtensorMap tmom; // fp64 moment field, box K2Geom<Q, R>::{HX, NV, G}
    Taps taps;
    double eps_add, eps_mul;
    int n;
    int nfit, nfc;    // FIT items, chunks
    int napp;         // APPLY items
    int ntr, ntc;     // K2 tile rows / columns per frame
    int* flags;       // zeroed per call, see the wave_* accessors below
};

// Work queues (all claims are atomicAdd tickets, so claiming is parallel, never a serial
// CAS race between CTAs):
//   FIT   : chunk tickets, always ready (inputs).
//   K2    : per tile ROW (group g = f * ntr + tr) a ticket counter over its ntc tiles; the
//           group at the head is claimable once the FIT rows it reads are complete.
//   APPLY : per tile row a group of APPLY items (the bands whose lower model row falls in
//           tile row tr), ticket counter over its 7-item chunks; claimable once the K2 tile
//           rows it blends are complete.
// A group's tickets past its size exhaust it and move the head on (one CAS per group).
// flags: [0] FIT tickets [1] APPLY head group [2] K2 head group [3] unused |
//   fit_row[n][By] items done per block row | fit_pre[n] complete leading block rows |
//   k2_row[n*ntr] tiles done | k2_pre[n] complete leading tile rows |
//   k2_tkt[n*ntr] | app_tkt[n*ntr]
__device__ __forceinline__ int* wave_fit_row(const WaveArgs& w) { return w.flags + 4; }
__device__ __forceinline__ int* wave_fit_pre(const WaveArgs& w) { return w.flags + 4 + w.n * w.fit.By; }
__device__ __forceinline__ int* wave_k2_row(const WaveArgs& w) { return wave_fit_pre(w) + w.n; }
__device__ __forceinline__ int* wave_k2_pre(const WaveArgs& w) { return wave_k2_row(w) + w.n * w.ntr; }
__device__ __forceinline__ int* wave_k2_tkt(const WaveArgs& w) { return wave_k2_pre(w) + w.n; }
__device__ __forceinline__ int* wave_app_tkt(const WaveArgs& w) { return wave_k2_tkt(w) + w.n * w.ntr; }

// Row counters: a finished unit (FIT item / K2 tile) adds 1 to its row with a release
// reduction (red.release: no return value, no acquire; an acquire-release atomic per item
// here stalled the streaming SMs ~5x).  Readiness of "the first `need` rows of frame f" is
// polled by the scheduler lane with RELAXED loads (acquire loads invalidate the SM's L1 on
// every poll), remembering how far it has seen complete rows (`seen`, per frame, private to
// the lane); one acquire fence after a successful claim then orders the claimer after every
// unit whose count it observed (fence-based acquire: relaxed reads of release writes).
struct WavePrefix {
    int f = -1, p = 0;  // frame, rows [0, p) seen complete
};
__device__ __forceinline__ bool wave_rows_ready(WavePrefix& seen, int f, const int* row, int need_rows, int units)
{
    if (seen.f != f) seen.f = f, seen.p = 0;
    while (seen.p < need_rows && ld_relaxed(&row[seen.p]) >= units) ++seen.p;
    return seen.p >= need_rows;
}

// APPLY group g = (f, tr): the item range [i0, i1) of the bands whose lower model row
// min(j, By - 1) lies in tile row tr (bands are nsub * nseg consecutive items each)
__device__ __forceinline__ void wave_app_group(const WaveArgs& w, int g, int& i0, int& i1)
{
    const int f = g / w.ntr, tr = g - f * w.ntr, per_band = w.app.nsub * w.app.nseg;
    const int j0 = tr * kK2TY, j1 = tr == w.ntr - 1 ? w.app.nband : min((tr + 1) * kK2TY, w.app.nband);
    const int base = f * w.app.nband * per_band;
    i0 = base + j0 * per_band;
    i1 = base + j1 * per_band;
}

// APPLY item index -> frame and geometry (items in frame, sub-band, segment order: top-down)
__device__ __forceinline__ ApplyGeom wave_apply_geom(const WaveArgs& w, int it, int& f)
{
    const int per = w.app.nband * w.app.nsub * w.app.nseg;
    f = it / per;
    const int rem = it - f * per;
    return apply_geom(w.app, rem / w.app.nseg, rem - (rem / w.app.nseg) * w.app.nseg);
}

// claim the most downstream ready task (scheduler lane only); never waits on unclaimed work.
// Returns {type, index, sub-index}; non-blocking (`block` false): kTaskNone instead of
// waiting when nothing is ready.
struct WaveSeen {
    WavePrefix fit, k2;  // complete FIT rows / K2 tile rows seen by this scheduler lane
};
template <int R>
__device__ __forceinline__ int4 wave_claim_(const WaveArgs& w, WaveSeen& seen, bool block);
#ifdef FLR_WAVE_TRACE
__device__ int g_wave_ntrace[1024];
#endif
template <int R>
__device__ __forceinline__ int4 wave_claim(const WaveArgs& w, WaveSeen& seen, bool block = true)
{
#ifdef FLR_WAVE_TRACE
    const long long t0 = gtimer();
    const int4 t = wave_claim_<R>(w, seen, block);
    const long long t1 = gtimer();
    if (t.x != kTaskNone) {
        const int i = g_wave_ntrace[blockIdx.x]++;
        WTRACE_REC(i, t.x, t.x == kTaskK2 ? t.z * 100 + t.w : t.y, t0, t1);
    }
    return t;
#else
    return wave_claim_<R>(w, seen, block);
#endif
}
template <int R>
__device__ __forceinline__ int4 wave_claim_(const WaveArgs& w, WaveSeen& seen, bool block)
{
    int* ctr = w.flags;
    const int ngrp = w.n * w.ntr;
    int nap = 32;
    for (;;) {
        // APPLY: the head group, once the K2 tile rows it blends are complete
        int g = ld_relaxed(&ctr[1]);
        while (g < ngrp) {
            const int f = g / w.ntr, tr = g - f * w.ntr;
            if (!wave_rows_ready(seen.k2, f, wave_k2_row(w) + f * w.ntr, tr + 1, w.ntc)) break;
            int i0, i1;
            wave_app_group(w, g, i0, i1);
            const int q = atomicAdd(&wave_app_tkt(w)[g], 1);
            if (q * kWaveNC < i1 - i0) {
                fence_acquire();  // after the K2 models counted above
                return make_int4(kTaskApply, i0 + q * kWaveNC, i1, 0);
            }
            atomicCAS(&ctr[1], g, g + 1);  // group exhausted: move the head on
            g = ld_relaxed(&ctr[1]);
        }
        if (g >= ngrp) return make_int4(kTaskDone, 0, 0, 0);  // every APPLY item claimed
        // K2: the head tile row, once the FIT rows within R of it are complete
        int k = ld_relaxed(&ctr[2]);
        while (k < ngrp) {
            const int f = k / w.ntr, tr = k - f * w.ntr;
            if (!wave_rows_ready(seen.fit, f, wave_fit_row(w) + f * w.fit.By, min((tr + 1) * kK2TY + R, w.fit.By),
                                 w.fit.nseg))
                break;
            const int q = atomicAdd(&wave_k2_tkt(w)[k], 1);
            if (q < w.ntc) {
                fence_acquire();  // after the FIT moments counted above
                return make_int4(kTaskK2, f, tr, q);
            }
            atomicCAS(&ctr[2], k, k + 1);
            k = ld_relaxed(&ctr[2]);
        }
        // FIT: always ready (the ticket counter may overshoot)
        if (ld_relaxed(&ctr[0]) < w.nfc) {
            const int c = atomicAdd(&ctr[0], 1);
            if (c < w.nfc) return make_int4(kTaskFit, c, 0, 0);
        }
        if (!block) return make_int4(kTaskNone, 0, 0, 0);
#ifdef FLR_WATCHDOG
        if (nap >= 1024) printf("FLR watchdog: claim block %d heads apply %d k2 %d of %d\n", blockIdx.x, g, k, ngrp);
#endif
        __nanosleep(nap);  // nothing ready: back off (in-flight work completes elsewhere)
        nap = min(nap * 2, 512);
    }
}

// The three task bodies are separate (non-inlined) functions: each gets the whole register
// file for itself instead of sharing it with the scheduler's and the other roles' live state
// (inlined into one kernel body they spilled ~0.5-1.2 KB per thread).
template <int Q, int D>
__device__ __noinline__ void wave_fit_item(const FitArgs& a, int it, int per_frame, const float* ring, uint64_t* full,
                                           uint64_t* empty, int& k, int lane)
{
    bool waited = true;
    fit_consume_item<Q, D, false, false>(a, it, per_frame, ring, full, empty, k, lane, waited);
}
template <int Q, class C>
__device__ __noinline__ void wave_apply_item(const ApplyArgs& a, int it, int f, const float* rows_st,
                                             const float* mod_st, uint64_t* rfull, uint64_t* rempty, uint64_t* mfull,
                                             uint64_t* mempty, int& kr, int& km, int lane)
{
    const ApplyGeom g = apply_geom(a, (it - f * a.nband * a.nsub * a.nseg) / a.nseg,
                                   (it - f * a.nband * a.nsub * a.nseg) % a.nseg);
    apply_consume_item<Q, false, false, C>(a, g, f, rows_st, mod_st, rfull, rempty, mfull, mempty, kr, km, lane);
}

// one K2 tile (frame f, tile row tr, column tc) by all 256 threads; publishes the tile
template <int Q, int R>
__device__ __noinline__ void wave_k2(const WaveArgs& w, int f, int tr, int tc, unsigned char* smem, uint64_t* kbar)
{
    // The producer and consumer warps reach this barrier from different code paths: make each
    // warp converged first (bar.sync is .aligned), and use the barrier form that counts
    // threads even if a warp were to arrive in parts.
    __syncwarp();
    asm volatile("barrier.sync 0;" ::: "memory");  // every ring stage consumed: the shared memory is free
    // (the scheduler lane's acquire of the FIT row counters is ordered before this thread's
    // TMA by the CTA barrier; the proxy fence orders the generic moment stores before it)
    if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
    k2_tile<Q, R>(&w.tmom, f, tc * kK2TX, tr * kK2TY, w.fit.Bx, w.fit.By, const_cast<float*>(w.app.models),
                  StreamDims<Q>::MS, w.eps_add, w.eps_mul, w.taps, reinterpret_cast<double*>(smem), kbar,
                  policy_evict_first());
    __syncwarp();
    asm volatile("barrier.sync 0;" ::: "memory");  // models stored; shared memory free for the rings again
    if (threadIdx.x == 0) red_release_add(&wave_k2_row(w)[f * w.ntr + tr], 1);
}

template <int Q, int D, int R>
__global__ void __launch_bounds__(WaveCfg<Q, R>::THREADS, 1) k_flr_wave(const __grid_constant__ WaveArgs w)
{
    using C = WaveCfg<Q, R>;
    using FC = FitWsCfg<Q>;
    constexpr int NC = C::NC, S = C::S, SM = C::SM, TQ = kWaveTQ;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* kbar = bars + NC * C::NBAR_C;
    uint64_t* tq_full = kbar + C::KG::S;
    uint64_t* tq_empty = tq_full + TQ;
    int4* tq = reinterpret_cast<int4*>(smem + C::TQ_OFF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NC * C::NBAR_C; ++i) mbar_init(&bars[i], 1);
        for (int i = 0; i < TQ; ++i) {
            mbar_init(&tq_full[i], 1);
            mbar_init(&tq_empty[i], NC);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();     // the workspace and the inputs may come from the previous grid
    pdl_trigger();  // dependents may start as SMs free up; they wait for our completion

    const int per_fit = w.fit.By * w.fit.nseg;
    if (warp == NC) {
        // ---------------- scheduler (lane 0) + producer (lane c feeds consumer c) ----------------
        const int c = lane;
        float* base = reinterpret_cast<float*>(smem) + (size_t)(c < NC ? c : 0) * C::WARPF;
        float* rows_st = base;
        float* mod_st = base + S * C::ROWF;
        uint64_t* rfull = bars + (c < NC ? c : 0) * C::NBAR_C;
        uint64_t* rempty = rfull + S;
        uint64_t* mfull = rempty + S;
        uint64_t* mempty = mfull + SM;
        const uint64_t pg_fit = policy_evict_last(), py_fit = policy_evict_first();  // guides stay for the apply
        const uint64_t pg_app = policy_evict_first(), pm = policy_evict_normal();
        int kr = 0, km = 0, nt = 0;
        WaveSeen seen;                     // scheduler lane's view of the row counters
        int4 nxt = make_int4(0, 0, 0, 0);  // scheduler lane: one task claimed ahead
        if (lane == 0) nxt = wave_claim<R>(w, seen);
        for (;;) {
            int4 t = make_int4(0, 0, 0, 0);
            if (lane == 0) {
                t = nxt;
                const int slot = nt % TQ;
                if (nt >= TQ) mbar_wait(&tq_empty[slot], ((nt / TQ) - 1) & 1);
                tq[slot] = t;
                mbar_arrive(&tq_full[slot]);  // release: the descriptor is visible to the consumers
                // try to claim the next task now (its latency overlaps this task's stages still
                // queued), but never WAIT before issuing this task: its rows may be what the next
                // ready task depends on
#ifdef FLR_WAVE_LOOKAHEAD
                nxt = t.x != kTaskDone ? wave_claim<R>(w, seen, false) : make_int4(kTaskNone, 0, 0, 0);
#else
                // no claim ahead: a CTA that has just issued its task takes the most downstream
                // task ready THEN (a claim made earlier would hold, e.g., a second FIT chunk
                // while K2 tiles wait for a free CTA -- measured slower)
                nxt = make_int4(kTaskNone, 0, 0, 0);
#endif

            }
            ++nt;
            t.x = __shfl_sync(0xffffffffu, t.x, 0);
            t.y = __shfl_sync(0xffffffffu, t.y, 0);
            t.z = __shfl_sync(0xffffffffu, t.z, 0);
            t.w = __shfl_sync(0xffffffffu, t.w, 0);
            __syncwarp();  // orders lane 0's acquire of the K2 / APPLY inputs before every lane's copies
            if (t.x == kTaskDone) break;
            if (t.x == kTaskK2) {
                wave_k2<Q, R>(w, t.y, t.z, t.w, smem, kbar);
                if (lane == 0 && nxt.x == kTaskNone) nxt = wave_claim<R>(w, seen);
                continue;
            }
            // stream chunk: lane c issues every stage of its item, non-blocking round robin
            const int it = t.x == kTaskFit ? t.y * NC + c : t.y + c;  // APPLY: items [t.y, t.z)
            int f = 0, by = 0, sg = 0, rows = 0, row = 0, todo = 0;  // todo: row stages left
            bool models = false;                                      // APPLY: the model stage is still due
            ApplyGeom g;
            if (c < NC) {
                if (t.x == kTaskFit && it < w.nfit) {
                    f = it / per_fit;
                    const int rem = it - f * per_fit;
                    by = rem / w.fit.nseg;
                    sg = rem - by * w.fit.nseg;
                    rows = min(D, w.fit.H - by * D);
                    todo = (rows + 1) / 2;
                } else if (t.x == kTaskApply && it < t.z) {
                    g = wave_apply_geom(w, it, f);
                    if (g.y0 < g.y1) todo = (g.y1 - g.y0 + 1) / 2, models = true;
                    row = g.y0;
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // K2's model stores -> bulk copies
                }
            }
            constexpr unsigned mask = 0xffffffffu;
#ifdef FLR_WATCHDOG
            long long tw = clock64();
#endif
            while (__any_sync(mask, todo > 0)) {
#ifdef FLR_WATCHDOG
                if (clock64() - tw > (1ll << 32) && todo > 0) {
                    printf("FLR watchdog: producer block %d lane %d task %d/%d todo %d models %d kr %d km %d\n",
                           blockIdx.x, c, t.x, t.y, todo, (int)models, kr, km);
                    __trap();
                }
#endif
                if (todo <= 0) continue;
                if (models) {  // an APPLY item's models first
                    const int s = km % SM;
                    if (km < SM || mbar_test_wait(&mempty[s], ((km / SM) - 1) & 1)) {
                        ws_proxy_fence();
                        apply_issue_models<Q>(w.app, g, f, mod_st + s * C::MODF, &mfull[s], pm);
                        ++km;
                        models = false;
                    }
                    continue;
                }
                const int s = kr % S;
                if (kr < S || mbar_test_wait(&rempty[s], ((kr / S) - 1) & 1)) {
                    ws_proxy_fence();
                    if (t.x == kTaskFit)
                        fit_issue_row<Q, D, false, false, kFS, 2>(w.fit, f, by, sg, row, rows_st + s * C::ROWF,
                                                                  &rfull[s], pg_fit, py_fit);
                    else
                        apply_issue_row<Q, false, false, 2>(w.app, g, f, row, rows_st + s * C::ROWF, &rfull[s], pg_app);
                    row += 2;
                    ++kr;
                    --todo;
                }
            }
            __syncwarp();
            if (lane == 0 && nxt.x == kTaskNone) nxt = wave_claim<R>(w, seen);
        }
    } else {
        // ---------------- consumer warp ----------------
        const int cw = warp;
        float* base = reinterpret_cast<float*>(smem) + (size_t)cw * C::WARPF;
        const float* rows_st = base;
        const float* mod_st = base + S * C::ROWF;
        uint64_t* rfull = bars + cw * C::NBAR_C;
        uint64_t* rempty = rfull + S;
        uint64_t* mfull = rempty + S;
        uint64_t* mempty = mfull + SM;
        int kr = 0, km = 0;
        for (int nt = 0;; ++nt) {
            const int slot = nt % TQ;
            mbar_wait(&tq_full[slot], (nt / TQ) & 1);
            const int4 t = tq[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&tq_empty[slot]);

            if (t.x == kTaskDone) break;
            if (t.x == kTaskK2) {
                wave_k2<Q, R>(w, t.y, t.z, t.w, smem, kbar);
                continue;
            }
            const int it = t.x == kTaskFit ? t.y * NC + cw : t.y + cw;
            if (t.x == kTaskFit) {
                if (it >= w.nfit) continue;
                wave_fit_item<Q, D>(w.fit, it, per_fit, rows_st, rfull, rempty, kr, lane);
                __syncwarp();
                if (lane == 0) {  // publish the item's moments to the K2 queue (release: after every lane's stores)
                    const int f = it / per_fit, by = (it - f * per_fit) / w.fit.nseg;
                    red_release_add(&wave_fit_row(w)[f * w.fit.By + by], 1);
                }
            } else {
                if (it >= t.z) continue;
                int f;
                const ApplyGeom g = wave_apply_geom(w, it, f);
                if (g.y0 >= g.y1) continue;
                wave_apply_item<Q, C>(w.app, it, f, rows_st, mod_st, rfull, rempty, mfull, mempty, kr, km, lane);
            }
        }
    }
}

}  // namespace flr
