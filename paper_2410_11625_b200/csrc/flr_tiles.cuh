// flr_tiles.cuh -- tiled sm_100a kernels of the staged FLR schedule:
//   K1 k_fit_moments : outer products + strided box downsample
//   K2 k_blur_rows + k_solve_rows / k_solve: row-strip blur of the moment field, then the
//                      per-block solve
//   K4 k_apply_tile  : bilinear model blend + application
// Full-resolution planes are streamed once per pass with 16-byte loads; all
// intermediates live at block resolution.
#pragma once
#include <cuda.h>

#include "flr_common.cuh"
#include "flr_pipe.cuh"
#include "flr_solve.cuh"

namespace flr {

__device__ __forceinline__ float4 ld_stream4(const float* p)
{
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void st_stream4(float* p, float4 v)
{
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// decode an S component (0 <= s < NS) into (i, j), i <= j, row-major upper triangle
__device__ __forceinline__ void s_decode(int Q, int s, int& i, int& j)
{
    i = 0;
    while (s >= Q - i) {
        s -= Q - i;
        ++i;
    }
    j = i + s;
}

// ===========================================================================
// K1: one CTA = one block row x one 128-pixel segment.  Warp w walks pixel rows
// w*RPW .. of the block row; lane l owns pixel quad (x0 .. x0+3), x0 = 128 s + 4 l,
// and D/4 lanes share a block.  Each lane accumulates in fp32 about the block's
// shift c = x(top-left pixel of the block) (design rule H1), lanes of a block
// combine with xor shuffles, warps combine through shared memory in fp64, and
// the shift is undone exactly in fp64 (x = d + c):
//   u_j = u'_j + n c_j,  S_ij = S'_ij + c_i u'_j + c_j u'_i + n c_i c_j,  XY_jc = XY'_jc + c_j Y_c.
// Output: fp64 moments [f][KM][By][Bx].  D in {4, 8, 16}.
// ===========================================================================
template <int D>
struct FitGeom {
    static constexpr int NW = D >= 8 ? 8 : D;  // warps per CTA
    static constexpr int RPW = D / NW;         // pixel rows per warp
    static constexpr int DQ = D / 4;           // lanes per block
    static constexpr int NB = 32 / DQ;         // blocks per 128-px segment
    static constexpr int THREADS = NW * 32;
};

template <int Q, int D>
constexpr size_t fit_smem_bytes()
{
    using G = FitGeom<D>;
    constexpr int KA = Dims<Q>::KM - 1;
    constexpr int KP = KA | 1;  // odd row stride: conflict-free partial writes
    return (size_t)G::NW * G::NB * KP * sizeof(float) + (size_t)G::NB * KA * sizeof(double) +
           (size_t)G::NB * Q * sizeof(float);
}

template <int Q, int D, bool VEC>
__global__ void __launch_bounds__(FitGeom<D>::THREADS) k_fit_moments(int W, int H, int Bx, int Bxp, int By,
                                                                     const float* __restrict__ guides,
                                                                     const float* __restrict__ radiance,
                                                                     double* __restrict__ mom)
{
    using Dm = Dims<Q>;
    using G = FitGeom<D>;
    constexpr int KA = Dm::KM - 1;  // accumulated components (all but n), index a = k - 1
    constexpr int KP = KA | 1;
    constexpr int NS = Dm::NS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double* tot = reinterpret_cast<double*>(smem_raw);                      // [NB][KA]
    float* part = reinterpret_cast<float*>(tot + G::NB * KA);              // [NW][NB][KP]
    float* csh = part + G::NW * G::NB * KP;                                // [NB][Q]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = blockIdx.x, by = blockIdx.y, f = blockIdx.z;
    const int x0 = seg * 128 + lane * 4;
    const int bx = x0 / D;
    const int lb = lane / G::DQ;
    const bool has_block = bx < Bx;
    const bool active = x0 < W;
    const size_t plane = (size_t)W * H;
    const float* Gp = guides + (size_t)f * Q * plane;
    const float* Yp = radiance + (size_t)f * 3 * plane;

    float c[Q];
    {
        const size_t p0 = (size_t)(by * D) * W + (size_t)(has_block ? bx * D : 0);
#pragma unroll
        for (int j = 0; j < Q; ++j) c[j] = has_block ? __ldg(Gp + j * plane + p0) : 0.f;
    }
    if (warp == 0 && (lane % G::DQ) == 0) {
#pragma unroll
        for (int j = 0; j < Q; ++j) csh[lb * Q + j] = c[j];
    }
    float U[Q], S[NS], Yc[3], XY[3 * Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) U[j] = 0.f;
#pragma unroll
    for (int j = 0; j < NS; ++j) S[j] = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) Yc[j] = 0.f;
#pragma unroll
    for (int j = 0; j < 3 * Q; ++j) XY[j] = 0.f;

#pragma unroll
    for (int rr = 0; rr < G::RPW; ++rr) {
        const int y = by * D + warp * G::RPW + rr;
        if (y >= H) break;  // warp-uniform
        const size_t p = (size_t)y * W + x0;
        float g[Q][4], yv[3][4];
        if (VEC) {
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                const float4 v = active ? ld_stream4(Gp + j * plane + p) : make_float4(c[j], c[j], c[j], c[j]);
                g[j][0] = v.x; g[j][1] = v.y; g[j][2] = v.z; g[j][3] = v.w;
            }
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const float4 v = active ? ld_stream4(Yp + j * plane + p) : make_float4(0.f, 0.f, 0.f, 0.f);
                yv[j][0] = v.x; yv[j][1] = v.y; yv[j][2] = v.z; yv[j][3] = v.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool ok = active && (x0 + k < W);
#pragma unroll
                for (int j = 0; j < Q; ++j) g[j][k] = ok ? __ldg(Gp + j * plane + p + k) : c[j];
#pragma unroll
                for (int j = 0; j < 3; ++j) yv[j][k] = ok ? __ldg(Yp + j * plane + p + k) : 0.f;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float d[Q];
#pragma unroll
            for (int j = 0; j < Q; ++j) d[j] = g[j][k] - c[j];
#pragma unroll
            for (int j = 0; j < Q; ++j) U[j] += d[j];
#pragma unroll
            for (int i = 0; i < Q; ++i)
#pragma unroll
                for (int j = i; j < Q; ++j) {
                    const int s = Dm::s_idx(i, j) - Dm::C_S;
                    S[s] = fmaf(d[i], d[j], S[s]);
                }
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) Yc[cc] += yv[cc][k];
#pragma unroll
            for (int j = 0; j < Q; ++j)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) XY[j * 3 + cc] = fmaf(d[j], yv[cc][k], XY[j * 3 + cc]);
        }
    }
#pragma unroll
    for (int m = 1; m < G::DQ; m <<= 1) {
#pragma unroll
        for (int j = 0; j < Q; ++j) U[j] += __shfl_xor_sync(0xffffffffu, U[j], m);
#pragma unroll
        for (int j = 0; j < NS; ++j) S[j] += __shfl_xor_sync(0xffffffffu, S[j], m);
#pragma unroll
        for (int j = 0; j < 3; ++j) Yc[j] += __shfl_xor_sync(0xffffffffu, Yc[j], m);
#pragma unroll
        for (int j = 0; j < 3 * Q; ++j) XY[j] += __shfl_xor_sync(0xffffffffu, XY[j], m);
    }
    {
        const int gi = lane % G::DQ;
        float* dst = part + (warp * G::NB + lb) * KP;
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            if (a % G::DQ != gi) continue;
            const int k = a + 1;
            float v;
            if (k < Dm::C_S) v = U[k - Dm::C_U];
            else if (k < Dm::C_Y) v = S[k - Dm::C_S];
            else if (k < Dm::C_XY) v = Yc[k - Dm::C_Y];
            else v = XY[k - Dm::C_XY];
            dst[a] = v;
        }
    }
    __syncthreads();
    // rows -> block totals, in fp64 (fixed order: deterministic)
    for (int i = threadIdx.x; i < G::NB * KA; i += G::THREADS) {
        const int b = i % G::NB, a = i / G::NB;
        double acc = 0.0;
#pragma unroll
        for (int w = 0; w < G::NW; ++w) acc += (double)part[(w * G::NB + b) * KP + a];
        tot[b * KA + a] = acc;
    }
    __syncthreads();
    // un-shift (fp64) and store the moment field, coalesced along bx
    const int rows = min(D, H - by * D);
    const size_t cs = (size_t)By * Bxp;
    for (int i = threadIdx.x; i < G::NB * Dm::KM; i += G::THREADS) {
        const int b = i % G::NB, k = i / G::NB;
        const int bxg = seg * G::NB + b;
        if (bxg >= Bx) continue;
        const double n = (double)(min(D, W - bxg * D) * rows);
        const double* T = tot + b * KA;  // T[k-1] = shifted component k
        const float* cb = csh + b * Q;
        double v;
        if (k == Dm::C_N) {
            v = n;
        } else if (k < Dm::C_S) {
            const int j = k - Dm::C_U;
            v = fma(n, (double)cb[j], T[k - 1]);
        } else if (k < Dm::C_Y) {
            int ii, jj;
            s_decode(Q, k - Dm::C_S, ii, jj);
            const double ci = cb[ii], cj = cb[jj];
            v = T[k - 1];
            v = fma(ci, T[Dm::C_U + jj - 1], v);
            v = fma(cj, T[Dm::C_U + ii - 1], v);
            v = fma(n * ci, cj, v);
        } else if (k < Dm::C_XY) {
            v = T[k - 1];
        } else {
            const int j = (k - Dm::C_XY) / 3, cc = (k - Dm::C_XY) % 3;
            v = fma((double)cb[j], T[Dm::C_Y + cc - 1], T[k - 1]);
        }
        mom[((size_t)f * Dm::KM + k) * cs + (size_t)by * Bxp + bxg] = v;
    }
}

// blur half-width (blocks) handled by the tiled K2 kernels (flr_k2.cuh, k_blur_rows)
constexpr int kTileMaxR = 8;

// ===========================================================================
// K2a (row-strip blur): the separable Gaussian of P:334 over a strip of kRowsCH block
// rows of ONE moment plane, full width.  Phase 1: one thread per PAIR of columns
// slides down the strip (kRowsCH + 2R coalesced 16-byte loads -> 2 kRowsCH vertical
// outputs; rows outside the field are zero = R3), results in shared memory with a
// zero x halo.  Phase 2: one thread per (row, kRowsCW consecutive columns) slides
// along the row (16-byte shared loads) into a second buffer; phase 3 stores the strip
// with 16-byte coalesced stores.  Every input value is read from L2 about once
// ((kRowsCH + 2R) / kRowsCH), against (TY+2R)(TX+2R)/(TX TY) for 2-D halo tiles.
// grid: (ceil(By / kRowsCH), n * KM), kRowsThreads threads; smem: blur_rows_smem(Bx, R).
// Needs an even row pitch Bxp >= Bx + (Bx & 1) (mom_pitch) and 16-byte aligned planes.
// ===========================================================================
#ifndef FLR_ROWS_CH
#define FLR_ROWS_CH 16
#endif
constexpr int kRowsCH = FLR_ROWS_CH, kRowsCW = 16, kRowsThreads = 128;
// shared row layout: column u (u = x + RE, RE = R rounded up to even) at rows_idx(u);
// 2 pad doubles after every kRowsCW columns keep the 16-byte accesses of threads that
// own consecutive chunks on distinct bank groups (stride 18 doubles)
__host__ __device__ constexpr int rows_idx(int u) { return u + 2 * (u / kRowsCW); }
__host__ __device__ constexpr int rows_re(int R) { return (R + 1) & ~1; }
__host__ __device__ constexpr int blur_rows_xp(int Bx, int R)
{
    return rows_idx(((Bx + kRowsCW - 1) / kRowsCW) * kRowsCW + 2 * rows_re(R)) + 2;
}
inline size_t blur_rows_smem(int Bx, int R) { return (size_t)2 * kRowsCH * blur_rows_xp(Bx, R) * sizeof(double); }

template <int R>
__global__ void __launch_bounds__(kRowsThreads, 3) k_blur_rows(const double* __restrict__ mom, int Bx, int Bxp, int By,
                                                            double* __restrict__ out, const __grid_constant__ Taps t)
{
    constexpr int CH = kRowsCH, CW = kRowsCW, RE = rows_re(R), NV = CH + 2 * R, NW = CW + 2 * RE;
    extern __shared__ __align__(16) double smr[];
    const int XP = blur_rows_xp(Bx, R);
    double* vs = smr;            // [CH][XP]: vertical pass
    double* hs = smr + CH * XP;  // [CH][XP]: result, column x at rows_idx(x)
    const int y0 = blockIdx.x * CH, nrow = min(CH, By - y0);
    const size_t ps = (size_t)By * Bxp;
    const double* src = mom + (size_t)blockIdx.y * ps;
    double* dst = out + (size_t)blockIdx.y * ps;
    pdl_wait();  // the moment field comes from the previous grid
    pdl_trigger();  // dependents launch only once we are past our own wait
#ifdef FLR_DBG_PHASES
    long long ts0 = clock64(), gt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
#endif
    const bool interior = y0 >= R && y0 + CH + R <= By;
    for (int x = 2 * threadIdx.x; x < Bx; x += 2 * blockDim.x) {
        double2 v[NV];
        const double* col = src + x;
        if (interior) {
            const double* p = col + (size_t)(y0 - R) * Bxp;
#pragma unroll
            for (int i = 0; i < NV; ++i) v[i] = __ldg(reinterpret_cast<const double2*>(p + (size_t)i * Bxp));
        } else {
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int y = y0 - R + i;
                v[i] = (y >= 0 && y < By) ? __ldg(reinterpret_cast<const double2*>(col + (size_t)y * Bxp))
                                          : make_double2(0.0, 0.0);
            }
        }
        const bool odd = x + 1 >= Bx;  // the pad column of an odd-width field counts as zero
        double* o = vs + rows_idx(x + RE);
#pragma unroll
        for (int r = 0; r < CH; ++r) {
            double a = t.g[R] * v[r + R].x, b = t.g[R] * v[r + R].y;
#pragma unroll
            for (int d = 1; d <= R; ++d) {
                a = fma(t.g[R + d], v[r + R - d].x + v[r + R + d].x, a);
                b = fma(t.g[R + d], v[r + R - d].y + v[r + R + d].y, b);
            }
            *reinterpret_cast<double2*>(o + r * XP) = make_double2(a, odd ? 0.0 : b);
        }
    }
    {  // zero x halo (R3): u in [0, RE) and [2 ceil(Bx/2) + RE, nch CW + 2 RE)
        const int xe = (Bx + 1) & ~1, ue = ((Bx + CW - 1) / CW) * CW + 2 * RE, nz = RE + ue - (xe + RE);
        for (int i = threadIdx.x; i < CH * nz; i += blockDim.x) {
            const int r = i / nz, j = i - r * nz;
            vs[r * XP + rows_idx(j < RE ? j : xe + j)] = 0.0;
        }
    }
#ifdef FLR_DBG_PHASES
    long long ts1 = clock64();
#endif
    __syncthreads();
#ifdef FLR_DBG_PHASES
    long long ts2 = clock64();
#endif
    const int nch = (Bx + CW - 1) / CW;
    for (int task = threadIdx.x; task < nrow * nch; task += blockDim.x) {
        const int r = task / nch, c = task - r * nch;
        const double* h = vs + r * XP + c * (CW + 2);  // u = c CW + i at c (CW + 2) + i + 2 (i / CW)
        double w[NW];
#pragma unroll
        for (int i = 0; i < NW; i += 2) {
            const double2 q = *reinterpret_cast<const double2*>(h + i + 2 * (i / CW));
            w[i] = q.x;
            w[i + 1] = q.y;
        }
        double* o = hs + r * XP + c * (CW + 2);
#pragma unroll
        for (int e = 0; e < CW; e += 2) {
            double a = t.g[R] * w[e + RE], b = t.g[R] * w[e + 1 + RE];
#pragma unroll
            for (int d = 1; d <= R; ++d) {
                a = fma(t.g[R + d], w[e + RE - d] + w[e + RE + d], a);
                b = fma(t.g[R + d], w[e + 1 + RE - d] + w[e + 1 + RE + d], b);
            }
            *reinterpret_cast<double2*>(o + e) = make_double2(a, b);
        }
    }
#ifdef FLR_DBG_PHASES
    long long ts3 = clock64();
#endif
    __syncthreads();
#ifdef FLR_DBG_PHASES
    long long ts4 = clock64();
#endif
#ifndef FLR_DBG_NOSTORE
    for (int r = 0; r < nrow; ++r)
        for (int x = 2 * threadIdx.x; x < Bx; x += 2 * blockDim.x)
            *reinterpret_cast<double2*>(dst + (size_t)(y0 + r) * Bxp + x) =
                *reinterpret_cast<const double2*>(hs + r * XP + rows_idx(x));
#else
    if (hs[threadIdx.x] == 12345.0) dst[threadIdx.x] = 1.0;
#endif
#ifdef FLR_DBG_PHASES
    if (threadIdx.x == 0) {
        extern __device__ long long g_flr_phase[];
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        long long* q = g_flr_phase + 10 * (blockIdx.y * gridDim.x + blockIdx.x);
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        q[0] = ts0, q[1] = ts1, q[2] = ts2, q[3] = ts3, q[4] = ts4, q[5] = clock64(), q[6] = sm, q[7] = gt;
        q[8] = gt0;
    }
#endif
}

// one thread per block: the appendix solve on the blurred moments (coalesced across bx)
template <int Q>
__global__ void __launch_bounds__(128) k_solve(int Bx, int Bxp, int By, const double* __restrict__ blurred,
                                              float* __restrict__ models, int mstride, double eps_add,
                                              double eps_mul)
{
    const int bx = blockIdx.x * blockDim.x + threadIdx.x, by = blockIdx.y, f = blockIdx.z;
    pdl_wait();  // the blurred field comes from the previous grid
    pdl_trigger();  // dependents launch only once we are past our own wait
    if (bx >= Bx) return;
    const size_t cs = (size_t)By * Bxp;
    const double* src = blurred + (size_t)f * Dims<Q>::KM * cs + (size_t)by * Bxp + bx;
    double m[Dims<Q>::KM];  // issue every load before the first use: one memory latency, not KM
#pragma unroll
    for (int k = 0; k < Dims<Q>::KM; ++k) m[k] = __ldg(src + (size_t)k * cs);
    solve_block<Q>([&](int k) { return m[k]; }, eps_add, eps_mul,
                   models + ((size_t)(f * By + by) * Bx + bx) * mstride);
}

// K2b (row solve): one CTA per 128 consecutive blocks of a block row.  The blurred
// components arrive by 1-D bulk copies (TMA engine, two mbarriers: n, u, S first so
// the Cholesky can start while Y, XY land) into shared memory [KM][128], where each
// thread reads only its own column; B^ overwrites the XY slots it is made from and
// the model is staged in the thread's own (consumed) S slots, then stored coalesced.
// Keeping the components out of registers lets 3 CTAs share an SM (<= 168 regs).
constexpr int kSolveRowN = 128;
template <int Q>
constexpr size_t solve_rows_smem() { return (size_t)Dims<Q>::KM * kSolveRowN * sizeof(double) + 2 * sizeof(uint64_t); }

struct StagedModel {  // float i of a thread's model in the S slots of its column
    double* col;
    __device__ __forceinline__ float& operator[](int i) const
    {
        return reinterpret_cast<float*>(col + (i >> 1) * kSolveRowN)[i & 1];
    }
};

template <int Q>
__global__ void __launch_bounds__(kSolveRowN, 3) k_solve_rows(int Bx, int Bxp, int By, const double* __restrict__ blurred,
                                                             float* __restrict__ models, double eps_add, double eps_mul)
{
    using Dm = Dims<Q>;
    constexpr int KM = Dm::KM, NT = kSolveRowN, MS = Dm::MSTRIDE;
    extern __shared__ __align__(16) double sms[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sms + KM * NT);
    const int bx0 = blockIdx.x * NT, by = blockIdx.y, f = blockIdx.z, t = threadIdx.x;
    const int nb = min(NT, Bx - bx0), nbe = (nb + 1) & ~1;  // even count: 16-byte bulk sizes
    if (t == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    pdl_wait();  // the blurred field comes from the previous grid
    pdl_trigger();  // dependents launch only once we are past our own wait
    __syncthreads();
    const size_t cs = (size_t)By * Bxp;
    const double* src = blurred + (size_t)f * KM * cs + (size_t)by * Bxp + bx0;
    if (t < 32) {
        const unsigned bytes = nbe * sizeof(double);
        if (t == 0) {
            mbar_arrive_expect_tx(&bar[0], bytes * Dm::C_Y);
            mbar_arrive_expect_tx(&bar[1], bytes * (KM - Dm::C_Y));
        }
        __syncwarp();
        const uint64_t pol = policy_evict_first();
        for (int k = t; k < KM; k += 32) bulk_g2s(sms + k * NT, src + k * cs, bytes, &bar[k < Dm::C_Y ? 0 : 1], pol);
    }
    double* col = sms + t;
    if (t < nb) {
        SmemB B{col + Dm::C_XY * NT, NT};
        bool waited = false;  // constant-folded: the solve is fully unrolled
        mbar_wait(&bar[0], 0);
        solve_block_b<Q>(
            [&](int k) {
                if (k >= Dm::C_Y && !waited) {
                    mbar_wait(&bar[1], 0);
                    waited = true;
                }
                return col[k * NT];
            },
            eps_add, eps_mul, StagedModel{col + Dm::C_S * NT}, B);
    }
    __syncthreads();
    // coalesced store of the nb staged models: [bx0 + b][i], i < MS (pad floats = 0)
    float* dst = models + ((size_t)(f * By + by) * Bx + bx0) * MS;
    for (int L = t; L < nb * MS; L += NT) {
        const int b = L / MS, i = L - b * MS;
        dst[L] = i < 3 * (Q + 1) ? StagedModel{sms + Dm::C_S * NT + b}[i] : 0.0f;
    }
}

// ===========================================================================
// K4: apply.  block_out % 8 == 0.  Pixel columns are cut into 8-px units
// [8u - off, 8u - off + 8), off = (D/2) % 8, and rows into 8-row tiles starting at
// 8t - off: every pixel of a unit (resp. every row of a tile) shares the same pair
// of bracketing block centres (b+1/2)D - 1/2 (R4).  One CTA = 8 rows x 32 units;
// the 2 x NC block models it needs are staged in shared memory; each thread
// y-blends its two model columns once and applies them to its 8 pixels:
//   I = (1 - t_x) x~.A_y(i0) + t_x x~.A_y(i1),  A_y(i) = A(j0,i) + t_y (A(j1,i) - A(j0,i)).
// Models: [f][By][Bx][MSTRIDE] fp32.
// ===========================================================================
constexpr int kApplyUnits = 32, kApplyRows = 8, kApplyNC = 34;

template <int Q, bool VEC>
__global__ void __launch_bounds__(kApplyUnits* kApplyRows) k_apply_tile(int W, int H, int D, int Bx, int By,
                                                                       const float* __restrict__ models,
                                                                       const float* __restrict__ guides,
                                                                       float* __restrict__ out)
{
    using Dm = Dims<Q>;
    constexpr int MS = Dm::MSTRIDE, P = Q + 1;
    __shared__ __align__(16) float sA[2][kApplyNC][MS];
    const int off = (D / 2) % 8;
    const int f = blockIdx.z;
    const int unit = blockIdx.x * kApplyUnits + (threadIdx.x % kApplyUnits);
    const int y = blockIdx.y * kApplyRows - off + (int)(threadIdx.x / kApplyUnits);
    const int ytile0 = blockIdx.y * kApplyRows - off;  // first row of the tile (may be < 0)
    const float invD = 1.0f / (float)D;
    // bracketing block rows of the tile (same for all its rows): from its first in-image row
    const int yref = max(ytile0, 0);
    const float fyr = ((float)yref + 0.5f) * invD - 0.5f;
    const int jb = (int)floorf(fyr);
    const int j0 = min(max(jb, 0), By - 1), j1 = min(max(jb + 1, 0), By - 1);
    // first block column touched by the CTA
    const int xcta = max(blockIdx.x * kApplyUnits * 8 - off, 0);
    const int ic0 = min(max((int)floorf(((float)xcta + 0.5f) * invD - 0.5f), 0), Bx - 1);
    const float* Mf = models + (size_t)f * By * Bx * MS;
    for (int i = threadIdx.x; i < 2 * kApplyNC * (MS / 4); i += blockDim.x) {
        const int v = i % (MS / 4), col = (i / (MS / 4)) % kApplyNC, r = i / ((MS / 4) * kApplyNC);
        const int bxs = min(ic0 + col, Bx - 1);
        const int bys = r ? j1 : j0;
        reinterpret_cast<float4*>(&sA[r][col][0])[v] =
            __ldg(reinterpret_cast<const float4*>(Mf + ((size_t)bys * Bx + bxs) * MS) + v);
    }
    __syncthreads();
    const int xu = unit * 8 - off;  // first pixel of the unit (may be < 0)
    if (y < 0 || y >= H || xu >= W) return;
    const float fy = ((float)y + 0.5f) * invD - 0.5f;
    const float ty = fy - floorf(fy);
    const float fxu = ((float)max(xu, 0) + 0.5f) * invD - 0.5f;
    const int ib = (int)floorf(fxu);
    const int i0 = min(max(ib, 0), Bx - 1), i1 = min(max(ib + 1, 0), Bx - 1);
    const float* a00 = &sA[0][i0 - ic0][0];
    const float* a10 = &sA[1][i0 - ic0][0];
    const float* a01 = &sA[0][i1 - ic0][0];
    const float* a11 = &sA[1][i1 - ic0][0];
    float m0[3 * P], m1[3 * P];
#pragma unroll
    for (int v = 0; v < MS / 4; ++v) {
        const float4 p = reinterpret_cast<const float4*>(a00)[v], q = reinterpret_cast<const float4*>(a10)[v];
        const float4 r = reinterpret_cast<const float4*>(a01)[v], s = reinterpret_cast<const float4*>(a11)[v];
        const float pa[4] = {p.x, p.y, p.z, p.w}, qa[4] = {q.x, q.y, q.z, q.w};
        const float ra[4] = {r.x, r.y, r.z, r.w}, sa[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int k = 4 * v + e;
            if (k < 3 * P) {
                m0[k] = fmaf(ty, qa[e] - pa[e], pa[e]);
                m1[k] = fmaf(ty, sa[e] - ra[e], ra[e]);
            }
        }
    }
    const size_t plane = (size_t)W * H;
    const float* Gp = guides + (size_t)f * Q * plane + (size_t)y * W;
    float* Op = out + (size_t)f * 3 * plane + (size_t)y * W;
    const float flx = (float)ib;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int xq = xu + 4 * h;
        if (xq < 0 || xq >= W) continue;
        float g[Q][4];
        if (VEC) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const float4 v = ld_stream4(Gp + q * plane + xq);
                g[q][0] = v.x; g[q][1] = v.y; g[q][2] = v.z; g[q][3] = v.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
                for (int e = 0; e < 4; ++e) g[q][e] = (xq + e < W) ? __ldg(Gp + q * plane + xq + e) : 0.f;
        }
        float o[3][4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float tx = ((float)(xq + e) + 0.5f) * invD - 0.5f - flx;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                float p0 = m0[cc], p1 = m1[cc];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    p0 = fmaf(g[q][e], m0[(1 + q) * 3 + cc], p0);
                    p1 = fmaf(g[q][e], m1[(1 + q) * 3 + cc], p1);
                }
                o[cc][e] = fmaf(tx, p1 - p0, p0);
            }
        }
        if (VEC) {
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) st_stream4(Op + cc * plane + xq, make_float4(o[cc][0], o[cc][1], o[cc][2], o[cc][3]));
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (xq + e < W)
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) Op[cc * plane + xq + e] = o[cc][e];
        }
    }
}

}  // namespace flr
