// flr_staged.cuh -- the staged sm_100a FLR kernels: K1 block moments, K2a un-shift,
// K2b horizontal blur, K3 vertical blur + solve, K4 apply.  One launch each.
//
// Paper: arXiv 2410.11625 (P:<line> = PAPER.md).  The paper's own four OpenCL
// kernels are prior art for the split, not the blueprint: here K1 and
// K4 are the only full-resolution passes, everything between them works at block
// resolution in fp64 (design rule H1).
#pragma once
#include "flr_common.cuh"
#include "flr_solve.cuh"

namespace flr {

__device__ __forceinline__ float4 ldg_stream(const float* p)
{
    // read-once full-resolution stream: do not keep in L1
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void stg_stream(float* p, float4 v)
{
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// K1 for small blocks (D in {1, 2}): one thread per block, scalar loads.
template <int Q>
__global__ void __launch_bounds__(128) k_moments_small(int W, int H, int Bx, int By, int D,
                                                       const float* __restrict__ guides,
                                                       const float* __restrict__ radiance,
                                                       float* __restrict__ raw)
{
    using Dm = Dims<Q>;
    const int bx = blockIdx.x * blockDim.x + threadIdx.x;
    const int by = blockIdx.y;
    const int f = blockIdx.z;
    if (bx >= Bx) return;
    const size_t plane = (size_t)W * H;
    const float* G = guides + (size_t)f * Q * plane;
    const float* Y = radiance + (size_t)f * 3 * plane;
    const size_t p0 = (size_t)(by * D) * W + bx * D;
    float c[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) c[j] = __ldg(G + j * plane + p0);
    float U[Q] = {}, S[Dm::NS] = {}, Yc[3] = {}, XY[3 * Q] = {};
    const int rows = min(D, H - by * D), cols = min(D, W - bx * D);
    for (int r = 0; r < rows; ++r)
        for (int k = 0; k < cols; ++k) {
            const size_t p = p0 + (size_t)r * W + k;
            float d[Q], y[3];
#pragma unroll
            for (int j = 0; j < Q; ++j) d[j] = __ldg(G + j * plane + p) - c[j];
#pragma unroll
            for (int j = 0; j < 3; ++j) y[j] = __ldg(Y + j * plane + p);
#pragma unroll
            for (int j = 0; j < Q; ++j) U[j] += d[j];
#pragma unroll
            for (int i = 0; i < Q; ++i)
#pragma unroll
                for (int j = i; j < Q; ++j) S[Dm::s_idx(i, j) - Dm::C_S] = fmaf(d[i], d[j], S[Dm::s_idx(i, j) - Dm::C_S]);
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) Yc[cc] += y[cc];
#pragma unroll
            for (int j = 0; j < Q; ++j)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) XY[j * 3 + cc] = fmaf(d[j], y[cc], XY[j * 3 + cc]);
        }
    const size_t cs = (size_t)By * Bx;
    float* out = raw + (size_t)f * Dm::KRAW * cs + (size_t)by * Bx + bx;
    out[0] = (float)(rows * cols);
#pragma unroll
    for (int j = 0; j < Q; ++j) out[(size_t)(Dm::C_U + j) * cs] = U[j];
#pragma unroll
    for (int j = 0; j < Dm::NS; ++j) out[(size_t)(Dm::C_S + j) * cs] = S[j];
#pragma unroll
    for (int j = 0; j < 3; ++j) out[(size_t)(Dm::C_Y + j) * cs] = Yc[j];
#pragma unroll
    for (int j = 0; j < 3 * Q; ++j) out[(size_t)(Dm::C_XY + j) * cs] = XY[j];
#pragma unroll
    for (int j = 0; j < Q; ++j) out[(size_t)(Dm::C_SH + j) * cs] = c[j];
}

// ---------------------------------------------------------------------------
// K2a: un-shift in fp64 (x = d + c):
//   u_j = u'_j + n c_j,  S_ij = S'_ij + c_i u'_j + c_j u'_i + n c_i c_j,
//   XY_jc = XY'_jc + c_j Y_c.   One thread per block; SoA fp64 output [f][KM][By][Bx].
// ---------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(128) k_unshift(int Bx, int Bxp, int By, const float* __restrict__ raw,
                                                 double* __restrict__ mom)
{
    using Dm = Dims<Q>;
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    const int f = blockIdx.y;
    const int nblk_frame = Bx * By;
    if (b >= nblk_frame) return;
    const size_t cs = (size_t)nblk_frame;  // input component stride (the raw field is not pitched)
    const float* in = raw + (size_t)f * Dm::KRAW * cs + b;
    const size_t co = (size_t)By * Bxp;  // output component stride (pitched rows)
    double* out = mom + (size_t)f * Dm::KM * co + (size_t)(b / Bx) * Bxp + (b % Bx);
    const double n = (double)in[0];
    double c[Q], u[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        c[j] = (double)in[(size_t)(Dm::C_SH + j) * cs];
        u[j] = (double)in[(size_t)(Dm::C_U + j) * cs];
    }
    out[0] = n;
#pragma unroll
    for (int j = 0; j < Q; ++j) out[(size_t)(Dm::C_U + j) * co] = fma(n, c[j], u[j]);
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = i; j < Q; ++j) {
            const int k = Dm::s_idx(i, j);
            double s = (double)in[(size_t)k * cs];
            s = fma(c[i], u[j], s);
            s = fma(c[j], u[i], s);
            s = fma(n * c[i], c[j], s);
            out[(size_t)k * co] = s;
        }
    double yc[3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        yc[cc] = (double)in[(size_t)(Dm::C_Y + cc) * cs];
        out[(size_t)(Dm::C_Y + cc) * co] = yc[cc];
    }
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            const int k = Dm::C_XY + j * 3 + cc;
            out[(size_t)k * co] = fma(c[j], yc[cc], (double)in[(size_t)k * cs]);
        }
}

// ---------------------------------------------------------------------------
// K2b: horizontal pass of the separable Gaussian blur of the moment field
// (P:299-309), fp64, zero padding (R3).  One thread per element
// of [f][KM][By][Bx]; `rows` = n*KM*By.
// ---------------------------------------------------------------------------
static __global__ void __launch_bounds__(256) k_hblur(int Bx, int Bxp, size_t rows, const double* __restrict__ in,
                                               double* __restrict__ out, const __grid_constant__ Taps t)
{
    const int bx = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t row = blockIdx.y + (size_t)blockIdx.z * gridDim.y;
    if (bx >= Bx || row >= rows) return;
    const double* src = in + row * Bxp;
    double acc = 0.0;
    const int lo = max(-t.R, -bx), hi = min(t.R, Bx - 1 - bx);
    for (int d = lo; d <= hi; ++d) acc = fma(t.g[t.R + d], __ldg(src + bx + d), acc);
    out[row * Bxp + bx] = acc;
}

// ---------------------------------------------------------------------------
// K3: vertical blur pass + the appendix's normalised, regularised solve
// (P:612-720), one thread per block, fp64 in registers.  (C^ + eps I) is SPD for
// eps > 0 (R13), so Cholesky replaces the paper's recursive block inverse
// (P:583-591): the solution is unique, so any exact solver gives it.
// Output: raw-basis model A (R6): A[1+j][c] = A^[j][c]/sigma^_j,
// A[0][c] = mu_Y,c - sum_j mu_X,j A[1+j][c], stored as fp32 with `mstride` floats
// per block ([f][By][Bx][mstride]).
// ---------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(128) k_vblur_solve(int Bx, int Bxp, int By, const double* __restrict__ hb,
                                                     float* __restrict__ models, int mstride,
                                                     double eps_add, double eps_mul,
                                                     const __grid_constant__ Taps t)
{
    using Dm = Dims<Q>;
    const int bx = blockIdx.x * blockDim.x + threadIdx.x;
    const int by = blockIdx.y * blockDim.y + threadIdx.y;
    const int f = blockIdx.z;
    if (bx >= Bx || by >= By) return;
    const size_t cs = (size_t)Bxp * By;
    const double* base = hb + (size_t)f * Dm::KM * cs + bx;
    const int lo = max(-t.R, -by), hi = min(t.R, By - 1 - by);
    // every component's vertical pass once, then the solve on the values (an on-the-fly
    // blur inside the solve's component accessor unrolled into ~40 K instructions)
    double vb[Dm::KM];
#pragma unroll 1
    for (int k = 0; k < Dm::KM; ++k) {
        const double* src = base + (size_t)k * cs;
        double acc = 0.0;
        for (int d = lo; d <= hi; ++d) acc = fma(t.g[t.R + d], __ldg(src + (size_t)(by + d) * Bxp), acc);
        vb[k] = acc;
    }
    solve_block<Q>([&](int k) { return vb[k]; }, eps_add, eps_mul, models + ((size_t)(f * By + by) * Bx + bx) * mstride);
}

// ---------------------------------------------------------------------------
// K4 (general): upsample and model application, one
// thread per output pixel, any block_out, any model stride.  The four block
// models around the pixel are blended bilinearly (centres (b+1/2)D-1/2, clamped,
// R4) and applied: I = x~ A.
// ---------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(256) k_apply_px(int W, int H, int D, int Bx, int By,
                                                  const float* __restrict__ models, int mstride,
                                                  const float* __restrict__ guides,
                                                  float* __restrict__ out)
{
    constexpr int P = Q + 1;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int f = blockIdx.z;
    if (x >= W) return;
    const float fx = ((float)x + 0.5f) / (float)D - 0.5f;
    const float fy = ((float)y + 0.5f) / (float)D - 0.5f;
    const float flx = floorf(fx), fly = floorf(fy);
    const float tx = fx - flx, ty = fy - fly;
    const int i0 = min(max((int)flx, 0), Bx - 1), i1 = min(max((int)flx + 1, 0), Bx - 1);
    const int j0 = min(max((int)fly, 0), By - 1), j1 = min(max((int)fly + 1, 0), By - 1);
    const float* Mf = models + (size_t)f * By * Bx * mstride;
    const float* A00 = Mf + ((size_t)j0 * Bx + i0) * mstride;
    const float* A01 = Mf + ((size_t)j0 * Bx + i1) * mstride;
    const float* A10 = Mf + ((size_t)j1 * Bx + i0) * mstride;
    const float* A11 = Mf + ((size_t)j1 * Bx + i1) * mstride;
    const size_t plane = (size_t)W * H;
    const size_t p = (size_t)y * W + x;
    float xt[P];
    xt[0] = 1.f;
#pragma unroll
    for (int q = 0; q < Q; ++q) xt[1 + q] = __ldg(guides + ((size_t)f * Q + q) * plane + p);
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        float a0 = 0.f, a1 = 0.f;  // x~.A_y0, x~.A_y1 (y-blended models at i0 and i1)
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const int k = i * 3 + cc;
            const float m0 = fmaf(ty, __ldg(A10 + k) - __ldg(A00 + k), __ldg(A00 + k));
            const float m1 = fmaf(ty, __ldg(A11 + k) - __ldg(A01 + k), __ldg(A01 + k));
            a0 = fmaf(xt[i], m0, a0);
            a1 = fmaf(xt[i], m1, a1);
        }
        out[((size_t)f * 3 + cc) * plane + p] = fmaf(tx, a1 - a0, a0);
    }
}

// K4 for Tikhonov models stored centred ([b0 | slopes | mu] per block, mstride floats,
// solve_block_tikhonov): the four bracketing blocks' predictions b0 + A . (x - mu) are
// evaluated separately and blended bilinearly -- equal to blending the raw models in exact
// arithmetic (R6), but without the fp32 cancellation of large slopes against the bias.
template <int Q>
__global__ void __launch_bounds__(256) k_apply_centered(int W, int H, int D, int Bx, int By,
                                                        const float* __restrict__ models, int mstride,
                                                        const float* __restrict__ guides, float* __restrict__ out)
{
    constexpr int P = Q + 1;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int f = blockIdx.z;
    if (x >= W) return;
    const float fx = ((float)x + 0.5f) / (float)D - 0.5f;
    const float fy = ((float)y + 0.5f) / (float)D - 0.5f;
    const float flx = floorf(fx), fly = floorf(fy);
    const float tx = fx - flx, ty = fy - fly;
    const int i0 = min(max((int)flx, 0), Bx - 1), i1 = min(max((int)flx + 1, 0), Bx - 1);
    const int j0 = min(max((int)fly, 0), By - 1), j1 = min(max((int)fly + 1, 0), By - 1);
    const float* Mf = models + (size_t)f * By * Bx * mstride;
    const float* A[4] = {Mf + ((size_t)j0 * Bx + i0) * mstride, Mf + ((size_t)j0 * Bx + i1) * mstride,
                         Mf + ((size_t)j1 * Bx + i0) * mstride, Mf + ((size_t)j1 * Bx + i1) * mstride};
    const float wgt[4] = {(1.f - tx) * (1.f - ty), tx * (1.f - ty), (1.f - tx) * ty, tx * ty};
    const size_t plane = (size_t)W * H;
    const size_t p = (size_t)y * W + x;
    float xg[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) xg[q] = __ldg(guides + ((size_t)f * Q + q) * plane + p);
    float o[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        float d[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) d[q] = xg[q] - __ldg(A[b] + 3 * P + q);
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            float v = __ldg(A[b] + cc);
#pragma unroll
            for (int q = 0; q < Q; ++q) v = fmaf(d[q], __ldg(A[b] + (1 + q) * 3 + cc), v);
            o[cc] = fmaf(wgt[b], v, o[cc]);
        }
    }
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) out[((size_t)f * 3 + cc) * plane + p] = o[cc];
}

}  // namespace flr
