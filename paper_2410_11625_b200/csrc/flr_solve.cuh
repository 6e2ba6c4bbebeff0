// flr_solve.cuh -- the appendix's normalised, regularised per-block solve
// as one fp64 in-register device function, shared by every kernel schedule.
//
//   n = M_00, mu_X = u_X / n, mu_Y = N_0 / n
//   W^ = S/n + eps_mul diag(mu^2) + eps_add I - (1 - eps_mul) mu mu^T (R7, R8)
//   sigma^ = sqrt(max(diag W^, 1e-300))                            (R11)
//   (only 1/sigma^ and 1/R_kk are needed: one rsqrt each, <= 1 ulp from sqrt-then-divide)
//   C^_ij = W^_ij / (sigma^_i sigma^_j)
//   B^_ic = (XY_ic / n - mu_i mu_Y,c) / sigma^_i                   (R9)
//   A^ = (C^ + eps_add I)^-1 B^
//   raw model (R6): A[1+j][c] = A^[j][c] / sigma^_j,  A[0][c] = mu_Y,c - sum_j mu_j A[1+j][c]
//
// (C^ + eps_add I) is symmetric positive definite for eps_add > 0 (R13), so the
// solve is a Cholesky factorisation + two triangular solves instead of the
// paper's recursive block inverse: the solution is unique, so any
// exact solver returns it up to rounding.
#pragma once
#include <type_traits>
#include "flr_common.cuh"

namespace flr {

// storage of the normalised right-hand sides B^[i][c] (registers or shared memory)
template <int Q>
struct RegB {
    double b[Q][3];
    __device__ __forceinline__ double& operator()(int i, int c) { return b[i][c]; }
};
struct SmemB {
    double* p;   // element (i, c) at p[(3 i + c) * stride]
    int stride;
    __device__ __forceinline__ double& operator()(int i, int c) { return p[(3 * i + c) * stride]; }
};

template <int Q, class MomentFn, class OutT>
__device__ __forceinline__ void solve_block_tikhonov(MomentFn&& m, double eps, OutT&& out, bool centered = false);

// eps_mul sentinels selecting the Tikhonov solve inside the library (users cannot pass a
// negative eps_mul, flr_api.cu): raw-basis models, or models centred at the window mean
constexpr double kTikhonovRaw = -1.0, kTikhonovCentered = -2.0;
__host__ __device__ inline bool tikhonov_centered(double eps_mul) { return eps_mul < -1.5; }

// `m(k)` returns the blurred fp64 moment component k (layout of flr_common.cuh).
// Writes 3(Q+1) floats to `out` (row 0 = bias).  The 3 right-hand sides are solved one
// channel at a time so the live set stays small (B may live in shared memory).
// `out[i]` is any float lvalue accessor (a pointer, or a shared-memory staging view).
template <int Q, class MomentFn, class BStore, class OutT>
__device__ __forceinline__ void solve_block_b(MomentFn&& m, double eps_add, double eps_mul, OutT&& out, BStore& B)
{
    if (eps_mul < 0.0) {  // Tikhonov mode sentinel (see solve_block_tikhonov)
        solve_block_tikhonov<Q>(m, eps_add, out, tikhonov_centered(eps_mul));
        return;
    }
    using Dm = Dims<Q>;
    const double n = m(Dm::C_N);
    const double inv_n = 1.0 / n;
    double mu[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) mu[j] = m(Dm::C_U + j) * inv_n;
    double Wh[Dm::NS];
    const double om = 1.0 - eps_mul;
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = i; j < Q; ++j) {
            double w = fma(m(Dm::s_idx(i, j)), inv_n, -om * mu[i] * mu[j]);
            if (i == j) w += fma(eps_mul * mu[i], mu[i], eps_add);
            Wh[Dm::s_idx(i, j) - Dm::C_S] = w;
        }
    double isig[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) isig[i] = rsqrt(fmax(Wh[Dm::s_idx(i, i) - Dm::C_S], 1e-300));
    double muY[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) muY[c] = m(Dm::C_Y + c) * inv_n;
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) B(i, c) = fma(m(Dm::C_XY + i * 3 + c), inv_n, -mu[i] * muY[c]) * isig[i];
    // C^ + eps I in place (upper triangle)
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
        for (int j = i; j < Q; ++j) {
            const int k = Dm::s_idx(i, j) - Dm::C_S;
            Wh[k] = Wh[k] * isig[i] * isig[j] + (i == j ? eps_add : 0.0);
        }
    // Cholesky C = R^T R (R upper, in place)
    double rinv[Q];
    static_for<Q>([&](auto K) {
        constexpr int k = decltype(K)::value;
        double dkk = Wh[Dm::s_idx(k, k) - Dm::C_S];
        static_for<k>([&](auto PP) {
            constexpr int p = decltype(PP)::value;
            const double r = Wh[Dm::s_idx(p, k) - Dm::C_S];
            dkk = fma(-r, r, dkk);
        });
        rinv[k] = rsqrt(dkk);
        static_for<Q - k - 1>([&](auto JJ) {
            constexpr int j = k + 1 + decltype(JJ)::value;
            double v = Wh[Dm::s_idx(k, j) - Dm::C_S];
            static_for<k>([&](auto PP) {
                constexpr int p = decltype(PP)::value;
                v = fma(-Wh[Dm::s_idx(p, k) - Dm::C_S], Wh[Dm::s_idx(p, j) - Dm::C_S], v);
            });
            Wh[Dm::s_idx(k, j) - Dm::C_S] = v * rinv[k];
        });
    });
    // per channel: R^T z = B, R A^ = z, raw model column (channels interleaved when B is
    // in registers; one at a time when it lives in shared memory to save registers)
    constexpr int UC = std::is_same<BStore, RegB<Q>>::value ? 3 : 1;
#pragma unroll UC
    for (int c = 0; c < 3; ++c) {
        double z[Q] = {};
        static_for<Q>([&](auto K) {
            constexpr int k = decltype(K)::value;
            double v = B(k, c);
            static_for<k>([&](auto PP) {
                constexpr int p = decltype(PP)::value;
                v = fma(-Wh[Dm::s_idx(p, k) - Dm::C_S], z[p], v);
            });
            z[k] = v * rinv[k];
        });
        static_for<Q>([&](auto KK) {
            constexpr int k = Q - 1 - decltype(KK)::value;
            double v = z[k];
            static_for<Q - 1 - k>([&](auto PP) {
                constexpr int p = k + 1 + decltype(PP)::value;
                v = fma(-Wh[Dm::s_idx(k, p) - Dm::C_S], z[p], v);
            });
            z[k] = v * rinv[k];
        });
        double bias = muY[c];
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            const double a = z[j] * isig[j];
            out[(1 + j) * 3 + c] = (float)a;
            bias = fma(-mu[j], a, bias);
        }
        out[c] = (float)bias;
    }
}

// Tikhonov solve (Eq. tikhonov, Fig. 3; R18, R22): the blurred
// moments as weighted means, A = (Mbar / n + eps I)^-1 (Nbar / n) on the full (Q+1) x (Q+1)
// system (the ones channel included, so eps also shrinks the bias), by Cholesky.
// Selected inside the library by eps_mul < 0 (flr_params.solver = FLR_SOLVER_TIKHONOV;
// a negative eps_mul is rejected at the ABI, so the sentinel never collides).
// `centered`: write [b0 (3) | slopes (3Q) | mu (Q)] with mu = the window mean of the guides
// and b0 = A0 + mu . A[1:] (in fp64), so the apply evaluates b0 + A[1:] . (x - mu): at
// eps ~1e-6 a nearly flat guide gets slopes ~cov/eps whose raw-basis evaluation
// A0 + A[1:] . x cancels catastrophically in fp32 (k_apply_centered).
// Two phases, so a caller that receives the blurred components in order (n, u, S, Y, then
// XY: flr_common.cuh) can factor the system before the cross moments arrive (flr_k2.cuh):
// factor() reads components [0, C_XY), finish() the rest.
template <int Q>
struct TikhonovSolve {
    static constexpr int P = Q + 1, PS = P * (P + 1) / 2;
    __device__ static constexpr int at(int i, int j) { return i * P - (i * (i - 1)) / 2 + (j - i); }  // i <= j
    double inv_n, T[PS], rinv[P], mu[Q];
    template <class MomentFn>
    __device__ __forceinline__ void factor(MomentFn&& m, double eps)
    {
        using Dm = Dims<Q>;
        inv_n = 1.0 / m(Dm::C_N);
        T[at(0, 0)] = 1.0 + eps;
#pragma unroll
        for (int j = 0; j < Q; ++j) mu[j] = m(Dm::C_U + j) * inv_n;
#pragma unroll
        for (int j = 0; j < Q; ++j) T[at(0, 1 + j)] = mu[j];
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
            for (int j = i; j < Q; ++j) T[at(1 + i, 1 + j)] = fma(m(Dm::s_idx(i, j)), inv_n, i == j ? eps : 0.0);
        static_for<P>([&](auto K) {
            constexpr int k = decltype(K)::value;
            double dkk = T[at(k, k)];
            static_for<k>([&](auto PP) {
                constexpr int p = decltype(PP)::value;
                dkk = fma(-T[at(p, k)], T[at(p, k)], dkk);
            });
            rinv[k] = rsqrt(dkk);
            static_for<P - k - 1>([&](auto JJ) {
                constexpr int j = k + 1 + decltype(JJ)::value;
                double v = T[at(k, j)];
                static_for<k>([&](auto PP) {
                    constexpr int p = decltype(PP)::value;
                    v = fma(-T[at(p, k)], T[at(p, j)], v);
                });
                T[at(k, j)] = v * rinv[k];
            });
        });
    }
    template <class MomentFn, class OutT>
    __device__ __forceinline__ void finish(MomentFn&& m, OutT&& out, bool centered)
    {
        using Dm = Dims<Q>;
        double c[P][3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) c[0][cc] = m(Dm::C_Y + cc) * inv_n;
#pragma unroll
        for (int i = 0; i < Q; ++i)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) c[1 + i][cc] = m(Dm::C_XY + i * 3 + cc) * inv_n;
        static_for<P>([&](auto K) {
            constexpr int k = decltype(K)::value;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                double v = c[k][cc];
                static_for<k>([&](auto PP) {
                    constexpr int p = decltype(PP)::value;
                    v = fma(-T[at(p, k)], c[p][cc], v);
                });
                c[k][cc] = v * rinv[k];
            }
        });
        static_for<P>([&](auto KK) {
            constexpr int k = P - 1 - decltype(KK)::value;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                double v = c[k][cc];
                static_for<P - 1 - k>([&](auto PP) {
                    constexpr int p = k + 1 + decltype(PP)::value;
                    v = fma(-T[at(k, p)], c[p][cc], v);
                });
                c[k][cc] = v * rinv[k];
            }
        });
        if (centered) {
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                double b0 = c[0][cc];
#pragma unroll
                for (int j = 0; j < Q; ++j) b0 = fma(c[1 + j][cc], mu[j], b0);
                out[cc] = (float)b0;
            }
#pragma unroll
            for (int i = 1; i < P; ++i)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) out[i * 3 + cc] = (float)c[i][cc];
#pragma unroll
            for (int j = 0; j < Q; ++j) out[3 * P + j] = (float)mu[j];
            return;
        }
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) out[i * 3 + cc] = (float)c[i][cc];
    }
};

template <int Q, class MomentFn, class OutT>
__device__ __forceinline__ void solve_block_tikhonov(MomentFn&& m, double eps, OutT&& out, bool centered)
{
    TikhonovSolve<Q> t;
    t.factor(m, eps);
    t.finish(m, out, centered);
}

// In two phases like TikhonovSolve: factor() reads n, u and S, finish() Y and the cross moments.
template <int Q>
struct DirectSolve {
    using Dm = Dims<Q>;
    double inv_n, mu[Q], M[Dm::NS], rinv[Q];
    // begin() reads n and u; row<K>() then assembles row K of M (S row K) and computes row K
    // of its Cholesky factor M = R^T R (R upper, in place), so a caller receiving S row by
    // row (flr_k2.cuh) factors as it goes; factor() = begin + every row.
    template <class MomentFn>
    __device__ __forceinline__ void begin(MomentFn&& m)
    {
        inv_n = 1.0 / m(Dm::C_N);
#pragma unroll
        for (int j = 0; j < Q; ++j) mu[j] = m(Dm::C_U + j) * inv_n;
    }
    template <int K, class MomentFn>
    __device__ __forceinline__ void row(MomentFn&& m, double eps_add, double eps_mul)
    {
        const double om = 1.0 - eps_mul;
#pragma unroll
        for (int j = K; j < Q; ++j) {
            double w = fma(m(Dm::s_idx(K, j)), inv_n, -om * mu[K] * mu[j]);
            if (j == K) {
                w += fma(eps_mul * mu[K], mu[K], eps_add);          // W^_ii
                w = fma(eps_add, fmax(w, 1e-300), w);                // + eps sigma^_i^2
            }
            M[Dm::s_idx(K, j) - Dm::C_S] = w;
        }
        double dkk = M[Dm::s_idx(K, K) - Dm::C_S];
        static_for<K>([&](auto PP) {
            constexpr int p = decltype(PP)::value;
            const double r = M[Dm::s_idx(p, K) - Dm::C_S];
            dkk = fma(-r, r, dkk);
        });
        rinv[K] = rsqrt(dkk);
        static_for<Q - K - 1>([&](auto JJ) {
            constexpr int j = K + 1 + decltype(JJ)::value;
            double v = M[Dm::s_idx(K, j) - Dm::C_S];
            static_for<K>([&](auto PP) {
                constexpr int p = decltype(PP)::value;
                v = fma(-M[Dm::s_idx(p, K) - Dm::C_S], M[Dm::s_idx(p, j) - Dm::C_S], v);
            });
            M[Dm::s_idx(K, j) - Dm::C_S] = v * rinv[K];
        });
    }
    template <class MomentFn>
    __device__ __forceinline__ void factor(MomentFn&& m, double eps_add, double eps_mul)
    {
        begin(m);
        static_for<Q>([&](auto K) { row<decltype(K)::value>(m, eps_add, eps_mul); });
    }
    // The right-hand sides, also incrementally: rhs_begin() reads Y; fwd<I>() forms the
    // cross covariances of guide I and runs row I of the forward substitution R^T z = c
    // (needs Cholesky rows 0..I); back_out() the back substitution R a = z and the raw model.
    double muY[3], c[Q][3];
    template <class MomentFn>
    __device__ __forceinline__ void rhs_begin(MomentFn&& m)
    {
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) muY[cc] = m(Dm::C_Y + cc) * inv_n;
    }
    template <int I, class MomentFn>
    __device__ __forceinline__ void fwd(MomentFn&& m)
    {
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            double v = fma(m(Dm::C_XY + I * 3 + cc), inv_n, -mu[I] * muY[cc]);
            static_for<I>([&](auto PP) {
                constexpr int p = decltype(PP)::value;
                v = fma(-M[Dm::s_idx(p, I) - Dm::C_S], c[p][cc], v);
            });
            c[I][cc] = v * rinv[I];
        }
    }
    template <class OutT>
    __device__ __forceinline__ void back_out(OutT&& out)
    {
        static_for<Q>([&](auto KK) {
            constexpr int k = Q - 1 - decltype(KK)::value;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                double v = c[k][cc];
                static_for<Q - 1 - k>([&](auto PP) {
                    constexpr int p = k + 1 + decltype(PP)::value;
                    v = fma(-M[Dm::s_idx(k, p) - Dm::C_S], c[p][cc], v);
                });
                c[k][cc] = v * rinv[k];
            }
        });
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            double bias = muY[cc];
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                out[(1 + j) * 3 + cc] = (float)c[j][cc];
                bias = fma(-mu[j], c[j][cc], bias);
            }
            out[cc] = (float)bias;
        }
    }
    template <class MomentFn, class OutT>
    __device__ __forceinline__ void finish(MomentFn&& m, OutT&& out)
    {
        rhs_begin(m);
        static_for<Q>([&](auto I) { fwd<decltype(I)::value>(m); });
        back_out(out);
    }
};

// The same solution without forming C^ (R13: any exact solve of the same system).  With
// D = diag(sigma^) (sigma^_i^2 = max(W^_ii, 1e-300)), C^ + eps I = D^-1 (W^ + eps D^2) D^-1
// and B^ = D^-1 cov_xy, so the raw slopes are A[1:] = D^-1 A^ = (W^ + eps D^2)^-1 cov_xy:
// one Cholesky of M = W^ + eps diag(max(W^_ii, 1e-300)) and 3 right-hand sides, no
// normalising rsqrt, no scaling of C^, B^ or A^ (about 25 % fewer fp64 operations).
template <int Q, class MomentFn, class OutT>
__device__ __forceinline__ void solve_block_direct(MomentFn&& m, double eps_add, double eps_mul, OutT&& out)
{
    DirectSolve<Q> d;
    d.factor(m, eps_add, eps_mul);
    d.finish(m, out);
}

template <int Q, class MomentFn>
__device__ __forceinline__ void solve_block(MomentFn&& m, double eps_add, double eps_mul, float* out)
{
    if (eps_mul < 0.0) {  // Tikhonov mode sentinel (see solve_block_tikhonov)
        solve_block_tikhonov<Q>(m, eps_add, out, tikhonov_centered(eps_mul));
        return;
    }
#ifdef FLR_SOLVE_NORMALISED
    RegB<Q> B;
    solve_block_b<Q>(m, eps_add, eps_mul, out, B);
#else
    solve_block_direct<Q>(m, eps_add, eps_mul, out);
#endif
}

}  // namespace flr
