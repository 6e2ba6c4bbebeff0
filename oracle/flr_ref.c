/*
 * flr_ref.c -- plain, slow, obviously-correct float64 CPU ORACLE for FLR.
 *
 * TEST INFRASTRUCTURE ONLY (see flr_ref.h).  No blocking, fusion or reordering
 * beyond what the paper states: every function below is the paper's definition
 * written out as loops, in the paper's order and notation.  Float32 inputs are
 * promoted to double on load; everything after that is double.  OpenMP only
 * distributes independent blocks / pixel rows over threads; each result is
 * computed by one thread in a fixed order, so the output does not depend on
 * the thread count.
 *
 * Citations: P:<line> = line of /root/reference/PAPER.md (arXiv 2410.11625);
 * R<k> = reading k of an ambiguous passage, listed in DESIGN.md section 3.
 *
 * Parity pins (tests/test_oracle_pins.py): brute-force per-block weighted least
 * squares (np.linalg.lstsq on raw pixels), the Q=1 closed form, the D=1 dense
 * windowed regression, affine exactness, constant images, the eps -> inf blur
 * limit, invariances and the bilinear-weight pattern.  No function here is
 * "parity unpinned".
 */
#include "flr_ref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXP 16 /* P = Q + 1 <= 16 */

static int ceil_div(int a, int b) { return (a + b - 1) / b; }

int flr_ref_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * Step 1-2. Outer products and strided box downsample:
 *   M_b = sum_{p in b} x~_p x~_p^T,   N_b = sum_{p in b} x~_p y_p^T,
 *   x~_p = [1, X_p,1 .. X_p,Q] (the first guide column is all ones).
 * The box filter is a SUM (R12); edge blocks are truncated (R5).
 * ------------------------------------------------------------------------- */
/* block sums; the radiance is given either as float (radiance) or as double (radiance_d) */
static int moments_impl(int n, int Q, int W, int H, int D, const float* guides,
                        const float* radiance, const double* radiance_d, double* M, double* N)
{
    if (n < 1 || Q < 1 || Q > MAXP - 1 || W < 1 || H < 1 || D < 1 || !guides ||
        !(radiance || radiance_d) || !M || !N)
        return 1;
    const int P = Q + 1;
    const int Bx = ceil_div(W, D), By = ceil_div(H, D);
    const long plane = (long)W * H;
    const long nblk = (long)n * By * Bx;

#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < nblk; ++idx) {
        const int f = (int)(idx / ((long)By * Bx));
        const int by = (int)((idx / Bx) % By);
        const int bx = (int)(idx % Bx);
        double* Mb = M + idx * P * P;
        double* Nb = N + idx * P * 3;
        for (int i = 0; i < P * P; ++i) Mb[i] = 0.0;
        for (int i = 0; i < P * 3; ++i) Nb[i] = 0.0;
        const float* G = guides + (long)f * Q * plane;
        const long yoff = (long)f * 3 * plane;
        const int y1 = (by + 1) * D < H ? (by + 1) * D : H;
        const int x1 = (bx + 1) * D < W ? (bx + 1) * D : W;
        for (int y = by * D; y < y1; ++y)
            for (int x = bx * D; x < x1; ++x) {
                const long p = (long)y * W + x;
                double xt[MAXP];
                double yv[3];
                xt[0] = 1.0;
                for (int q = 0; q < Q; ++q) xt[1 + q] = (double)G[q * plane + p];
                for (int c = 0; c < 3; ++c)
                    yv[c] = radiance ? (double)radiance[yoff + c * plane + p] : radiance_d[yoff + c * plane + p];
                for (int i = 0; i < P; ++i)
                    for (int j = 0; j < P; ++j) Mb[i * P + j] += xt[i] * xt[j];
                for (int i = 0; i < P; ++i)
                    for (int c = 0; c < 3; ++c) Nb[i * 3 + c] += xt[i] * yv[c];
            }
    }
    return 0;
}

int flr_ref_moments(int n, int Q, int W, int H, int D,
                    const float* guides, const float* radiance,
                    double* M, double* N)
{
    return radiance ? moments_impl(n, Q, W, H, D, guides, radiance, NULL, M, N) : 1;
}

/* Gaussian window taps: unnormalised, peak 1 (R2). */
int flr_ref_gauss_taps(double s, int R, double* g)
{
    if (!(s > 0.0) || R < 0 || !g) return 1;
    for (int i = -R; i <= R; ++i) g[R + i] = exp(-(double)(i * i) / (2.0 * s * s));
    return 0;
}

/* ---------------------------------------------------------------------------
 * Step 3. Gaussian blur of the moment field at block resolution (P:315-316,
 * P:334), written as the 2-D windowed sum it defines (the separable x/y split
 * of the GPU path is a reordering the oracle does not make):
 *   Mbar_b = sum_{dy=-R..R} sum_{dx=-R..R} g_dy g_dx M_{b+d},  b+d in grid (R3).
 * ------------------------------------------------------------------------- */
int flr_ref_blur(int n, int P, int Bx, int By, double s, int R,
                 const double* M, const double* N, double* Mbar, double* Nbar)
{
    if (n < 1 || P < 2 || P > MAXP || Bx < 1 || By < 1 || R < 0 || !(s > 0.0) || !M ||
        !N || !Mbar || !Nbar)
        return 1;
    double* g = (double*)malloc(sizeof(double) * (2 * R + 1));
    if (!g) return 1;
    flr_ref_gauss_taps(s, R, g);
    const long nblk = (long)n * By * Bx;

#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < nblk; ++idx) {
        const long f = idx / ((long)By * Bx);
        const int by = (int)((idx / Bx) % By);
        const int bx = (int)(idx % Bx);
        double* Mo = Mbar + idx * P * P;
        double* No = Nbar + idx * P * 3;
        for (int i = 0; i < P * P; ++i) Mo[i] = 0.0;
        for (int i = 0; i < P * 3; ++i) No[i] = 0.0;
        for (int dy = -R; dy <= R; ++dy) {
            const int yy = by + dy;
            if (yy < 0 || yy >= By) continue;
            for (int dx = -R; dx <= R; ++dx) {
                const int xx = bx + dx;
                if (xx < 0 || xx >= Bx) continue;
                const double w = g[R + dy] * g[R + dx];
                const long src = (f * By + yy) * Bx + xx;
                const double* Mi = M + src * P * P;
                const double* Ni = N + src * P * 3;
                for (int i = 0; i < P * P; ++i) Mo[i] += w * Mi[i];
                for (int i = 0; i < P * 3; ++i) No[i] += w * Ni[i];
            }
        }
    }
    free(g);
    return 0;
}

/* Solve Cm X = B for X (Q x 3) by Gaussian elimination with partial pivoting.
 * Cm is Q x Q (destroyed), B is Q x 3 (overwritten with X).  Returns 2 on an
 * exactly zero pivot. */
static int gauss_solve(int Q, double* Cm, double* B)
{
    for (int k = 0; k < Q; ++k) {
        int piv = k;
        double best = fabs(Cm[k * Q + k]);
        for (int r = k + 1; r < Q; ++r)
            if (fabs(Cm[r * Q + k]) > best) {
                best = fabs(Cm[r * Q + k]);
                piv = r;
            }
        if (best == 0.0) return 2;
        if (piv != k) {
            for (int j = 0; j < Q; ++j) {
                double t = Cm[k * Q + j];
                Cm[k * Q + j] = Cm[piv * Q + j];
                Cm[piv * Q + j] = t;
            }
            for (int c = 0; c < 3; ++c) {
                double t = B[k * 3 + c];
                B[k * 3 + c] = B[piv * 3 + c];
                B[piv * 3 + c] = t;
            }
        }
        for (int r = k + 1; r < Q; ++r) {
            const double m = Cm[r * Q + k] / Cm[k * Q + k];
            for (int j = k; j < Q; ++j) Cm[r * Q + j] -= m * Cm[k * Q + j];
            for (int c = 0; c < 3; ++c) B[r * 3 + c] -= m * B[k * 3 + c];
        }
    }
    for (int k = Q - 1; k >= 0; --k)
        for (int c = 0; c < 3; ++c) {
            double acc = B[k * 3 + c];
            for (int j = k + 1; j < Q; ++j) acc -= Cm[k * Q + j] * B[j * 3 + c];
            B[k * 3 + c] = acc / Cm[k * Q + k];
        }
    return 0;
}

/* ---------------------------------------------------------------------------
 * Steps 4-5. The appendix's normalised, regularised solve:
 *   n = M_00
 *   mu_X = u_X / n,  u_X = M_0,1:
 *   S = M_1:,1:
 *   W^ = S/n + eps_mul diag(mu_X^T mu_X) + eps_add I
 *        - (1 - eps_mul) mu_X^T mu_X                     (R7, R8)
 *   sigma^ = sqrt(diag W^)   (floored at 1e-300, R11)
 *   C^_ij = W^_ij / (sigma^_i sigma^_j)
 *   mu_Y = N_0,: / n
 *   B^_ij = (N_1+i,j / n - mu_X,i mu_Y,j) / sigma^_i      (R9)
 *   A^ = (C^ + eps_add I)^-1 B^                          (R13)
 *   y = ((x - mu_X) / sigma^) A^ + mu_Y
 * and the last line written as one raw-basis affine model (R6):
 *   A[1+j][c] = A^[j][c] / sigma^_j,  A[0][c] = mu_Y,c - sum_j mu_X,j A[1+j][c].
 * ------------------------------------------------------------------------- */
int flr_ref_solve_block(int P, const double* M, const double* N,
                        double eps_add, double eps_mul, double* A)
{
    if (P < 2 || P > MAXP || !M || !N || !A) return 1;
    const int Q = P - 1;
    double muX[MAXP], muY[3], sig[MAXP];
    double What[MAXP * MAXP], Chat[MAXP * MAXP], Bhat[MAXP * 3];

    const double n = M[0];
    for (int j = 0; j < Q; ++j) muX[j] = M[0 * P + (1 + j)] / n;
    for (int c = 0; c < 3; ++c) muY[c] = N[0 * 3 + c] / n;

    for (int i = 0; i < Q; ++i)
        for (int j = 0; j < Q; ++j) {
            const double S_ij = M[(1 + i) * P + (1 + j)];
            double w = S_ij / n - (1.0 - eps_mul) * muX[i] * muX[j];
            if (i == j) w += eps_mul * muX[i] * muX[i] + eps_add;
            What[i * Q + j] = w;
        }
    for (int i = 0; i < Q; ++i) {
        double d = What[i * Q + i];
        if (d < 1e-300) d = 1e-300;
        sig[i] = sqrt(d);
    }
    for (int i = 0; i < Q; ++i)
        for (int j = 0; j < Q; ++j) Chat[i * Q + j] = What[i * Q + j] / (sig[i] * sig[j]);
    for (int i = 0; i < Q; ++i)
        for (int c = 0; c < 3; ++c)
            Bhat[i * 3 + c] = (N[(1 + i) * 3 + c] / n - muX[i] * muY[c]) / sig[i];

    for (int i = 0; i < Q; ++i) Chat[i * Q + i] += eps_add;
    if (gauss_solve(Q, Chat, Bhat)) return 2; /* Bhat now holds A^ */

    for (int c = 0; c < 3; ++c) {
        double bias = muY[c];
        for (int j = 0; j < Q; ++j) {
            const double a = Bhat[j * 3 + c] / sig[j];
            A[(1 + j) * 3 + c] = a;
            bias -= muX[j] * a;
        }
        A[0 * 3 + c] = bias;
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * Tikhonov solve (Eq. tikhonov; Fig. 3): the Gaussian-blurred
 * outer products of Fig. 3 are weighted MEANS (torchvision's kernel sums to one), so
 * with block moments the system is written on Mbar / n and Nbar / n, n = Mbar_00 the
 * blurred pixel count (R22):
 *   A = (Mbar / n + eps I)^-1 (Nbar / n)        over the full P x P system:
 * the ones channel is part of X, so eps also shrinks the bias (R18).
 * ------------------------------------------------------------------------- */
int flr_ref_solve_block_tikhonov(int P, const double* M, const double* N, double eps, double* A)
{
    if (P < 2 || P > MAXP || !M || !N || !A) return 1;
    double Cm[MAXP * MAXP], B[MAXP * 3];
    const double n = M[0];
    for (int i = 0; i < P; ++i)
        for (int j = 0; j < P; ++j) Cm[i * P + j] = M[i * P + j] / n + (i == j ? eps : 0.0);
    for (int i = 0; i < P; ++i)
        for (int c = 0; c < 3; ++c) B[i * 3 + c] = N[i * 3 + c] / n;
    if (gauss_solve(P, Cm, B)) return 2;
    for (int i = 0; i < P * 3; ++i) A[i] = B[i];
    return 0;
}

static int fit_impl_mode(int n, int Q, int W, int H, int D_fit, int U, double sigma, int R,
                         double eps_add, double eps_mul, int tikhonov, const float* guides,
                         const float* radiance, const double* radiance_d, double* A);

static int fit_impl(int n, int Q, int W, int H, int D_fit, int U, double sigma, int R,
                    double eps_add, double eps_mul, const float* guides, const float* radiance,
                    const double* radiance_d, double* A)
{
    return fit_impl_mode(n, Q, W, H, D_fit, U, sigma, R, eps_add, eps_mul, 0, guides, radiance,
                         radiance_d, A);
}

static int fit_impl_mode(int n, int Q, int W, int H, int D_fit, int U, double sigma, int R,
                         double eps_add, double eps_mul, int tikhonov, const float* guides,
                         const float* radiance, const double* radiance_d, double* A)
{
    if (n < 1 || Q < 1 || Q > MAXP - 1 || W < 1 || H < 1 || D_fit < 1 || U < 1 ||
        !(sigma > 0.0) || R < 0 || !(eps_add >= 0.0) || !(eps_mul >= 0.0) ||
        !(eps_mul < 1.0) || !guides || !(radiance || radiance_d) || !A)
        return 1;
    const int P = Q + 1;
    const int Bx = ceil_div(W, D_fit), By = ceil_div(H, D_fit);
    const long nblk = (long)n * By * Bx;
    double* M = (double*)malloc(sizeof(double) * nblk * P * P);
    double* N = (double*)malloc(sizeof(double) * nblk * P * 3);
    double* Mb = (double*)malloc(sizeof(double) * nblk * P * P);
    double* Nb = (double*)malloc(sizeof(double) * nblk * P * 3);
    int rc = 1;
    if (!M || !N || !Mb || !Nb) goto done;
    if ((rc = moments_impl(n, Q, W, H, D_fit, guides, radiance, radiance_d, M, N))) goto done;
    /* blur std in blocks: sigma (output pixels) / block size in output pixels */
    if ((rc = flr_ref_blur(n, P, Bx, By, sigma / ((double)D_fit * U), R, M, N, Mb, Nb)))
        goto done;
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (long idx = 0; idx < nblk; ++idx)
        bad |= tikhonov ? flr_ref_solve_block_tikhonov(P, Mb + idx * P * P, Nb + idx * P * 3, eps_add,
                                                       A + idx * P * 3)
                        : flr_ref_solve_block(P, Mb + idx * P * P, Nb + idx * P * 3, eps_add, eps_mul,
                                              A + idx * P * 3);
    rc = bad ? 2 : 0;
done:
    free(M);
    free(N);
    free(Mb);
    free(Nb);
    return rc;
}

int flr_ref_fit(int n, int Q, int W, int H, int D_fit, int U,
                double sigma, int R, double eps_add, double eps_mul,
                const float* guides, const float* radiance, double* A)
{
    if (!radiance) return 1;
    return fit_impl(n, Q, W, H, D_fit, U, sigma, R, eps_add, eps_mul, guides, radiance, NULL, A);
}

int flr_ref_fit_tikhonov(int n, int Q, int W, int H, int D_fit, int U, double sigma, int R, double eps,
                         const float* guides, const float* radiance, double* A)
{
    if (!radiance) return 1;
    return fit_impl_mode(n, Q, W, H, D_fit, U, sigma, R, eps, 0.0, 1, guides, radiance, NULL, A);
}

/* ---------------------------------------------------------------------------
 * Step 6. Upsample and model application.
 * Block centres sit at (b + 1/2) D_out - 1/2 (R4); beyond the outermost
 * centres the edge model is used.  The model PARAMETERS are interpolated (P:318,
 * R6) and the blended model is applied: I = x~ A.
 * ------------------------------------------------------------------------- */
int flr_ref_apply(int n, int Q, int W, int H, int D_out, int Bx, int By,
                  const double* A, const float* guides, double* out)
{
    if (n < 1 || Q < 1 || Q > MAXP - 1 || W < 1 || H < 1 || D_out < 1 || Bx < 1 ||
        By < 1 || !A || !guides || !out)
        return 1;
    const int P = Q + 1;
    const long plane = (long)W * H;
    const long nrows = (long)n * H;

#pragma omp parallel for schedule(static)
    for (long ri = 0; ri < nrows; ++ri) {
        const long f = ri / H;
        const int y = (int)(ri % H);
        const double fy = (y + 0.5) / D_out - 0.5;
        const double fly = floor(fy);
        const double ty = fy - fly;
        int j0 = (int)fly, j1 = j0 + 1;
        if (j0 < 0) j0 = 0;
        if (j0 > By - 1) j0 = By - 1;
        if (j1 < 0) j1 = 0;
        if (j1 > By - 1) j1 = By - 1;
        for (int x = 0; x < W; ++x) {
            const double fx = (x + 0.5) / D_out - 0.5;
            const double flx = floor(fx);
            const double tx = fx - flx;
            int i0 = (int)flx, i1 = i0 + 1;
            if (i0 < 0) i0 = 0;
            if (i0 > Bx - 1) i0 = Bx - 1;
            if (i1 < 0) i1 = 0;
            if (i1 > Bx - 1) i1 = Bx - 1;
            const double* A00 = A + ((f * By + j0) * Bx + i0) * P * 3;
            const double* A01 = A + ((f * By + j0) * Bx + i1) * P * 3;
            const double* A10 = A + ((f * By + j1) * Bx + i0) * P * 3;
            const double* A11 = A + ((f * By + j1) * Bx + i1) * P * 3;
            const double w00 = (1.0 - ty) * (1.0 - tx), w01 = (1.0 - ty) * tx;
            const double w10 = ty * (1.0 - tx), w11 = ty * tx;
            double Ab[MAXP * 3];
            for (int k = 0; k < P * 3; ++k)
                Ab[k] = w00 * A00[k] + w01 * A01[k] + w10 * A10[k] + w11 * A11[k];
            const long p = (long)y * W + x;
            double xt[MAXP];
            xt[0] = 1.0;
            for (int q = 0; q < Q; ++q) xt[1 + q] = (double)guides[(f * Q + q) * plane + p];
            for (int c = 0; c < 3; ++c) {
                double acc = 0.0;
                for (int i = 0; i < P; ++i) acc += xt[i] * Ab[i * 3 + c];
                out[(f * 3 + c) * plane + p] = acc;
            }
        }
    }
    return 0;
}

int flr_ref_denoise(int n, int Q, int W, int H, int D, double sigma, int R,
                    double eps_add, double eps_mul,
                    const float* guides, const float* radiance, double* out)
{
    return flr_ref_denoise_upsample(n, Q, W, H, D, 1, sigma, R, eps_add, eps_mul, guides,
                                    radiance, guides, out);
}

int flr_ref_denoise_upsample(int n, int Q, int W_lo, int H_lo, int D_fit, int U,
                             double sigma, int R, double eps_add, double eps_mul,
                             const float* guides_lo, const float* radiance_lo,
                             const float* guides_hi, double* out)
{
    if (n < 1 || Q < 1 || Q > MAXP - 1 || W_lo < 1 || H_lo < 1 || D_fit < 1 || U < 1 ||
        !guides_hi || !out)
        return 1;
    const int P = Q + 1;
    const int Bx = ceil_div(W_lo, D_fit), By = ceil_div(H_lo, D_fit);
    double* A = (double*)malloc(sizeof(double) * (long)n * By * Bx * P * 3);
    if (!A) return 1;
    int rc = flr_ref_fit(n, Q, W_lo, H_lo, D_fit, U, sigma, R, eps_add, eps_mul, guides_lo,
                         radiance_lo, A);
    if (!rc) rc = flr_ref_apply(n, Q, W_lo * U, H_lo * U, D_fit * U, Bx, By, A, guides_hi, out);
    free(A);
    return rc;
}

/* The paper's input/output protocol around FLR:
 *   y   = P / max(A, floor)          per pixel and channel (demodulate; floor: R20)
 *   I   = FLR(guides, y)             fit + apply in fp64 as above
 *   out = A * I (+ direct)           remodulate with the unfloored albedo, then add the
 *                                    noise-free direct radiance if given (R21)
 * The demodulated radiance is kept in double (never rounded to float). */
int flr_ref_denoise_modulated(int n, int Q, int W, int H, int D, double sigma, int R,
                              double eps_add, double eps_mul, double floor,
                              const float* guides, const float* radiance_mod, const float* albedo,
                              const float* direct, double* out)
{
    if (n < 1 || Q < 1 || Q > MAXP - 1 || W < 1 || H < 1 || D < 1 || !(floor > 0.0) ||
        !guides || !radiance_mod || !albedo || !out)
        return 1;
    const long total = (long)n * 3 * W * H;
    const int P = Q + 1;
    const int Bx = ceil_div(W, D), By = ceil_div(H, D);
    double* y = (double*)malloc(sizeof(double) * total);
    double* A = (double*)malloc(sizeof(double) * (long)n * By * Bx * P * 3);
    int rc = 1;
    if (!y || !A) goto done;
    for (long i = 0; i < total; ++i) {
        const double a = (double)albedo[i];
        y[i] = (double)radiance_mod[i] / (a > floor ? a : floor);
    }
    rc = fit_impl(n, Q, W, H, D, 1, sigma, R, eps_add, eps_mul, guides, NULL, y, A);
    if (!rc) rc = flr_ref_apply(n, Q, W, H, D, Bx, By, A, guides, out);
    if (!rc)
        for (long i = 0; i < total; ++i)
            out[i] = (double)albedo[i] * out[i] + (direct ? (double)direct[i] : 0.0);
done:
    free(y);
    free(A);
    return rc;
}
