/*
 * flr_ref.h -- float64 CPU ORACLE for Fast Local Regression (FLR).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2410_11625_b200/, libflr.so) never links, imports
 * or calls anything under oracle/, and this file shares no code, header,
 * helper or table with it.
 *
 * What it computes (arXiv 2410.11625, cited as P:<line of PAPER.md>):
 *   fit   = block moments
 *         -> Gaussian blur of the moment field
 *         -> appendix normalise + regularise + solve per block
 *   apply = bilinear blend of the per-block models, then I = x A
 *   joint denoise+upsample: fit at low resolution, apply with hi-res guides
 *   albedo protocol: demodulate, denoise, remodulate, add direct light
 * Readings of ambiguous passages (R1..R19) are listed in DESIGN.md section 3.
 *
 * Conventions (all arrays row-major, C order, host memory, caller-owned):
 *   Q guide planes, P = Q + 1 (the implicit ones channel is x~_0 = 1)
 *   guides   float  [n][Q][H][W]
 *   radiance float  [n][3][H][W]
 *   M        double [n][By][Bx][P][P]   block sums of x~ x~^T (full symmetric)
 *   N        double [n][By][Bx][P][3]   block sums of x~ y^T
 *   A        double [n][By][Bx][P][3]   raw-basis model, row 0 = bias
 *   out      double [n][3][H][W]
 * Return value: 0 on success, 1 on an invalid argument (nothing written).
 */
#ifndef FLR_REF_H
#define FLR_REF_H
#ifdef __cplusplus
extern "C" {
#endif

/* Step 1-2: per-block sums over block b's pixels [bx*D, min((bx+1)*D, W)) x
 * [by*D, min((by+1)*D, H)); edge blocks are truncated (R5). */
int flr_ref_moments(int n, int Q, int W, int H, int D,
                    const float* guides, const float* radiance,
                    double* M, double* N);

/* Gaussian taps g_i = exp(-i^2 / (2 s^2)), |i| <= R (R1, R2); g has 2R+1 entries,
 * g[R + i] = g_i. */
int flr_ref_gauss_taps(double s, int R, double* g);

/* Step 3: Mbar_b = sum_{dy,dx in [-R,R], b+d inside grid} g_dy g_dx M_{b+d}
 * (zero padding, R3); same for N.  s = sigma / D_out in block units. */
int flr_ref_blur(int n, int P, int Bx, int By, double s, int R,
                 const double* M, const double* N, double* Mbar, double* Nbar);

/* Step 4-5 for ONE block: appendix chain, Gaussian elimination with
 * partial pivoting for (C^ + eps I) A^ = B^, then the raw model (R6):
 *   A[1+j][c] = A^[j][c] / sigma^_j,   A[0][c] = mu_Y,c - sum_j mu_X,j A[1+j][c].
 * M is P x P, N is P x 3, A is P x 3.  Returns 2 if the system is singular. */
int flr_ref_solve_block(int P, const double* M, const double* N,
                        double eps_add, double eps_mul, double* A);

/* Steps 1-5 over every block of every frame.  D_fit = block size in fit pixels,
 * U = upsample factor (1 for plain denoise); the blur std in block units is
 * s = sigma / (D_fit * U) with sigma in OUTPUT pixels. */
int flr_ref_fit(int n, int Q, int W, int H, int D_fit, int U,
                double sigma, int R, double eps_add, double eps_mul,
                const float* guides, const float* radiance, double* A);

/* Step 6: for every output pixel, f = (x + 1/2)/D_out - 1/2, i0 = floor(f),
 * t = f - i0, i1 = i0 + 1, both clamped to [0, B-1] (R4); same for y.  The four
 * models are blended bilinearly and applied: I = x~ . A. */
int flr_ref_apply(int n, int Q, int W, int H, int D_out, int Bx, int By,
                  const double* A, const float* guides, double* out);

/* fit + apply with the same guides (D_out = D). */
int flr_ref_denoise(int n, int Q, int W, int H, int D, double sigma, int R,
                    double eps_add, double eps_mul,
                    const float* guides, const float* radiance, double* out);

/* fit on (guides_lo, radiance_lo) with D_fit, apply on guides_hi with
 * D_out = D_fit * U, W_hi = U W_lo, H_hi = U H_lo. */
int flr_ref_denoise_upsample(int n, int Q, int W_lo, int H_lo, int D_fit, int U,
                             double sigma, int R, double eps_add, double eps_mul,
                             const float* guides_lo, const float* radiance_lo,
                             const float* guides_hi, double* out);

/* The paper's protocol around FLR: radiance_mod = albedo-modulated
 * noisy indirect lighting, albedo [n][3][H][W]; y = radiance_mod / max(albedo, floor),
 * I = denoise(guides, y), out = albedo * I + direct (direct may be NULL = zero).
 * Readings R20 (floor) and R21 (direct composite) in DESIGN.md. */
int flr_ref_denoise_modulated(int n, int Q, int W, int H, int D, double sigma, int R,
                              double eps_add, double eps_mul, double floor,
                              const float* guides, const float* radiance_mod,
                              const float* albedo, const float* direct, double* out);

/* Tikhonov variant of steps 4-5 (Eq. tikhonov, Fig. 3; R18, R22):
 * A = (M / n + eps I)^-1 (N / n) on the full P x P system, n = M[0][0], by Gaussian
 * elimination with partial pivoting.  Returns 2 if singular. */
int flr_ref_solve_block_tikhonov(int P, const double* M, const double* N, double eps, double* A);

/* Steps 1-3 as flr_ref_fit, then the Tikhonov solve per block. */
int flr_ref_fit_tikhonov(int n, int Q, int W, int H, int D_fit, int U, double sigma, int R, double eps,
                         const float* guides, const float* radiance, double* A);

/* Number of OpenMP threads the oracle will use (1 when built without OpenMP). */
int flr_ref_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
