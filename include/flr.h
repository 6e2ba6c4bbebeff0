/*
 * flr.h -- C ABI of the B200 (sm_100a) Fast Local Regression library, libflr.so.
 *
 * Fast Local Regression (FLR) of Salmi, Csefalvay & Imber, "Fast Local Neural
 * Regression for Low-Cost, Path Traced Lambertian Global Illumination",
 * arXiv 2410.11625.  Citations P:<n> are lines of the paper's LaTeX source
 * (reference PAPER.md); R<k> are the readings of ambiguous passages listed in
 * DESIGN.md section 3.
 *
 * The operation (the paper's statement of the problem):
 *   given Q noise-free guide planes X (the ones channel x~_0 = 1 is implicit,
 *   P:224) and noisy RGB radiance Y, fit one affine model A_b in R^{(Q+1) x 3}
 *   per D x D pixel block from Gaussian-windowed block moments, with
 *   the appendix's normalised, regularised solve, then apply the
 *   bilinearly blended per-block models at every output pixel: I = x~ A (P:274-278,
 *   P:318).  The joint denoise + upsample variant fits at low resolution and
 *   applies with high-resolution guides.
 *
 * Data layout (every buffer planar float32, C-contiguous, row stride = width):
 *   guides    [n][Q][H][W]
 *   radiance  [n][3][H][W]
 *   models    [n][By][Bx][Q+1][3]  raw basis, row 0 = bias (the paper's A_k)
 *   out       [n][3][H][W]
 *   with Bx = ceil(W_fit / block), By = ceil(H_fit / block).
 *
 * Ownership and execution:
 *   * Every data pointer is a caller-owned CUDA DEVICE pointer on the current
 *     device.  The library allocates nothing; scratch memory is the caller's
 *     `workspace` (device memory, >= flr_workspace_size bytes, 256-byte aligned).
 *   * Inputs and outputs must not alias.  No hidden global state: calls are
 *     reentrant and may run concurrently on different streams with different
 *     workspaces.
 *   * Work is enqueued asynchronously on `stream` (NULL = legacy default
 *     stream); nothing synchronises the device or the host.  Results are
 *     visible after stream-ordered completion.  Results are deterministic
 *     (fixed reduction order, no floating-point atomics).
 *   * Numerics: block moments are accumulated in fp32 about a per-block shift
 *     (a pixel of the block) and un-shifted exactly in fp64; blur, normalise
 *     and solve run in fp64; models are stored in fp32 and applied in fp32.
 *     Parity bar against the fp64 oracle: |gpu - ref| <= 1e-5 + 1e-4 |ref|.
 *
 * Errors: arguments are validated before anything is launched; a failing
 * check returns a non-zero flr_status and enqueues nothing.  After launching,
 * cudaGetLastError() != cudaSuccess maps to FLR_ERR_CUDA.  Nothing is thrown
 * or aborted across the ABI.  Non-finite inputs are not sanitised; they
 * propagate to the outputs of the affected blocks.
 */
#ifndef FLR_H
#define FLR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* flr_stream_t; /* identical to cudaStream_t */

typedef enum {
    FLR_OK = 0,
    FLR_ERR_INVALID_VALUE = 1, /* null pointer, Q/block/sigma/eps out of range */
    FLR_ERR_SHAPE = 2,         /* sizes < 1, hi/lo size mismatch, model grid mismatch */
    FLR_ERR_ALIGNMENT = 3,     /* pointer not 4-byte aligned, workspace not 256-byte aligned */
    FLR_ERR_WORKSPACE = 4,     /* workspace_bytes smaller than flr_workspace_size */
    FLR_ERR_UNSUPPORTED = 5,   /* valid but not implemented (e.g. an unknown variant) */
    FLR_ERR_CUDA = 6           /* a CUDA launch failed; see cudaGetLastError */
} flr_status;

/* Kernel schedule.  All variants compute the same result within the parity
 * bar; AUTO picks the fastest one for the shape. */
typedef enum {
    FLR_VARIANT_AUTO = 0,   /* the fastest schedule for the shape (currently STAGED) */
    FLR_VARIANT_STAGED = 1, /* moments -> blur+solve -> apply, one launch each */
    FLR_VARIANT_FUSED = 2   /* one persistent kernel per call: every CTA claims FIT chunks,
                               blur+solve tiles and APPLY chunks from workspace queues as
                               their inputs complete (row wavefront; bitwise equal to STAGED).
                               Compiled for Q in {4, 8}, block in {4, 8}, radius in {3, 5},
                               output block a multiple of 8, 16-byte aligned planes with
                               W % 4 == 0, fp32 guides, the appendix solver;
                               FLR_ERR_UNSUPPORTED otherwise */
} flr_variant;

/* Per-block solver. */
typedef enum {
    FLR_SOLVER_APPENDIX = 0, /* the paper's normalised, regularised solve, eps_add + eps_mul */
    FLR_SOLVER_TIKHONOV = 1  /* Eq. tikhonov with Fig. 3's semantics:
                                A = (Mbar/n + eps_add I)^-1 Nbar/n on the full (Q+1) system, the
                                bias included (R18, R22); eps_mul is ignored.  flr_fit returns
                                raw-basis models; the denoise calls with fp32 guides evaluate
                                each block's model about its window mean, b0 + A.(x - mu), and
                                blend the four predictions (exact arithmetic: the same result;
                                in fp32 it avoids cancelling slopes ~cov/eps against the bias) */
} flr_solver;

typedef struct {
    int32_t block;    /* D_fit: block size in FIT pixels, in {1,2,4,8,16}; default 8 */
    int32_t upsample; /* U >= 1: output pixels per fit pixel (1 = plain denoise) */
    int32_t radius;   /* blur half-width R in blocks; 0 = auto = ceil(2 sigma / (block*U)) (R1) */
    int32_t variant;  /* flr_variant */
    double sigma;     /* Gaussian window std in OUTPUT pixels, > 0; default 10 */
    double eps_add;   /* additive regulariser epsilon >= 0; default 1e-5 */
    double eps_mul;   /* multiplicative regulariser epsilon^ in [0,1); default 1e-4 */
    int32_t solver;   /* flr_solver; default FLR_SOLVER_APPENDIX */
    int32_t flags;    /* FLR_FLAG_* bits; default 0 */
} flr_params;

/* The call's inputs (guides, radiance, albedo, direct light) were complete before the kernel
 * that precedes the call on `stream` began (e.g. written by a copy, or by an earlier call's
 * caller): the moment kernel then starts streaming them while that kernel drains, instead of
 * waiting for it (programmatic dependent launch).  Its dependents still launch only after
 * the preceding kernel completed, so the library's own workspace is never raced.  Without
 * the flag every call waits for the preceding kernel before reading its inputs. */
#define FLR_FLAG_INPUTS_READY 1

/* Fill *p with the defaults: block 8, upsample 1, radius 0 (auto), variant AUTO,
 * sigma 10, eps_add 1e-5, eps_mul 1e-4, solver APPENDIX, flags 0.  No-op on NULL. */
void flr_default_params(flr_params* p);

/* Static human-readable name of a status; never NULL. */
const char* flr_status_string(flr_status s);

/* Effective blur radius in blocks for params p (resolves radius == 0).  Returns -1
 * when p is NULL or invalid. */
int32_t flr_effective_radius(const flr_params* p);

/* Bytes of device workspace needed by flr_fit / flr_denoise /
 * flr_denoise_upsample for n frames of W_fit x H_fit fit pixels with Q guides. */
flr_status flr_workspace_size(int32_t n, int32_t Q, int32_t W_fit, int32_t H_fit,
                              const flr_params* p, size_t* bytes);

/* Fit: guides_fit [n][Q][H_fit][W_fit] and radiance_fit
 * [n][3][H_fit][W_fit] -> models [n][By][Bx][Q+1][3] (raw basis).  The blur std in
 * blocks is sigma / (block * upsample) (sigma is in output pixels). */
flr_status flr_fit(int32_t n, int32_t Q, int32_t W_fit, int32_t H_fit,
                   const float* guides_fit, const float* radiance_fit, const flr_params* p,
                   float* models, void* workspace, size_t workspace_bytes, flr_stream_t stream);

/* Apply: models [n][By][Bx][Q+1][3] whose blocks span
 * block_out OUTPUT pixels, guides_out [n][Q][H_out][W_out] -> out [n][3][H_out][W_out].
 * Requires Bx == ceil(W_out / block_out) and By == ceil(H_out / block_out).  Block
 * centres at (b + 1/2) block_out - 1/2, clamped at the borders (R4). */
flr_status flr_apply(int32_t n, int32_t Q, int32_t W_out, int32_t H_out, int32_t block_out,
                     int32_t Bx, int32_t By, const float* models, const float* guides_out,
                     float* out, flr_stream_t stream);

/* Denoise = fit + apply with the same guides (p->upsample must be 1). */
flr_status flr_denoise(int32_t n, int32_t Q, int32_t W, int32_t H, const float* guides,
                       const float* radiance, const flr_params* p, float* out,
                       void* workspace, size_t workspace_bytes, flr_stream_t stream);

/* Joint denoise + upsample: fit on (guides_lo, radiance_lo) with
 * block p->block, apply on guides_hi with block_out = block * U, U = p->upsample;
 * requires W_hi == U * W_lo and H_hi == U * H_lo. */
flr_status flr_denoise_upsample(int32_t n, int32_t Q, int32_t W_lo, int32_t H_lo,
                                const float* guides_lo, const float* radiance_lo,
                                int32_t W_hi, int32_t H_hi, const float* guides_hi,
                                const flr_params* p, float* out, void* workspace,
                                size_t workspace_bytes, flr_stream_t stream);

/* Half-precision guide planes: the paper's guide network runs in fp16
 * (P:414), so its enhanced guides X' arrive as IEEE binary16.  These entry
 * points take guides as binary16 bit patterns (uint16_t) and otherwise behave exactly as
 * their fp32 counterparts; every fp16 value is converted exactly to fp32 on load, so the
 * result equals the fp32 path run on the same values widened to fp32.  Radiance, models
 * and output stay fp32.  Only the TMA streaming kernels read fp16 planes, so they need
 * W % 8 == 0 (fit and output widths), 16-byte aligned planes, block in {4, 8, 16} and an
 * output block size (block * upsample) that is a multiple of 8; any other shape returns
 * FLR_ERR_UNSUPPORTED (nothing launched).  FLR_VARIANT_FUSED is not available here.
 * FLNR's split guides (fit on X'_model, apply X'_map) are the
 * denoise_upsample call with p->upsample == 1 and guides_lo = X'_model,
 * guides_hi = X'_map. */
flr_status flr_fit_f16(int32_t n, int32_t Q, int32_t W_fit, int32_t H_fit, const uint16_t* guides_fit,
                       const float* radiance_fit, const flr_params* p, float* models, void* workspace,
                       size_t workspace_bytes, flr_stream_t stream);
flr_status flr_denoise_f16(int32_t n, int32_t Q, int32_t W, int32_t H, const uint16_t* guides,
                           const float* radiance, const flr_params* p, float* out, void* workspace,
                           size_t workspace_bytes, flr_stream_t stream);
flr_status flr_denoise_upsample_f16(int32_t n, int32_t Q, int32_t W_lo, int32_t H_lo, const uint16_t* guides_lo,
                                    const float* radiance_lo, int32_t W_hi, int32_t H_hi,
                                    const uint16_t* guides_hi, const flr_params* p, float* out, void* workspace,
                                    size_t workspace_bytes, flr_stream_t stream);

/* The paper's protocol around FLR: the renderer's indirect
 * radiance is albedo-modulated, FLR denoises the DEMODULATED signal, and the result is
 * remodulated and the noise-free direct light added:
 *   y   = radiance_mod / max(albedo, albedo_floor)      per pixel and channel (R20)
 *   I   = flr_denoise(guides, y)                         (p->upsample must be 1)
 *   out = albedo * I + direct                            (R21; direct == NULL means zero)
 * radiance_mod, albedo, direct, out: [n][3][H][W] device planes; guides [n][Q][H][W].
 * albedo_floor > 0 (finite) only guards the division (SPEC's 1e-3 convention).
 * When W % 4 == 0, the planes are 16-byte aligned and p->block is 4, 8 or 16 the
 * demodulation runs inside the moment kernel's loads and (for block 8/16) the
 * remodulation inside the apply kernel's stores; any other shape runs two extra
 * elementwise kernels (the demodulated radiance is staged in `out`).  Same workspace as
 * flr_denoise.  Errors as flr_denoise; FLR_ERR_INVALID_VALUE for a NULL albedo or a
 * non-positive floor. */
flr_status flr_denoise_modulated(int32_t n, int32_t Q, int32_t W, int32_t H, const float* guides,
                                 const float* radiance_mod, const float* albedo, const float* direct,
                                 float albedo_floor, const flr_params* p, float* out, void* workspace,
                                 size_t workspace_bytes, flr_stream_t stream);

/* Optional per-launch timing for benchmarks.  `events` holds `capacity`
 * caller-created cudaEvent_t handles (create them with timing enabled).  The
 * traced calls record events[i] on `stream` immediately before their i-th
 * kernel launch and one more event after the last launch, so launch i took
 * cudaEventElapsedTime(events[i], events[i+1]).  `recorded` returns how many
 * events were recorded (launches + 1, or capacity if smaller).  The trace does
 * not change what is computed. */
typedef struct {
    void** events;    /* cudaEvent_t[capacity], caller-owned */
    int32_t capacity;
    int32_t recorded; /* out */
} flr_event_trace;

/* flr_denoise / flr_denoise_upsample with an optional event trace (NULL = none). */
flr_status flr_denoise_traced(int32_t n, int32_t Q, int32_t W, int32_t H, const float* guides,
                              const float* radiance, const flr_params* p, float* out,
                              void* workspace, size_t workspace_bytes, flr_stream_t stream,
                              flr_event_trace* trace);
flr_status flr_denoise_upsample_traced(int32_t n, int32_t Q, int32_t W_lo, int32_t H_lo,
                                       const float* guides_lo, const float* radiance_lo,
                                       int32_t W_hi, int32_t H_hi, const float* guides_hi,
                                       const flr_params* p, float* out, void* workspace,
                                       size_t workspace_bytes, flr_stream_t stream,
                                       flr_event_trace* trace);
flr_status flr_denoise_upsample_f16_traced(int32_t n, int32_t Q, int32_t W_lo, int32_t H_lo,
                                           const uint16_t* guides_lo, const float* radiance_lo, int32_t W_hi,
                                           int32_t H_hi, const uint16_t* guides_hi, const flr_params* p, float* out,
                                           void* workspace, size_t workspace_bytes, flr_stream_t stream,
                                           flr_event_trace* trace);
flr_status flr_denoise_f16_traced(int32_t n, int32_t Q, int32_t W, int32_t H, const uint16_t* guides,
                                  const float* radiance, const flr_params* p, float* out, void* workspace,
                                  size_t workspace_bytes, flr_stream_t stream, flr_event_trace* trace);
flr_status flr_denoise_modulated_traced(int32_t n, int32_t Q, int32_t W, int32_t H, const float* guides,
                                        const float* radiance_mod, const float* albedo, const float* direct,
                                        float albedo_floor, const flr_params* p, float* out, void* workspace,
                                        size_t workspace_bytes, flr_stream_t stream, flr_event_trace* trace);

/* Number of kernel launches the last successful call on this thread enqueued
 * (bench accounting; thread-local, not part of the computation). */
int32_t flr_last_launch_count(void);

/* Kernel name of launch i (0 <= i < flr_last_launch_count()) of the last successful
 * call on this thread; "" when out of range.  Static storage, never NULL. */
const char* flr_last_launch_name(int32_t i);

#ifdef __cplusplus
}
#endif
#endif /* FLR_H */
