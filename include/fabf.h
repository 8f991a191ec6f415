/*
 * fabf.h -- C ABI of the B200 (sm_100a) fast adaptive bilateral filter.
 *
 * Implements the per-pixel pipeline of Algorithm 1 of Gavaskar & Chaudhury,
 * "Fast Adaptive Bilateral Filtering", arXiv 1811.02308 (P:446-477 of
 * /root/reference/PAPER.md), with a box spatial kernel of half-width rho
 * (reading R1):
 *
 *   g-hat(i) = alpha_i + (beta_i - alpha_i) * (sum_k c_k I_{k+1}) / (sum_k c_k I_k)   eq.(29)
 *
 * where alpha_i / beta_i are the window min / max (eq.(8)), c the
 * degree-N moment-matching polynomial of the stretched local histogram
 * (eqs.(14),(19),(24) P:246-345; computed in the equivalent Legendre basis,
 * DESIGN.md section "Kernels"), and I_k the Gaussian integrals of eq.(28)
 * (P:382-441).  Pixels with alpha_i == beta_i return f(i) exactly.
 *
 * All image arguments are float32, batch x height x width, row-major,
 * contiguous.  img, theta and sigma share one intensity scale (any scale: the
 * filter is affine-equivariant, reading R4).  sigma(i) > 0 and finite
 * inputs are preconditions (unspecified output otherwise).
 *
 * Border handling: half-sample symmetric reflection (reading R2),
 * which needs 2*rho+1 <= min(height, width).
 *
 * Errors: every entry point returns a fabf_status_t; no C++ exception crosses
 * the ABI.  fabf_last_error_message() gives a thread-local detail string.
 * CUDA errors raised asynchronously by earlier work on the stream surface on a
 * later call (or on the caller's own synchronisation).
 *
 * Threading / ownership: the caller owns every image buffer and the stream;
 * a plan owns its device workspace.  Use one plan from one stream at a time.
 */
#ifndef FABF_H_
#define FABF_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FABF_VERSION 100 /* 1.0.0 */
#define FABF_MAX_N 10    /* largest supported polynomial degree N */

typedef enum {
  FABF_OK = 0,
  FABF_ERR_INVALID_ARGUMENT = 1, /* null/misaligned pointer, bad size, rho/N out of range, overlap */
  FABF_ERR_UNSUPPORTED = 2,      /* device is not sm_100 (B200), or N > FABF_MAX_N       */
  FABF_ERR_CUDA = 3,             /* a CUDA API call or kernel launch failed               */
  FABF_ERR_OUT_OF_MEMORY = 4     /* device or host allocation failed                      */
} fabf_status_t;

/* plan flags */
#define FABF_FLAG_LITERAL 0x1u /* eq.(29) exactly as printed: no guard (reading R7)       */
#define FABF_FLAG_CLAMP 0x2u   /* clamp g-hat to [alpha_i, beta_i] after the guard (reading R7)    */
#define FABF_FLAG_DEBUG 0x4u   /* validate the preconditions on the device every call: f, theta
                                  finite, sigma finite and > 0 (fabf_debug_status reads the result) */
#define FABF_FLAG_FUSED 0x8u   /* compute the bounds alpha, beta (step a1) inside the per-pixel
                                  kernel for every rho (one kernel reads f, theta, sigma and
                                  writes g-hat: north_star (e)).  Without it they are
                                  computed inside the kernel only for rho <= 5 on calls of at
                                  most 2^21 pixels and by a separate bounds kernel otherwise,
                                  the faster choice on B200.                 */

/* per-pixel diagnostic code bits (fabf_diag_t.code) */
#define FABF_CODE_IDENTITY 0x1u /* alpha == beta: g-hat = f(i)                               */
#define FABF_CODE_GUARD 0x2u    /* guard fired: T2 <= 0 or kappa > 1e3 -> N = 0 value          */
#define FABF_CODE_SMALL_LAMBDA 0x4u /* lambda < 2: integrals by fixed-node quadrature        */
#define FABF_CODE_FALLBACK 0x8u /* moments recomputed exactly (centring amplification flag)  */
#define FABF_CODE_FAR_THETA 0x10u /* theta_0 outside [-1, 2]: adaptive quadrature            */

typedef struct fabf_plan_s* fabf_plan_t;

/* Create a plan for images of shape batch x height x width (all >= 1,
 * batch*height*width < 2^31).  Allocates the plan's device workspace (alpha /
 * beta planes, per-64x64-tile bounds, the list of pixels flagged for the
 * exact-moment fallback and its counter) on the current device; no allocation
 * happens later in fabf_filter.  flags: FABF_FLAG_* (0 = guarded, unclamped).
 * Returns FABF_ERR_UNSUPPORTED when the current device is not compute
 * capability 10.0 (this library contains sm_100a code only).                  */
fabf_status_t fabf_plan(fabf_plan_t* plan, int batch, int height, int width, unsigned flags);

/* The filter.  img, theta, sigma, out: DEVICE pointers (float32,
 * batch*height*width, 16-byte aligned); out must not overlap any input.
 * rho >= 0 with 2*rho+1 <= min(height, width); 0 <= N <= FABF_MAX_N.
 * rho == 0 is an exact copy (every window is a single sample); rho <= 96.
 * stream: a cudaStream_t (NULL = legacy default stream).  Asynchronous, does
 * not synchronise and does not read device memory on the host; capturable
 * into a CUDA graph (tests/test_gpu_parity.py replays a captured call).
 * Kernels: rho <= 5 -> one fused kernel (bounds computed inside it) plus the
 * fallback kernel; rho > 5 -> bounds kernel, filter kernel, fallback kernel.
 * The output may differ from fabf_filter_host / fabf_filter_diag in the last
 * bits (segment boundaries set the tile-local centring).        */
fabf_status_t fabf_filter(fabf_plan_t plan, const float* img, const float* theta,
                          const float* sigma, int rho, int N, float* out, void* stream);

/* Optional per-pixel diagnostics (device pointers, batch*height*width each;
 * any member may be NULL).  kappa = sum_k |(2k+1) nu_k J_k| / T2 is the
 * condition number of the eq.(29) normaliser in the Legendre basis; t2n = T2/n
 * (n = (2rho+1)^2); code = FABF_CODE_* bits.                                   */
typedef struct {
  float* alpha;
  float* beta;
  float* kappa;
  float* t2n;
  unsigned char* code;
} fabf_diag_t;

/* fabf_filter plus diagnostics (diag may be NULL: then identical to
 * fabf_filter).                                                                */
fabf_status_t fabf_filter_diag(fabf_plan_t plan, const float* img, const float* theta,
                               const float* sigma, int rho, int N, float* out,
                               const fabf_diag_t* diag, void* stream);

/* Step a1 alone: alpha = window min, beta = window max (eq.(8)), box
 * half-width rho, same borders as fabf_filter.  Device pointers as above.      */
fabf_status_t fabf_bounds(fabf_plan_t plan, const float* img, int rho, float* alpha,
                          float* beta, void* stream);

/* End-to-end convenience: HOST pointers (pinned memory recommended: pageable
 * memory serialises the copies).  Copies the inputs to plan-owned device
 * buffers (allocated on first use) and the result back, pipelined by row
 * bands of whole 64-row tiles (up to 6 per frame, env FABF_HOST_BANDS=1..16
 * overrides; every band >= rho + 1 rows, the last one the smallest): inputs
 * on a plan-owned copy stream in the order img_{k+1}, theta_k, sigma_k, the
 * kernels of band k on `stream` as soon as those are resident, the output of
 * band k on a second copy stream.  Synchronises before returning.  Same
 * argument rules and errors as fabf_filter.                                    */
fabf_status_t fabf_filter_host(fabf_plan_t plan, const float* img, const float* theta,
                               const float* sigma, int rho, int N, float* out, void* stream);

/* NEXT-1: the paper's default spatial kernel (eq.(4)): omega(j) =
 * exp(-|j|^2 / 2 rho^2) on Omega = [-3 rho, 3 rho]^2 instead of the box.  The
 * bounds alpha, beta are the min / max over that whole window (every sample has
 * omega > 0); the moments of Algorithm 1 line 6 are Gaussian-weighted, by
 * exact separable FIR in fp64 (O(rho) per pixel and power -- the paper's own
 * runs used direct FIR too).  Same pointer rules, flags and errors as
 * fabf_filter with the window half-width 3 rho: 6 rho + 1 <= min(height,
 * width), 0 <= rho <= 16.  Three kernels (bounds, moments + per-pixel, exact
 * fallback).                                                                 */
fabf_status_t fabf_filter_gauss(fabf_plan_t plan, const float* img, const float* theta, const float* sigma,
                                int rho, int N, float* out, void* stream);

/* NEXT-2: the sharpening / noise-removal application (after Zhang &
 * Allebach): the range-kernel maps are produced on the device from f alone,
 *   theta(i) = f(i) + zeta(i), zeta = f - fbar (fbar: box mean over the same
 *              (2 rho + 1)^2 window Omega),
 *   sigma(i) = sigma_hi - (sigma_hi - sigma_lo) min(|LoG f|(i) / log_sat, 1)
 * (the paper says only "an affine mapping on the absolute value" of the LoG
 * response that maps low values to high sigma: the LoG scale and the map are
 * parameters, reading R15).  LoG: the sampled, normalised Gaussian of
 * std log_scale on |x| <= ceil(4 log_scale) (<= 16) and its analytic second
 * derivative, borders reflected.                                              */
typedef struct {
  float log_scale; /* LoG Gaussian std (pixels)                    */
  float sigma_lo;  /* sigma where |LoG| >= log_sat (edges)         */
  float sigma_hi;  /* sigma where LoG = 0 (flat areas)             */
  float log_sat;   /* |LoG| (intensity units) at which sigma_lo is reached */
} fabf_sharpen_t;

/* The maps alone: theta, sigma (device, batch x height x width fp32) from img.
 * Asynchronous.  INVALID_ARGUMENT for bad parameters or overlapping buffers.   */
fabf_status_t fabf_sharpen_maps(fabf_plan_t plan, const float* img, int rho, const fabf_sharpen_t* prm,
                                float* theta, float* sigma, void* stream);

/* The whole application: the maps into plan-owned buffers (allocated on first
 * use, shared with fabf_filter_host), then fabf_filter with them -- img and out
 * are the only caller buffers (4 + 4 bytes per pixel cross PCIe end to end).  */
fabf_status_t fabf_filter_sharpen(fabf_plan_t plan, const float* img, int rho, int N, const fabf_sharpen_t* prm,
                                  float* out, void* stream);

/* NEXT-2, second application: texture filtering.  The sigma map is
 * produced on the device from f alone,
 *   mRTV(i)  = Delta(i) max_{j in W_i} |grad f(j)| / (sum_{j in W_i} |grad f(j)| + eps)
 *   Delta(i) = max_{W_i} f - min_{W_i} f
 *   sigma(i) = sigma_hi - (sigma_hi - sigma_lo) min(mRTV(i) / mrtv_sat, 1)
 * ("an affine transformation of mRTV, sigma high whenever mRTV is low", P:847;
 * the paper fixes neither W_i, the gradient stencil, eps nor the map: DESIGN.md
 * reading R19 -- W_i the box of half-width `patch`, forward differences with
 * the image reflected at its borders, Euclidean norm).                        */
typedef struct {
  int patch;          /* half-width of the neighbourhood W_i, 0..16             */
  float sigma_lo;     /* sigma where mRTV >= mrtv_sat (strong edges)            */
  float sigma_hi;     /* sigma where mRTV = 0 (texture, flat areas)             */
  float mrtv_sat;     /* mRTV (intensity units) at which sigma_lo is reached    */
  float eps;          /* the paper's epsilon (> 0, intensity units)             */
  float second_scale; /* sigma factor of the second smoothing pass (paper: 0.8) */
} fabf_texture_t;

/* The map alone: sigma (and, if `mrtv` is not NULL, mRTV itself) as device
 * batch x height x width fp32 planes.  Asynchronous.  INVALID_ARGUMENT for bad
 * parameters or overlapping buffers.                                           */
fabf_status_t fabf_texture_maps(fabf_plan_t plan, const float* img, const fabf_texture_t* prm, float* sigma,
                                float* mrtv, void* stream);

/* The whole application ("we apply Algorithm 1 thrice"): pass 1 =
 * fabf_filter(img; theta = img, sigma); pass 2 = fabf_filter(pass 1; theta =
 * pass 1, second_scale * sigma) with the SAME map; out = the sharpening
 * application (fabf_filter_sharpen's rule, window half-width rho_sharpen) of
 * pass 2.  Maps and intermediates live in plan-owned buffers (allocated on
 * first use, shared with fabf_filter_host); `pass1` / `pass2`, when not NULL,
 * are device planes that receive the intermediates instead.  Every pass obeys
 * the plan's flags; fabf_last_fallback_count reports the last pass.
 * Asynchronous on `stream`; errors as fabf_filter / fabf_sharpen_maps.         */
fabf_status_t fabf_filter_texture(fabf_plan_t plan, const float* img, int rho, int N, const fabf_texture_t* tprm,
                                  int rho_sharpen, const fabf_sharpen_t* sprm, float* out, float* pass1,
                                  float* pass2, void* stream);

/* The same three passes with the CALLER's sigma map (device, batch x height x
 * width fp32, > 0, 16-byte aligned; pass 1 uses it as it is, pass 2 scaled by
 * second_scale).  This is how the paper treats colour images (P:848, P:853:
 * mRTV and sigma "on a grayscale version of the color image", the channels
 * then filtered one by one): fabf_texture_maps on the grey plane, that map
 * repeated for every channel plane of a planar batch, then this call.         */
fabf_status_t fabf_filter_texture_map(fabf_plan_t plan, const float* img, const float* sigma_map,
                                      float second_scale, int rho, int N, int rho_sharpen,
                                      const fabf_sharpen_t* sprm, float* out, float* pass1, float* pass2,
                                      void* stream);

/* The baseline the paper compares with (NEXT-4): Mozerov & van de Weijer's
 * uniform-prior filter with Delta = 0 (Fig.3) -- eq.(29) at
 * N = 0 fitted on [f(i), 2 fbar(i) - f(i)] (fbar = the box mean over the same
 * (2 rho + 1)^2 window) instead of [alpha_i, beta_i]; f(i) where that interval
 * is a point.  Same arguments, pointer rules and errors as fabf_filter
 * (without N); FABF_FLAG_LITERAL / CLAMP do not apply (the N = 0 ratio needs
 * no guard).                                                                  */
fabf_status_t fabf_filter_mozerov(fabf_plan_t plan, const float* img, const float* theta,
                                  const float* sigma, int rho, float* out, void* stream);

/* Colour / multi-channel images, filtered channel by channel as the paper does
 * (P:855): img, theta, sigma and out are DEVICE buffers of B/C images of
 * height x width x `channels` fp32, channel-interleaved (pixel-major, the
 * usual RGB layout), 16-byte alignment not required.  The plan's batch B
 * counts planes (images x channels) and must be a multiple of `channels`.
 * The channels are moved to plan-owned planar buffers (allocated on first
 * use, shared with fabf_filter_host), filtered as a batch of planes exactly
 * as fabf_filter would, and moved back.  Asynchronous on `stream`.  Errors as
 * fabf_filter, plus INVALID_ARGUMENT if `channels` does not divide the batch. */
fabf_status_t fabf_filter_interleaved(fabf_plan_t plan, const float* img, const float* theta,
                                      const float* sigma, int channels, int rho, int N, float* out,
                                      void* stream);

/* Number of pixels the last fabf_filter* call on this plan routed to the
 * exact-moment fallback (synchronises the plan's stream to read it).         */
fabf_status_t fabf_last_fallback_count(fabf_plan_t plan, long long* count);

/* Number of kernels the last fabf_filter / fabf_filter_diag / fabf_filter_host
 * / fabf_filter_events / fabf_filter_profile call on this plan launched (all
 * bands of a host call; set when the call returns, no synchronisation).
 * INVALID_ARGUMENT for NULL pointers.                                         */
fabf_status_t fabf_last_launch_count(fabf_plan_t plan, int* count);

/* FABF_FLAG_DEBUG plans only: the device-side precondition check of the last
 * fabf_filter* call on this plan (f and theta finite, sigma finite and > 0 --
 * the preconditions of eq.(29), whose violation otherwise gives unspecified
 * values).  Synchronises the plan's last stream, then writes the number of
 * violating pixels to *bad_count and the flat index (b*H*W + y*W + x) of the
 * first one to *first_bad (-1 if none).  The check costs one extra read of
 * f, theta, sigma per call.  INVALID_ARGUMENT for NULL pointers or a plan
 * made without the flag.                                                      */
fabf_status_t fabf_debug_status(fabf_plan_t plan, long long* bad_count, long long* first_bad);

/* Profiling variant of fabf_filter: same work on the same stream, with CUDA
 * events recorded between the kernels; synchronises the stream and writes the
 * device time (ms) of each stage to stage_ms[0..3] = {bounds (step a1),
 * always 0 (kept for layout), moments + per-pixel filter (a2-a8), exact-moment
 * fallback}.                                                                   */
fabf_status_t fabf_filter_profile(fabf_plan_t plan, const float* img, const float* theta,
                                  const float* sigma, int rho, int N, float* out, void* stream,
                                  float stage_ms[4]);

/* Same work as fabf_filter, recording five caller-owned CUDA events
 * (cudaEvent_t, created with timing enabled, passed as void*) on `stream`
 * around the kernels: events[0] before the bounds kernel, [1] and [2] after
 * it, [3] after the moments + per-pixel kernel, [4] after the fallback kernel.
 * Does not synchronise: per-kernel device times of a timed region without
 * perturbing it.  Errors as fabf_filter; NULL events -> INVALID_ARGUMENT.     */
fabf_status_t fabf_filter_events(fabf_plan_t plan, const float* img, const float* theta,
                                 const float* sigma, int rho, int N, float* out, void* stream,
                                 void* const events[5]);

/* Free the plan (NULL is a no-op).  No work using the plan may be pending.   */
fabf_status_t fabf_destroy(fabf_plan_t plan);

const char* fabf_status_string(fabf_status_t status);
const char* fabf_last_error_message(void);
int fabf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FABF_H_ */
