/*
 * pa.h — C ABI of libpa: the PA-SFM differentiable acoustic radiation operator
 * (arXiv 2604.09643) on NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n (the paper's LaTeX source), S:n = SPEC.md line n,
 * R<k> = a reading of the paper listed in DESIGN.md §3.
 *
 * The operator (Eq. gpu_forward_model; Eq. 1):
 *
 *   traces[f][e][j] = sum_k p0[k] * D/(2r) * K(|D|) * [|D| <= kappa*sigma]
 *   r = |x_fe - y_k|,  D = r - c (t0 + j dt),  x_fe = R_f tmpl[e] + t_f  (Stage 4)
 *   K = "the designated kernel function", scale s = sigma (pa_acq.kernel, R23):
 *     PA_KERNEL_GAUSS  K = exp(-D^2 / (2 s^2))   [default]
 *     PA_KERNEL_EXP    K = exp(-|D| / s)           (outgoing term of P:313-316)
 *     PA_KERNEL_POW    K = (D^2 + s^2)^(-nu)       (outgoing term of P:318-322)
 *   y_k = origin + pitch * (i, j, l),  k = i + nx*(j + ny*l)    (x fastest, R7)
 *
 * Units: mm, µs, mm/µs.  Arithmetic: fp32 with fp64 per-tile anchors.  For the
 * Gaussian kernel the forward and the adjoint evaluate the sum through approximations below fp32
 * accumulation level (a rank-R separable pulse basis with fixed-point deposits; Taylor moment
 * filters — reading R24); pa_get_plan_info reports the orders and measured errors for a geometry,
 * and geometries outside the bounds run the direct kernels.
 *
 * Conventions for every entry point
 *   - Array arguments are caller-owned DEVICE pointers (cudaMalloc / torch), fp32,
 *     C-contiguous, 4-byte aligned, unless stated "host".  Outputs are overwritten.
 *     The library keeps no pointer after a call returns.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).  Kernels are
 *     enqueued asynchronously on it.  Validation (arguments, supported geometry, degenerate
 *     geometry) runs before any output is written; in pa_forward / pa_adjoint / pa_pose_grad /
 *     pa_adjoint_pose the degenerate-geometry check enqueues a tiny kernel and synchronises
 *     `stream` to read its verdict.  pa_step does NOT synchronise: its check stays on the
 *     device (a degenerate step skips its Adam updates) and pa_step_status() reports it.
 *   - F == 0 is a no-op returning PA_OK.
 *   - Results are bitwise deterministic run-to-run for a fixed GPU, shapes and inputs
 *     (no floating-point atomics: the forward's shared-memory deposits are fixed-point
 *     integer additions, which are associative; all floating-point reductions in fixed order).
 *   - Errors: the status code; pa_last_error() returns a thread-local message.
 *   - A pa_ctx owns only internal workspace (pose-gradient partials, scratch) and a cache of the
 *     last geometry's plan (its host-side factorisation, ~20-40 ms, is recomputed only when the
 *     grid, acquisition, E or policy change); use one context per stream.  Calls on different
 *     contexts may run concurrently.
 */
#ifndef PA_H
#define PA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PA_OK = 0,
    PA_EINVAL = 1,        /* non-positive dims/pitch/c/dt/nt/sigma, kappa < 4, bad cfg       */
    PA_ESHAPE = 2,        /* E < 1, F < 0, null or misaligned pointer                         */
    PA_EDEGENERATE = 3,   /* an element lies within 1e-6 mm of a voxel centre (R10) */
    PA_ECUDA = 4,         /* a CUDA call or launch failed                                     */
    PA_ENOMEM = 5,        /* workspace allocation failed                                      */
    PA_EUNSUPPORTED = 6   /* geometry outside every kernel (see pa_get_plan_info): the Gaussian
                             fast path runs any L_min = floor(2 kappa sigma/(c dt)) in [21, 512]
                             (nt + L_min row accumulators permitting); the direct kernels (the
                             exponential and power-law families; shorter Gaussian windows) run
                             spread <= L_min < 160 with L_min + spread <= 128, spread =
                             floor(sqrt(3) pitch/(c dt)) + 2; every other window runs the generic
                             kernels (any L_min and family, nt <= 51200); TGV 3 nx ny nz < 2^31 */
} pa_status;

/* Voxel grid.  Voxel (i,j,l) centre = origin + pitch*(i,j,l); p0[l][j][i]. */
typedef struct {
    int32_t nx, ny, nz;
    float origin[3];
    float pitch;
} pa_grid;

/* Kernel families of the designated kernel K (f3 of SURVEY §8; reading R23). */
typedef enum {
    PA_KERNEL_GAUSS = 0, /* exp(-D^2/2s^2): the paper's kernel (Eq. gaussian_far_field)    */
    PA_KERNEL_EXP = 1,   /* exp(-|D|/s): far field of the exponential distribution  */
    PA_KERNEL_POW = 2    /* (D^2+s^2)^-nu, nu in (1/2, 16]: far field of the power law     */
} pa_kernel;

/* Acquisition + kernel.  Sample j at t0 + j*dt (R5); speed of sound c;
 * kernel scale sigma (the Gaussian width; s of the other families, R23); window
 * |D| <= kappa*sigma, kappa >= 4 (R4; kappa <= 30 for PA_KERNEL_EXP so that the factored
 * recurrence constants stay in fp32 range).  `kernel` is a pa_kernel; `nu` is read only for
 * PA_KERNEL_POW.  Bad kernel / nu / kappa -> PA_EINVAL. */
typedef struct {
    float c, t0, dt;
    int32_t nt;
    float sigma, kappa;
    int32_t kernel;
    float nu;
} pa_acq;

typedef struct pa_ctx pa_ctx;

/* Create a context bound to `device` (cudaSetDevice is NOT changed for the caller's thread
 * beyond the duration of the call).  *ctx = NULL on failure. */
pa_status pa_create(pa_ctx **ctx, int device);
void pa_destroy(pa_ctx *ctx);

/* Kernel-selection policy of a context (default 0: the fastest kernels the geometry supports,
 * DESIGN.md §6).  Bits force the alternatives, for tests and diagnostics: the direct forward K1,
 * the direct adjoint K2, or prefer the rank-R-basis adjoint K2s / the moment-filter adjoint K2c.
 * A forced direct kernel whose window class does not hold the geometry runs as the generic kernels
 * (K1g / K2g + K3g); a preferred adjoint that is unavailable falls back to the default choice.
 * Unknown bits -> PA_EINVAL.  The policy is per context (no global state). */
enum {
    PA_POLICY_DEFAULT = 0,
    PA_POLICY_FWD_DIRECT = 1,
    PA_POLICY_ADJ_DIRECT = 2,
    PA_POLICY_ADJ_SVD = 4,
    PA_POLICY_ADJ_TAYLOR = 8
};
pa_status pa_set_policy(pa_ctx *ctx, int32_t policy);

/* Thread-local description of the last error on this thread ("" if none). */
const char *pa_last_error(void);

/* Library version string. */
const char *pa_version(void);

/* Running count of CUDA kernels this library has enqueued from the calling thread (every
 * entry point, all streams).  Difference it around a region to count that region's launches. */
long long pa_launch_count(void);

/*
 * a2 — forward radiation (Eq. gpu_forward_model).
 *   tmpl   [E][3]      array template x^_e
 *   poses  [F][12]     R_f row-major 3x3 then t_f (x_fe = R_f x^_e + t_f)
 *   p0     [nz][ny][nx] initial-pressure amplitudes P_c
 *   traces [F][E][nt]  output (overwritten)
 */
pa_status pa_forward(pa_ctx *ctx, const pa_grid *grid, const pa_acq *acq, const float *tmpl, int32_t E,
                     const float *poses, int32_t F, const float *p0, float *traces, void *stream);

/*
 * a4 — adjoint back-projection, the exact transpose of pa_forward:
 *   grad_p0[k] = sum_f sum_e sum_j cot[f][e][j] * D/(2r) K(|D|) [|D| <= kappa sigma]
 *   cot [F][E][nt] cotangent dL/dtraces;  grad_p0 [nz][ny][nx] output (overwritten).
 */
pa_status pa_adjoint(pa_ctx *ctx, const pa_grid *grid, const pa_acq *acq, const float *tmpl, int32_t E,
                     const float *poses, int32_t F, const float *cot, float *grad_p0, void *stream);

/*
 * a5+a6 — pose gradient ("sensor spatial coordinates"; Stage 4 P:109-115):
 *   grad_elem[f][e] = sum_k p0[k] sum_j cot[f][e][j] d/dr[D K(|D|)/(2r)] (x_fe - y_k)/r
 *                     (window indicator held constant, R11)
 *   grad_pose[f] = [ dL/dR_f (row-major 3x3) = sum_e grad_elem[f][e] tmpl[e]^T , dL/dt_f = sum_e grad_elem[f][e] ]
 *   grad_pose [F][12] output; grad_elem [F][E][3] output or NULL.
 */
pa_status pa_pose_grad(pa_ctx *ctx, const pa_grid *grid, const pa_acq *acq, const float *tmpl, int32_t E,
                       const float *poses, int32_t F, const float *p0, const float *cot, float *grad_pose,
                       float *grad_elem, void *stream);

/* Fused a4+a5+a6 in one pass over (voxel, element, sample): both outputs of pa_adjoint and
 * pa_pose_grad (identical values).  grad_elem may be NULL. */
pa_status pa_adjoint_pose(pa_ctx *ctx, const pa_grid *grid, const pa_acq *acq, const float *tmpl, int32_t E,
                          const float *poses, int32_t F, const float *p0, const float *cot, float *grad_p0,
                          float *grad_pose, float *grad_elem, void *stream);

/*
 * Unit of work: exact number of (voxel, element, sample) terms with
 * |D| <= kappa sigma and 0 <= j < nt, evaluated in fp64 with the literal predicate.
 *   total (host, int64) ; per_frame (host [F] int64, nullable).  Synchronises `stream`.
 */
pa_status pa_count(pa_ctx *ctx, const pa_grid *grid, const pa_acq *acq, const float *tmpl, int32_t E,
                   const float *poses, int32_t F, int64_t *total, int64_t *per_frame, void *stream);

/*
 * a3 — loss and cotangent from traces (Eq. 2 data term P:85 / Eq. 3 NC P:91-93, Eq. 4 mask P:112-114):
 *   kind 0 (MSE): L = sum (y - S)^2, cot = 2 (y - S)
 *   kind 1 (NC):  per row (f,e): L_fe = -cov(y,S)/(sd_y sd_S) (population), cot = dL/dy
 *   y, S, cot [F][E][nt]; row_mask [F][E] uint8 or NULL (masked rows: zero loss and cotangent);
 *   cot may alias y.  loss (device, 1 float) = sum of row losses in fixed order;
 *   row_loss (device [F][E] float, nullable) receives the per-row losses (NC: -correlation).
 */
pa_status pa_loss(pa_ctx *ctx, int32_t kind, const float *y, const float *S, const uint8_t *row_mask, int32_t F,
                  int32_t E, int32_t nt, float *cot, float *loss, float *row_loss, void *stream);

/* All-reduce callback (sum, in place, on `stream`) — lets the caller's NCCL process group
 * combine dL/dp0 across frame shards (Stage 5).  Return 0 on success.  NULL = one rank. */
typedef int (*pa_allreduce_fn)(float *buf, size_t n, void *stream, void *user);

typedef struct {
    float lr_p0, lr_rot, lr_trans;  /* Adam learning rates: p0, Euler angles, translation        */
    float beta1, beta2, eps;        /* Adam                                     */
    int32_t step;                   /* Adam step t >= 1 (bias correction)                         */
    int32_t loss_kind;              /* 0 MSE (Eq. 2), 1 NC (Eq. 3/4)                              */
    int32_t update_p0, update_pose; /* apply the p0 / pose updates (update_pose = 0 with grad_euler
                                       NULL skips the pose gradient: the adjoint runs without it)  */
    float tgv_lambda;               /* Eq. 2 weight of the TGV^2 term (0 = off; R20)        */
    float tgv_alpha1, tgv_alpha0;   /* TGV^2 first / second order weights (R20)        */
    float tgv_eps;                  /* smoothing of the norms, phi(v) = sqrt(|v|^2+eps^2) - eps   */
} pa_step_cfg;

/*
 * Eq. 2 regulariser, TGV^2 reading R20: with forward differences and
 * O = {x : x_d <= n_d - 2},
 *   L = alpha1 sum_O phi(grad P - w) + alpha0 sum_O phi(E w),  E w = (grad w + grad w^T)/2
 *   P [nz][ny][nx], w [3][nz][ny][nx] (components x, y, z); value (device, 1 float);
 *   grad_P, grad_w outputs (overwritten).  HBM-bound stencil, deterministic.
 *   Errors: PA_EUNSUPPORTED when 3 nx ny nz >= 2^31 (32-bit offsets); pa_step with
 *   tgv_lambda > 0 returns the same.
 */
pa_status pa_tgv(pa_ctx *ctx, const pa_grid *grid, const float *P, const float *w, float alpha1, float alpha0,
                 float eps, float *value, float *grad_P, float *grad_w, void *stream);

/*
 * One SfM iteration over this rank's F frames (Alg. 1 Stages 1/4/5 objective):
 *   poses <- Euler ZYX(euler_t) (R8), y = forward(p0), (L, cot) = loss(y, meas),
 *   grad_p0 = adjoint(cot) [all-reduced across ranks by `ar`], grad_pose, dL/dEuler,
 *   Adam on p0 with clamp p0 >= 0, Adam on euler_t (angles lr_rot, translation lr_trans).
 *   meas      [F][E][nt]   measured traces S
 *   row_mask  [F][E] uint8 or NULL
 *   p0        [nz][ny][nx] in/out;   euler_t [F][6] (a, b, c, tx, ty, tz) in/out
 *   adam_p0   [2][nz*ny*nx] (m, v) in/out;   adam_pose [2][F][6] in/out
 *   grad_p0   [nz*ny*nx]   out (after the all-reduce), caller-owned so `ar` can name it
 *   loss      [2]          out: local loss, global loss (after `ar` on a copy)
 *   grad_euler [F][6]      out or NULL
 *   row_loss  [F][E]       out or NULL: per-row losses of this rank's frames (before the update),
 *                          for host-side inlier decisions (Eq. 4 mask)
 *   tgv_w     [3][nvox]    TGV auxiliary field, in/out (Adam with lr_p0); NULL iff tgv_lambda == 0
 *   adam_w    [2][3][nvox] its Adam state; NULL iff tgv_lambda == 0
 *   With tgv_lambda > 0, grad_p0 on return includes lambda * dTGV/dP (added after the
 *   all-reduce, identically on every rank) and loss[1] includes lambda * TGV.
 *   `ar` is called on the calling thread, in order, for grad_p0 (nvox floats) and for loss + 1
 *   (1 float); it must enqueue the sum on `stream` (or complete it before returning) so that the
 *   kernels pa_step enqueues after it see the reduced values.  A non-zero return -> PA_ECUDA.
 *   No host synchronisation: the degenerate-geometry check (R10) runs on the device; when it
 *   fires the step's Adam updates are skipped (p0, euler_t, tgv_w and every Adam state are left
 *   unchanged; grad_p0 / loss are unspecified) and pa_step_status() returns PA_EDEGENERATE.
 *   All other errors are returned by pa_step itself, before any device work.
 */
pa_status pa_step(pa_ctx *ctx, const pa_grid *grid, const pa_acq *acq, const float *tmpl, int32_t E, int32_t F,
                  const float *meas, const uint8_t *row_mask, float *p0, float *euler_t, float *adam_p0,
                  float *adam_pose, const pa_step_cfg *cfg, pa_allreduce_fn ar, void *user, float *grad_p0,
                  float *loss, float *grad_euler, float *row_loss, float *tgv_w, float *adam_w, void *stream);

/* Plan of the kernels pa_forward / pa_adjoint_pose / pa_step run for this geometry (host only:
 * no device work, no context).  For tests and diagnostics.  PA_EUNSUPPORTED /
 * PA_EINVAL as the entry points for a geometry outside the compiled window classes. */
typedef struct {
    int32_t lmin;        /* L_min = floor(2 kappa sigma / (c dt)): windows have L_min or L_min+1 samples */
    int32_t fwd_deposit; /* 1: the deposit-form forward K1d runs (Gaussian kernel); 0: direct K1 */
    int32_t dep_rank;    /* K1d: separable rank R of the pulse factorisation                     */
    int32_t dep_warps;   /* K1d: warps per CTA (8: two CTAs per SM, 16: one)                    */
    double dep_err;      /* K1d: max |G - sum_m phi_m psi_m| / max |G| on a fine grid (R24)     */
    int32_t adj_taylor;  /* 1: the moment-filter adjoint K2a + K2c is available; 0: direct K2     */
    int32_t tay_order;   /* K2a/K2c: Taylor order M of the moment filters                       */
    double tay_err;      /* K2a/K2c: host bound on the Taylor remainder, relative to sum |terms| */
    int32_t adj_svd;     /* 1: the adjoint runs in the forward's basis (K2s: when K2c's bounds fail)  */
    double svd_derr;     /* K2s: max error of d/dt of the factorisation (pose moment), relative  */
    int32_t dep_groups;  /* K1d: round-accumulator copies (2 when pitch < 4 c dt, else 1)         */
    int32_t dep_ring;    /* K1d: positions of the round-accumulator ring (= nt + L_min: no ring)  */
    int32_t adj_kernel;  /* the adjoint that runs: 0 direct K2, 1 moment-filter K2a+K2c, 2 K2s     */
    int32_t direct_class;/* direct kernels (K1/K2): L_min of the compiled class, or -capacity of the
                            runtime class (L_min + cluster spread <= capacity), 0 if none fits     */
    int32_t dep_round;   /* K1d: tiles per warp per round (8 when its ring keeps the CTAs per SM, else 4) */
    int32_t generic;     /* 1: a pass runs the generic kernels K1g / K2g+K3g (no direct class holds L_min) */
} pa_plan_info;
pa_status pa_get_plan_info(const pa_grid *grid, const pa_acq *acq, int32_t E, pa_plan_info *out);
/* The same for a context (its pa_set_policy applied). */
pa_status pa_ctx_plan_info(pa_ctx *ctx, const pa_grid *grid, const pa_acq *acq, int32_t E, pa_plan_info *out);

/* Verdict of the last pa_step on this context: synchronises on the step's degenerate-geometry
 * check (not on the rest of the step) and returns PA_EDEGENERATE (message naming the frame,
 * element and voxel) if it fired, else PA_OK.  Idempotent until the next pa_step. */
pa_status pa_step_status(pa_ctx *ctx);

/* Kernel-level timing of the last pa_step / pa_forward / pa_adjoint_pose call on this context
 * (CUDA events recorded on `stream`): ms of the forward kernel and of the adjoint+pose kernel.
 * Synchronises the events.  Either pointer may be NULL. */
pa_status pa_last_kernel_ms(pa_ctx *ctx, float *forward_ms, float *adjoint_ms);

#ifdef __cplusplus
}
#endif
#endif /* PA_H */
