// pa_plan.h — host-side declarations shared by libpa's translation units: the per-call plan (geometry
// constants, the kernels chosen for it) and the launchers each kernel family's .cu file instantiates.
// Device code lives in pa_kernels.cuh; the C ABI in pa_api.cu.  Citations as in pa_kernels.cuh.
#pragma once
#include "pa.h"
#include "pa_kernels.cuh"

#include <cstddef>

namespace pa {

// ------------------------------------------------------------------ errors / launch accounting
pa_status fail(pa_status s, const char *fmt, ...);
extern thread_local long long g_nlaunch;  // kernels enqueued by this thread (pa_launch_count)

#define CUDA_TRY(x)                                                                          \
    do {                                                                                     \
        cudaError_t _e = (x);                                                                \
        if (_e != cudaSuccess) return fail(PA_ECUDA, "%s: %s", #x, cudaGetErrorString(_e)); \
    } while (0)

// ------------------------------------------------------------------ direct-kernel window classes
// K1 / K2 (the direct kernels: exponential and power-law families, Gaussian fallback) keep the window
// in registers / staged segments whose sizes are compile-time: L_min, the cluster window-base spread
// OMAX, the tile span SPAN and the segment SEG.
struct Klass {
    int lmin, omax, span, seg;
};
constexpr Klass kClasses[] = {{53, 11, 58, 128}, {26, 6, 30, 64}, {106, 21, 114, 256}};
constexpr int kNumClasses = (int)(sizeof kClasses / sizeof kClasses[0]);
// Runtime classes of the direct kernels (r2, R26): L_min, the cluster spread OMAX and the recurrence centre
// come from the plan; K1 holds a register window of capacity rc >= L_min + OMAX and a flush buffer for a
// tile span <= span; K2 stages segments of the plan's length (L_min + 1 <= ADJ_LCAP).  Plan::klass =
// KLASS_RT + index.
struct RtKlass {
    int rc, span;
};
constexpr RtKlass kRtClasses[] = {{48, 80}, {80, 96}, {128, 128}};
constexpr int kNumRtClasses = (int)(sizeof kRtClasses / sizeof kRtClasses[0]);
constexpr int KLASS_RT = 100;

// kernel-selection policy of a context (pa_set_policy; PA_POLICY_* in pa.h)
struct Plan {
    Geo g;
    FwdConst fc;      // direct forward K1 constants
    AdjConst ac;      // direct adjoint K2 constants
    TayFilt tf;       // K2a filter taps
    TayConst tc;      // K2c series constants
    bool tay_ok;      // Taylor remainder below the bound for this geometry (K2a/K2c available)
    int tay_NF;       // its record size (8 or 12 floats; TayCfg)
    int tay_pad;      // zero positions on each side of a K2a record row
    int tay_sentinel; // record index base of a culled (tile, element) in K2c (lands in the leading padding)
    double tay_err;   // host bound on the remainder (relative to sum |terms|)
    DepConst dc;      // deposit-form forward constants (Gaussian)
    SvdConst sv;      // the same factorisation for the adjoint K2s (unscaled)
    double svd_derr;  // measured error of its t-derivative (the pose moment), relative to max |dG/dt|
    bool dep_ok;      // factorisation error below the bound for this geometry (K1d available)
    int dep_R;        // separable rank (5 or 6)
    int dep_nw;       // K1d warps per CTA (8: two CTAs per SM; 16: one)
    int dep_g;        // K1d round-accumulator copies (lane l deposits into copy l % dep_g)
    int dep_tpr;      // K1d tiles per warp per round (8 when it keeps the resident CTAs per SM of 4, else 4)
    double dep_err;   // measured error of the factorisation (relative to max |G|)
    int klass;        // direct-kernel class (index into kClasses) or -1
    int fam;          // pa_kernel (KF_*)
    int policy;       // PA_POLICY_* bits
    bool fwd_dep;     // the forward runs K1d (else the direct K1, or K1g when no direct class holds it)
    int adj;          // the adjoint: ADJ_TAY (K2a/K2c), ADJ_SVD (K2s) or ADJ_DIRECT (K2, or K2g/K3g)
    bool gen;         // no direct-kernel class holds the geometry: the direct passes run the generic K1g/K2g/K3g
    int gen_nw;       // K1g warps per CTA (warp-private traces of nt floats in shared memory)
    double gen_dt, gen_sig;  // fp64 copies of dt and sigma for the generic kernels' literal window predicate
};
enum { ADJ_DIRECT = 0, ADJ_TAY = 1, ADJ_SVD = 2 };

struct AdjLaunch {
    int P = 0, Fc = 0;
    size_t smem = 0;
};

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Device workspace of a context used by the adjoint launchers (frame-chunk filters).
pa_status ctx_filter_ws(pa_ctx *ctx, size_t bytes, float **out);
int ctx_nsm(const pa_ctx *ctx);
unsigned *ctx_pmax(pa_ctx *ctx);  // one device word for K1d's max |p0|

// ------------------------------------------------------------------ launchers (one .cu per family)
// forward: mode FWD_TRACE / FWD_MSE / FWD_NC (pa_kernels.cuh), meas/mask/rowloss for the fused a3
pa_status launch_forward_dep(pa_ctx *ctx, const Plan &pl, const float *poses, const float *tmpl, const float *p0,
                             float *out, int mode, const float *meas, const uint8_t *mask, double *rowloss,
                             cudaStream_t st);
pa_status launch_forward_direct(const Plan &pl, const float *poses, const float *tmpl, const float *p0, float *out,
                                int mode, const float *meas, const uint8_t *mask, double *rowloss, cudaStream_t st);
// adjoint (+ pose partials): dry = size the launch only (L), no device work
pa_status launch_adjoint_tay(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses, const float *tmpl,
                             const float *p0, const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry,
                             cudaStream_t st);
pa_status launch_adjoint_svd(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses, const float *tmpl,
                             const float *p0, const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry,
                             cudaStream_t st);
pa_status launch_adjoint_direct(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses,
                                const float *tmpl, const float *p0, const float *cot, float *grad_p0, float *partial,
                                AdjLaunch &L, bool dry, cudaStream_t st);
// generic kernels (k_generic.cu): any window length and family, literal window predicate, fp64 geometry
pa_status launch_forward_generic(const Plan &pl, const float *poses, const float *tmpl, const float *p0, float *out,
                                 int mode, const float *meas, const uint8_t *mask, double *rowloss, cudaStream_t st);
pa_status launch_adjoint_generic(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses,
                                 const float *tmpl, const float *p0, const float *cot, float *grad_p0, float *partial,
                                 AdjLaunch &L, bool dry, cudaStream_t st);
// family-specific direct launchers (k_direct_<family>.cu)
pa_status launch_forward_direct_gauss(const Plan &, const float *, const float *, const float *, float *, int,
                                      const float *, const uint8_t *, double *, cudaStream_t);
pa_status launch_forward_direct_exp(const Plan &, const float *, const float *, const float *, float *, int,
                                    const float *, const uint8_t *, double *, cudaStream_t);
pa_status launch_forward_direct_pow(const Plan &, const float *, const float *, const float *, float *, int,
                                    const float *, const uint8_t *, double *, cudaStream_t);
pa_status launch_adjoint_direct_gauss(pa_ctx *, const Plan &, bool, bool, const float *, const float *,
                                      const float *, const float *, float *, float *, AdjLaunch &, bool, cudaStream_t);
pa_status launch_adjoint_direct_exp(pa_ctx *, const Plan &, bool, bool, const float *, const float *, const float *,
                                    const float *, float *, float *, AdjLaunch &, bool, cudaStream_t);
pa_status launch_adjoint_direct_pow(pa_ctx *, const Plan &, bool, bool, const float *, const float *, const float *,
                                    const float *, float *, float *, AdjLaunch &, bool, cudaStream_t);

}  // namespace pa
