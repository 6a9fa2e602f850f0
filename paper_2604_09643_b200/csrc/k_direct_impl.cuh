// k_direct_impl.cuh — launchers of the direct kernels K1 (forward) and K2 (adjoint + element gradient) for one
// kernel family FAM; included once per family by k_direct_<family>.cu (parallel compilation).
#pragma once
#include "pa_plan.h"

#include <algorithm>

namespace pa {
namespace direct {

template <int LMIN, int OMAX, int SPAN, int FAM, int RC = LMIN + OMAX>
pa_status fwd_t(const Plan &pl, const float *poses, const float *tmpl, const float *p0, float *out, int mode,
                const float *meas, const uint8_t *mask, double *rowloss, cudaStream_t st)
{
    using C = FwdCfg<LMIN, OMAX, SPAN, RC>;
    const size_t smem = (size_t)FWD_WARPS * C::warp_floats(pl.g.nt) * sizeof(float);
    if (smem > 227 * 1024) return fail(PA_EUNSUPPORTED, "nt=%d too long for the forward kernel's shared memory", pl.g.nt);
    auto kern = k_forward<LMIN, OMAX, SPAN, FAM, RC>;
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ++g_nlaunch;
    kern<<<pl.g.F * pl.g.E, FWD_WARPS * 32, smem, st>>>(pl.g, pl.fc, poses, tmpl, p0, out, mode, meas, mask, rowloss);
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

template <int FAM>
pa_status forward(const Plan &pl, const float *poses, const float *tmpl, const float *p0, float *out, int mode,
                  const float *meas, const uint8_t *mask, double *rowloss, cudaStream_t st)
{
    switch (pl.klass) {
    case 0: return fwd_t<53, 11, 58, FAM>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    case 1: return fwd_t<26, 6, 30, FAM>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    case 2: return fwd_t<106, 21, 114, FAM>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    // runtime classes (L_min, OMAX, centre from the plan; register-window capacity RC, tile span SPAN)
    case KLASS_RT + 0: return fwd_t<0, 0, kRtClasses[0].span, FAM, kRtClasses[0].rc>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    case KLASS_RT + 1: return fwd_t<0, 0, kRtClasses[1].span, FAM, kRtClasses[1].rc>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    case KLASS_RT + 2: return fwd_t<0, 0, kRtClasses[2].span, FAM, kRtClasses[2].rc>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    default: return fail(PA_EUNSUPPORTED, "no direct forward kernel class for this geometry");
    }
}

template <int LMIN, int SEG, bool POSE, bool ADJ, int FAM>
pa_status adj_t(pa_ctx *ctx, const Plan &pl, const float *poses, const float *tmpl, const float *p0, const float *cot,
                float *grad_p0, float *partial, AdjLaunch &L, bool dry, cudaStream_t st)
{
    auto kern = k_adjoint<LMIN, SEG, POSE, ADJ, FAM>;
    const int E = pl.g.E, F = pl.g.F;
    const int SEGr = SEG > 0 ? SEG : pl.g.seg;  // runtime class: the plan's segment length
    int Fc = POSE ? 64 : F;
    size_t smem = AdjCfg::smem_floats(E, SEGr, Fc, POSE) * sizeof(float);
    // prefer 2 CTAs/SM with a frame chunk >= 8, else the largest chunk that fits one CTA/SM
    const size_t two = 113 * 1024, one = 227 * 1024;
    if (POSE) {
        Fc = 64;
        while (Fc > 8 && AdjCfg::smem_floats(E, SEGr, Fc, POSE) * sizeof(float) > two) Fc -= 4;
        if (AdjCfg::smem_floats(E, SEGr, Fc, POSE) * sizeof(float) > two) {
            Fc = 64;
            while (Fc > 1 && AdjCfg::smem_floats(E, SEGr, Fc, POSE) * sizeof(float) > one) Fc -= 1;
        }
        Fc = Fc < F ? Fc : (F > 0 ? F : 1);
        smem = AdjCfg::smem_floats(E, SEGr, Fc, POSE) * sizeof(float);
    }
    if (smem > one) return fail(PA_EUNSUPPORTED, "E=%d too large for the adjoint kernel's shared memory", E);
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, ADJ_THREADS, smem));
    if (occ < 1) occ = 1;
    int P = occ * ctx_nsm(ctx);
    if (P > pl.g.ntiles) P = pl.g.ntiles;
    L.P = P;
    L.Fc = Fc;
    L.smem = smem;
    if (dry) return PA_OK;
    ++g_nlaunch;
    kern<<<P, ADJ_THREADS, smem, st>>>(pl.g, pl.ac, poses, tmpl, p0, cot, grad_p0, partial, Fc);
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

template <int LMIN, int SEG, int FAM>
pa_status adj_c(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses, const float *tmpl,
                const float *p0, const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry,
                cudaStream_t st)
{
    if (pose && adj) return adj_t<LMIN, SEG, true, true, FAM>(ctx, pl, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    if (pose) return adj_t<LMIN, SEG, true, false, FAM>(ctx, pl, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    return adj_t<LMIN, SEG, false, true, FAM>(ctx, pl, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
}

template <int FAM>
pa_status adjoint(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses, const float *tmpl,
                  const float *p0, const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry,
                  cudaStream_t st)
{
    switch (pl.klass) {
    case 0: return adj_c<53, 128, FAM>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    case 1: return adj_c<26, 64, FAM>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    case 2: return adj_c<106, 256, FAM>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    case KLASS_RT + 0:
    case KLASS_RT + 1:
    case KLASS_RT + 2: return adj_c<0, 0, FAM>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    default: return fail(PA_EUNSUPPORTED, "no direct adjoint kernel class for this geometry");
    }
}

}  // namespace direct
}  // namespace pa

#define PA_DIRECT_FAMILY(NAME, FAM)                                                                                   \
    namespace pa {                                                                                                    \
    pa_status launch_forward_direct_##NAME(const Plan &pl, const float *poses, const float *tmpl, const float *p0,    \
                                           float *out, int mode, const float *meas, const uint8_t *mask,              \
                                           double *rowloss, cudaStream_t st)                                          \
    {                                                                                                                 \
        return direct::forward<FAM>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);                         \
    }                                                                                                                 \
    pa_status launch_adjoint_direct_##NAME(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses,      \
                                           const float *tmpl, const float *p0, const float *cot, float *grad_p0,      \
                                           float *partial, AdjLaunch &L, bool dry, cudaStream_t st)                   \
    {                                                                                                                 \
        return direct::adjoint<FAM>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);          \
    }                                                                                                                 \
    }
