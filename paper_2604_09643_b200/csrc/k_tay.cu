// k_tay.cu — launcher of the moment-filter adjoint K2a (filters) + K2c (adjoint + element gradient), Gaussian
// (a4 + a5; pa_kernels.cuh).  Per frame chunk sized so that the chunk's filters stay in L2.
#include "pa_plan.h"

#include <algorithm>

namespace pa {

namespace {
template <int NF, bool POSE, bool ADJ>
pa_status launch_tay_t(pa_ctx *ctx, const Plan &pl, const float *poses, const float *tmpl, const float *p0,
                       const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry, cudaStream_t st)
{
    using T = TayCfg<NF>;
    const int E = pl.g.E, F = pl.g.F, E4 = (E + 3) & ~3;
    const int njp = pl.g.nt + pl.g.lmin + 2 * pl.tay_pad;  // zero-padded record row
    const size_t per_frame = (size_t)E * njp * T::NF * sizeof(float);
    int Fc = (int)std::max<size_t>(1, std::min<size_t>(64, (size_t(48) << 20) / per_frame));
    auto smem_of = [&](int fc) {
        return (size_t)PA_ADJ_TPC * E4 * sizeof(AncT) +
               ((size_t)(TAY_NT / 32) * E * 3 + (POSE ? (size_t)fc * E * 3 : 0)) * sizeof(float);
    };
    while (Fc > 1 && smem_of(Fc) > (size_t)(228 / PA_ADJ_MINB - 1) * 1024) --Fc;  // keep PA_ADJ_MINB CTAs per SM
    Fc = std::min(Fc, std::max(1, 65535 / E));  // K2a grid.y = Fc E
    Fc = std::min(Fc, F > 0 ? F : 1);
    const size_t smem = smem_of(Fc);
    if (smem > 227 * 1024) return fail(PA_EUNSUPPORTED, "E=%d too large for the adjoint kernel's shared memory", E);
    auto kern = k_adjoint_tay2<NF, POSE, ADJ>;
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TAY_NT, smem));
    if (occ < 1) occ = 1;
    int P = occ * ctx_nsm(ctx);
    const int nwork = pl.g.ntx * pl.g.nty * (PA_ADJ_TPC == 2 ? (pl.g.ntz + 1) / 2 : pl.g.ntz);  // tile pairs / tiles
    if (P > nwork) P = nwork;
    L.P = P;
    L.Fc = Fc;
    L.smem = smem;
    if (dry) return PA_OK;
    float *Fg = nullptr;
    pa_status s;
    if ((s = ctx_filter_ws(ctx, (size_t)Fc * per_frame, &Fg))) return s;
    for (int f0 = 0; f0 < F; f0 += Fc) {
        const int fn = std::min(Fc, F - f0);
        ++g_nlaunch;
        k_adj_filter<NF><<<dim3((njp + 255) / 256, fn * E), 256, 0, st>>>(pl.g, pl.tf, cot, f0, fn, njp, Fg);
        CUDA_TRY(cudaGetLastError());
        ++g_nlaunch;
        kern<<<P, TAY_NT, smem, st>>>(pl.g, pl.tc, poses, tmpl, p0, Fg, grad_p0, partial, f0, fn, njp,
                                           pl.tay_pad, pl.tay_sentinel);
        CUDA_TRY(cudaGetLastError());
    }
    return PA_OK;
}

template <int NF>
pa_status launch_tay_m(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses, const float *tmpl,
                       const float *p0, const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry,
                       cudaStream_t st)
{
    if (pose && adj) return launch_tay_t<NF, true, true>(ctx, pl, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    if (pose) return launch_tay_t<NF, true, false>(ctx, pl, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    return launch_tay_t<NF, false, true>(ctx, pl, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
}
}  // namespace

pa_status launch_adjoint_tay(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses, const float *tmpl,
                             const float *p0, const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry,
                             cudaStream_t st)
{
    if (pl.tay_NF == 8) return launch_tay_m<8>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    if (pl.tay_NF == 12) return launch_tay_m<12>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    return fail(PA_EUNSUPPORTED, "no moment-filter adjoint for record size %d", pl.tay_NF);
}

}  // namespace pa
