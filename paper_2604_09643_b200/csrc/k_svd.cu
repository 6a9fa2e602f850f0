// k_svd.cu — launcher of the adjoint in the forward's rank-R basis, K2s-a (filter records) + K2s (adjoint +
// element gradient), Gaussian (a4 + a5; pa_kernels.cuh).
#include "pa_plan.h"

#include <algorithm>

namespace pa {

namespace {
template <int R, bool POSE, bool ADJ>
pa_status launch_svd_t(pa_ctx *ctx, const Plan &pl, const float *poses, const float *tmpl, const float *p0,
                       const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry, cudaStream_t st)
{
    const int E = pl.g.E, F = pl.g.F, NJ = pl.g.nt + pl.g.lmin;
    const size_t per_frame = (size_t)E * NJ * SVD_NF * sizeof(float);
    int Fc = (int)std::max<size_t>(1, std::min<size_t>(64, (size_t(48) << 20) / per_frame));
    auto smem_of = [&](int fc) {
        return ((size_t)E * 12 * 2 + (size_t)(ADJ_THREADS / 32) * E * 3 + (POSE ? (size_t)fc * E * 3 : 0)) * sizeof(float);
    };
    while (Fc > 1 && smem_of(Fc) > 113 * 1024) --Fc;
    Fc = std::min(Fc, std::max(1, 65535 / E));  // filter grid.y = Fc E
    Fc = std::min(Fc, F > 0 ? F : 1);
    const size_t smem = smem_of(Fc);
    if (smem > 227 * 1024) return fail(PA_EUNSUPPORTED, "E=%d too large for the adjoint kernel's shared memory", E);
    auto kern = k_adjoint_svd<R, POSE, ADJ>;
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, ADJ_THREADS, smem));
    if (occ < 1) occ = 1;
    int P = occ * ctx_nsm(ctx);
    const int nwork = pl.g.ntx * pl.g.nty * ((pl.g.ntz + 1) / 2);  // tile pairs
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
        k_adj_svd_filter<R><<<dim3((NJ + 255) / 256, fn * E), 256, 0, st>>>(pl.g, pl.sv, cot, f0, fn, Fg);
        CUDA_TRY(cudaGetLastError());
        ++g_nlaunch;
        kern<<<P, ADJ_THREADS, smem, st>>>(pl.g, pl.sv, poses, tmpl, p0, Fg, grad_p0, partial, f0, fn);
        CUDA_TRY(cudaGetLastError());
    }
    return PA_OK;
}

template <int R>
pa_status launch_svd_r(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses, const float *tmpl,
                       const float *p0, const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry,
                       cudaStream_t st)
{
    if (pose && adj) return launch_svd_t<R, true, true>(ctx, pl, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    if (pose) return launch_svd_t<R, true, false>(ctx, pl, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    return launch_svd_t<R, false, true>(ctx, pl, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
}
}  // namespace

pa_status launch_adjoint_svd(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses, const float *tmpl,
                             const float *p0, const float *cot, float *grad_p0, float *partial, AdjLaunch &L, bool dry,
                             cudaStream_t st)
{
    if (pl.dep_R == 7) return launch_svd_r<7>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    if (pl.dep_R == 6) return launch_svd_r<6>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
    return launch_svd_r<5>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, L, dry, st);
}

}  // namespace pa
