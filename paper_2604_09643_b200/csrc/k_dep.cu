// k_dep.cu — launcher of the deposit-form forward K1d (a2 + fused a3, Gaussian; pa_kernels.cuh).
#include "pa_plan.h"

namespace pa {

namespace {
template <int R, int NW, int NG, int TPR>
pa_status launch_dep_t(pa_ctx *ctx, const Plan &pl, const float *poses, const float *tmpl, const float *p0, float *out,
                       int mode, const float *meas, const uint8_t *mask, double *rowloss, cudaStream_t st)
{
    const size_t smem = DepCfg<R, NW, NG, TPR>::smem_bytes(pl.g.nt, pl.g.lmin, pl.dc.nr);
    auto kern = k_fwd_dep<R, NW, NG, TPR>;
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    unsigned *pm = ctx_pmax(ctx);
    CUDA_TRY(cudaMemsetAsync(pm, 0, sizeof(unsigned), st));
    const long long nvox = (long long)pl.g.nx * pl.g.ny * pl.g.nz;
    ++g_nlaunch;
    k_absmax<<<ctx_nsm(ctx) * 4, 256, 0, st>>>(p0, nvox, pm);  // |p0| max: the fixed-point normalisation
    CUDA_TRY(cudaGetLastError());
    ++g_nlaunch;
    kern<<<pl.g.F * pl.g.E, NW * 32, smem, st>>>(pl.g, pl.dc, poses, tmpl, p0, pm, out, mode, meas, mask, rowloss);
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

template <int R, int TPR>
pa_status launch_dep_rt(pa_ctx *ctx, const Plan &pl, const float *poses, const float *tmpl, const float *p0, float *out,
                        int mode, const float *meas, const uint8_t *mask, double *rowloss, cudaStream_t st)
{
    if (pl.dep_g == 2) {
        if (pl.dep_nw == 8) return launch_dep_t<R, 8, 2, TPR>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
        return launch_dep_t<R, 16, 2, TPR>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    }
    if (pl.dep_nw == 8) return launch_dep_t<R, 8, 1, TPR>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    return launch_dep_t<R, 16, 1, TPR>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
}

template <int R>
pa_status launch_dep_r(pa_ctx *ctx, const Plan &pl, const float *poses, const float *tmpl, const float *p0, float *out,
                       int mode, const float *meas, const uint8_t *mask, double *rowloss, cudaStream_t st)
{
    if (pl.dep_tpr == 8) return launch_dep_rt<R, 8>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    return launch_dep_rt<R, 4>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
}
}  // namespace

pa_status launch_forward_dep(pa_ctx *ctx, const Plan &pl, const float *poses, const float *tmpl, const float *p0,
                             float *out, int mode, const float *meas, const uint8_t *mask, double *rowloss,
                             cudaStream_t st)
{
    if (pl.dep_R == 7) return launch_dep_r<7>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    if (pl.dep_R == 6) return launch_dep_r<6>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    if (pl.dep_R == 5) return launch_dep_r<5>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    return launch_dep_r<4>(ctx, pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
}

}  // namespace pa
