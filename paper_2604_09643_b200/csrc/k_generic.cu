// k_generic.cu — the generic kernels K1g / K2g / K3g: forward, adjoint and element gradient of Eq.
// gpu_forward_model for ANY window length and any kernel family (R23, R26), for the geometries no
// other kernel holds (exponential / power-law windows longer than the direct kernels' register windows,
// Gaussian windows beyond PA_LMAX, short windows with a large cluster spread).  Plain and slow: every term is
// evaluated directly, the geometry in fp64 and the window by the literal predicate |r - c (t0 + j dt)| <=
// kappa sigma (the definition itself, R4), so no window class, recurrence or factorisation is involved.
// Deterministic (fixed summation orders, no atomics):
//   K1g  one CTA per (frame, element) row, one warp per voxel at a time, the warp's lanes splitting the
//        voxel's window samples (distinct samples: plain adds into the warp's private trace in shared
//        memory); warp traces summed in fixed order, then the row epilogue (trace / MSE / NC, a3);
//   K2g  one thread per voxel, every (frame, element) row and window sample in order;
//   K3g  one CTA per row, one warp per voxel, lanes over samples: sum_j g d/dr[D K(D)/(2r)] reduced by a
//        fixed shuffle tree, G[f,e] += p0 (x - y)/r per warp, warps summed in order -> pose partial (P = 1).
// DESIGN.md §6 (K1g/K2g/K3g) and R23 for K'(D).
#include "pa_plan.h"

namespace pa {

namespace {

struct GenConst {
    double c, t0, dt, kc;  // sound speed, time origin, sampling interval (fp64 of the fp32 inputs), kappa sigma
    double sig;            // sigma (the family's scale s)
    double nu;             // power-law exponent
};

// K(D) and (K + D K')/K of family FAM (R23): Gaussian e^{-D^2/2s^2}; exponential e^{-|D|/s}; power law
// (D^2 + s^2)^{-nu}
template <int FAM>
__device__ __forceinline__ void gen_k(const GenConst &q, double D, float &K, float &dfac)
{
    const float d = (float)D, s = (float)q.sig;
    if constexpr (FAM == KF_GAUSS) {
        const float u = d / s;
        K = expf(-0.5f * u * u);
        dfac = 1.0f - u * u;
    } else if constexpr (FAM == KF_EXP) {
        const float u = fabsf(d) / s;
        K = expf(-u);
        dfac = 1.0f - u;
    } else {
        const float w = d * d + s * s;
        K = powf(w, -(float)q.nu);
        dfac = 1.0f - 2.0f * (float)q.nu * d * d / w;
    }
}

// window [jlo, jhi] of distance r: solved, then corrected against the literal predicate; false if empty
__device__ __forceinline__ bool gen_window(const Geo &g, const GenConst &q, double r, int &jlo, int &jhi)
{
    auto in = [&](int j) { return fabs(r - q.c * (q.t0 + (double)j * q.dt)) <= q.kc; };
    const double cdt = q.c * q.dt;
    double lo = ceil((r - q.kc - q.c * q.t0) / cdt), hi = floor((r + q.kc - q.c * q.t0) / cdt);
    lo = lo < 0.0 ? 0.0 : lo;
    hi = hi > (double)(g.nt - 1) ? (double)(g.nt - 1) : hi;
    if (lo > hi + 1.0) return false;
    jlo = (int)lo;
    jhi = (int)hi;
    while (jlo > 0 && in(jlo - 1)) --jlo;
    while (jlo <= jhi && !in(jlo)) ++jlo;
    while (jhi < g.nt - 1 && in(jhi + 1)) ++jhi;
    while (jhi >= jlo && !in(jhi)) --jhi;
    return jlo <= jhi;
}

__device__ __forceinline__ void voxel_centre(const Geo &g, long long v, double y[3])
{
    const long long sxy = (long long)g.nx * g.ny;
    const int l = (int)(v / sxy), rem = (int)(v - (long long)l * sxy);
    const int j = rem / g.nx, i = rem - j * g.nx;
    y[0] = g.ox + g.h * i;
    y[1] = g.oy + g.h * j;
    y[2] = g.oz + g.h * l;
}

template <int FAM>
__global__ void __launch_bounds__(256) k_fwd_gen(Geo g, GenConst q, const float *__restrict__ poses,
                                                 const float *__restrict__ tmpl, const float *__restrict__ p0,
                                                 float *__restrict__ out, int mode, const float *__restrict__ meas,
                                                 const uint8_t *__restrict__ row_mask, double *__restrict__ rowloss)
{
    extern __shared__ float tr[];  // [nw][nt] warp-private traces
    __shared__ double red[256];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nt = g.nt;
    for (int i = threadIdx.x; i < nw * nt; i += blockDim.x) tr[i] = 0.0f;
    __syncthreads();
    const int fe = blockIdx.x, f = fe / g.E, e = fe - f * g.E;
    double x[3];
    elem_pos(poses, tmpl, f, e, x);
    const long long nv = (long long)g.nx * g.ny * g.nz;
    float *mine = tr + warp * nt;
    for (long long v = warp; v < nv; v += nw) {
        const float P = __ldg(p0 + v);
        if (P == 0.0f) continue;  // warp-uniform: a zero amplitude adds nothing
        double y[3];
        voxel_centre(g, v, y);
        const double r = sqrt((x[0] - y[0]) * (x[0] - y[0]) + (x[1] - y[1]) * (x[1] - y[1]) + (x[2] - y[2]) * (x[2] - y[2]));
        int jlo, jhi;
        if (!gen_window(g, q, r, jlo, jhi)) continue;
        const float cf = (float)(0.5 / r) * P;
        for (int j = jlo + lane; j <= jhi; j += 32) {  // one lane per sample: no two lanes on a sample
            const double D = r - q.c * (q.t0 + (double)j * q.dt);
            float K, df;
            gen_k<FAM>(q, D, K, df);
            mine[j] = __fmaf_rn(cf * (float)D, K, mine[j]);
        }
        __syncwarp();
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        float s = tr[j];
        for (int w = 1; w < nw; ++w) s += tr[w * nt + j];  // fixed order
        tr[j] = s;
    }
    __syncthreads();
    fwd_epilogue(g, tr, fe, out, mode, meas, row_mask, rowloss, red);
}

template <int FAM>
__global__ void __launch_bounds__(256) k_adj_gen(Geo g, GenConst q, const float *__restrict__ poses,
                                                 const float *__restrict__ tmpl, const float *__restrict__ cot,
                                                 float *__restrict__ grad_p0)
{
    const long long nv = (long long)g.nx * g.ny * g.nz;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (long long)gridDim.x * blockDim.x) {
        double y[3];
        voxel_centre(g, v, y);
        float z = 0.0f;
        for (int f = 0; f < g.F; ++f)
            for (int e = 0; e < g.E; ++e) {
                double x[3];
                elem_pos(poses, tmpl, f, e, x);
                const double r = sqrt((x[0] - y[0]) * (x[0] - y[0]) + (x[1] - y[1]) * (x[1] - y[1]) +
                                      (x[2] - y[2]) * (x[2] - y[2]));
                int jlo, jhi;
                if (!gen_window(g, q, r, jlo, jhi)) continue;
                const float *gr = cot + ((size_t)f * g.E + e) * g.nt;
                const float cf = (float)(0.5 / r);
                float s = 0.0f;
                for (int j = jlo; j <= jhi; ++j) {
                    const double D = r - q.c * (q.t0 + (double)j * q.dt);
                    float K, df;
                    gen_k<FAM>(q, D, K, df);
                    s = __fmaf_rn(__ldg(gr + j) * (float)D, K, s);
                }
                z = __fmaf_rn(cf, s, z);
            }
        grad_p0[v] = z;
    }
}

template <int FAM>
__global__ void __launch_bounds__(256) k_pose_gen(Geo g, GenConst q, const float *__restrict__ poses,
                                                  const float *__restrict__ tmpl, const float *__restrict__ p0,
                                                  const float *__restrict__ cot, float *__restrict__ partial)
{
    __shared__ float wg[8][3];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fe = blockIdx.x, f = fe / g.E, e = fe - f * g.E;
    double x[3];
    elem_pos(poses, tmpl, f, e, x);
    const float *gr = cot + (size_t)fe * g.nt;
    const long long nv = (long long)g.nx * g.ny * g.nz;
    float G0 = 0.f, G1 = 0.f, G2 = 0.f;
    for (long long v = warp; v < nv; v += nw) {
        const float P = __ldg(p0 + v);
        if (P == 0.0f) continue;
        double y[3];
        voxel_centre(g, v, y);
        const double d0 = x[0] - y[0], d1 = x[1] - y[1], d2 = x[2] - y[2];
        const double r = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        int jlo, jhi;
        if (!gen_window(g, q, r, jlo, jhi)) continue;
        // d/dr [D K(D)/(2r)] = K (1 + D K'/K)/(2r) - D K/(2 r^2)   (the window indicator held constant, R11)
        const float ir = (float)(1.0 / r);
        float s = 0.0f;
        for (int j = jlo + lane; j <= jhi; j += 32) {
            const double D = r - q.c * (q.t0 + (double)j * q.dt);
            float K, df;
            gen_k<FAM>(q, D, K, df);
            s = __fmaf_rn(__ldg(gr + j) * K, __fmaf_rn(-(float)D, ir, df), s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float c = 0.5f * ir * ir * P * s;  // dL/dr x P / r
        G0 = __fmaf_rn(c, (float)d0, G0);
        G1 = __fmaf_rn(c, (float)d1, G1);
        G2 = __fmaf_rn(c, (float)d2, G2);
    }
    if (lane == 0) {
        wg[warp][0] = G0;
        wg[warp][1] = G1;
        wg[warp][2] = G2;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        float s = 0.0f;
        for (int w = 0; w < nw; ++w) s += wg[w][threadIdx.x];  // fixed order
        partial[(size_t)fe * 3 + threadIdx.x] = s;            // pose partials [P = 1][F][E][3]
    }
}

GenConst gen_const(const Plan &pl)
{
    GenConst q;
    q.c = pl.g.c;
    q.t0 = pl.g.t0;
    q.dt = pl.gen_dt;
    q.kc = pl.g.ksig_d;
    q.sig = pl.gen_sig;
    q.nu = pl.g.nu;
    return q;
}

template <int FAM>
pa_status fwd_gen_t(const Plan &pl, const float *poses, const float *tmpl, const float *p0, float *out, int mode,
                    const float *meas, const uint8_t *mask, double *rowloss, cudaStream_t st)
{
    const int nw = pl.gen_nw;
    const size_t smem = (size_t)nw * pl.g.nt * sizeof(float);
    CUDA_TRY(cudaFuncSetAttribute(k_fwd_gen<FAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ++g_nlaunch;
    k_fwd_gen<FAM><<<pl.g.F * pl.g.E, nw * 32, smem, st>>>(pl.g, gen_const(pl), poses, tmpl, p0, out, mode, meas,
                                                          mask, rowloss);
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

template <int FAM>
pa_status adj_gen_t(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses, const float *tmpl,
                    const float *p0, const float *cot, float *grad_p0, float *partial, cudaStream_t st)
{
    const long long nv = (long long)pl.g.nx * pl.g.ny * pl.g.nz;
    if (adj) {
        const long long nb = std::min<long long>((nv + 255) / 256, (long long)ctx_nsm(ctx) * 8);
        ++g_nlaunch;
        k_adj_gen<FAM><<<(unsigned)nb, 256, 0, st>>>(pl.g, gen_const(pl), poses, tmpl, cot, grad_p0);
        CUDA_TRY(cudaGetLastError());
    }
    if (pose) {
        ++g_nlaunch;
        k_pose_gen<FAM><<<pl.g.F * pl.g.E, 256, 0, st>>>(pl.g, gen_const(pl), poses, tmpl, p0, cot, partial);
        CUDA_TRY(cudaGetLastError());
    }
    return PA_OK;
}

}  // namespace

pa_status launch_forward_generic(const Plan &pl, const float *poses, const float *tmpl, const float *p0, float *out,
                                 int mode, const float *meas, const uint8_t *mask, double *rowloss, cudaStream_t st)
{
    switch (pl.fam) {
    case KF_EXP: return fwd_gen_t<KF_EXP>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    case KF_POW: return fwd_gen_t<KF_POW>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    default: return fwd_gen_t<KF_GAUSS>(pl, poses, tmpl, p0, out, mode, meas, mask, rowloss, st);
    }
}

pa_status launch_adjoint_generic(pa_ctx *ctx, const Plan &pl, bool pose, bool adj, const float *poses,
                                 const float *tmpl, const float *p0, const float *cot, float *grad_p0, float *partial,
                                 AdjLaunch &L, bool dry, cudaStream_t st)
{
    L.P = 1;  // K3g writes the summed element gradient of each row: one partial
    L.Fc = pl.g.F;
    L.smem = 0;
    if (dry || pl.g.F == 0) return PA_OK;
    switch (pl.fam) {
    case KF_EXP: return adj_gen_t<KF_EXP>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, st);
    case KF_POW: return adj_gen_t<KF_POW>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, st);
    default: return adj_gen_t<KF_GAUSS>(ctx, pl, pose, adj, poses, tmpl, p0, cot, grad_p0, partial, st);
    }
}

}  // namespace pa
