// pa_kernels.cuh — device code of libpa (PA-SFM acoustic radiation operator, sm_100a).
//
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, R<k> = DESIGN.md §3 reading,
// K<k> = kernel id of DESIGN.md §6.  This file shares no code with oracle/.
//
// Geometry of the arithmetic (DESIGN.md §6 "precision"):
//   * voxels are processed in 8x8x4 tiles; per (tile, element) an fp64 anchor
//     rho = |y_c - x| (tile centre y_c) and D_A = rho - c t0 = J_A a + C_A (|C_A| <= a/2)
//     are formed once; per voxel, r - rho = (2 d.delta + |delta|^2)/(r + rho) is evaluated in
//     fp32 on small numbers, so D = r - c t_j = (r - rho) + C_A - (j - J_A) a keeps ~1e-7 mm.
//   * exp(-D^2/2s^2) along a window is a two-term recurrence E_{i+1} = E_i * q0 * B^i with
//     B^i = exp(-i a^2/s^2) precomputed in fp64 on the host (kernel parameter), so errors do
//     not compound in q.
//   * the window [jlo, jlo+L) of every (voxel, element) pair is produced by ONE function
//     (pair()) used by both the forward and the adjoint, so the GPU forward and adjoint are
//     exact transposes of each other up to fp32 rounding (R17).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace pa {

constexpr int TX = 8, TY = 8, TZ = 4;  // voxel tile (anchor unit) — 256 voxels
#ifndef PA_FWD_PHASES
#define PA_FWD_PHASES 2
#endif
#ifndef PA_FWD_NV
#define PA_FWD_NV 4
#endif
#ifndef PA_ADJ_HORNER
#define PA_ADJ_HORNER 1  // adjoint moments by Horner (1) or by the explicit recurrence (0)
#endif
constexpr int FWD_WARPS = 4;           // warps per forward CTA
constexpr int ADJ_THREADS = 256;       // one thread per tile voxel

struct Geo {
    int nx, ny, nz, nt;
    int ntx, nty, ntz, ntiles;
    int E, F;
    double ox, oy, oz, h;       // grid (fp64 copies of the fp32 inputs)
    double c, t0, a_d, inv_a_d, ksig_d;  // a_d = c*dt in fp64
    double rt_d;                // tile half-diagonal (mm)
    float hf, af, inv_a, ksig;  // fp32 working constants
    float k2, two_a_k2, a2_k2;  // log2(e)/(2 s^2), 2a*k2, a^2*k2
    float s2, inv_s2, rt;
    int mF, mA;                 // recurrence centres (forward cluster window / adjoint pair window)
    int lmin;                   // L_min = floor(2 kappa sigma / (c dt)): window length (L in {lmin, lmin+1})
    unsigned njp_m1;            // K2c: last record index of a zero-padded filter row
    int omax, seg;              // direct kernels of a runtime class: cluster window-base spread, segment length
    float ls, nu;               // exponential: log2(e)/s; power law: nu   (kernel families, R23)
};

// Kernel families of the designated kernel K(D) (R23): template parameter FAM.
enum { KF_GAUSS = 0, KF_EXP = 1, KF_POW = 2 };

// Step-index constants of the factored Gaussian (DESIGN.md §6 "recurrence"):
//   exp(-D_i^2/2s^2) = u_i * C_i,  D_i = D_m - (i - m) a,  C_i = exp(-(i-m)^2 a^2 / 2s^2),
//   u_i = u_0 p^i,  p = exp(a D_m / s^2),  u_0 = exp(-(D_m^2 + 2 m a D_m) / 2s^2).
// Exponential family: exp(-|D_i|/s) = min(A K_i, B / K_i) with K_i = exp((i - m) a / s),
// A = exp(-D_m/s), B = exp(D_m/s) (one of the two is the value, the other its reciprocal).
struct FwdConst {
    float2 C2[64];   // Gaussian: (C_2k, C_2k+1) about the cluster-window centre mF; exp: (K_2k, K_2k+1)
    float2 I2[64];   // (-2k, -2k-1): step indices for packed D_i = D_J - i a
    float2 X2[64];   // exp: (1/K_2k, 1/K_2k+1)
};
constexpr int ADJ_LCAP = 160;  // longest window (L_min + 1) of the direct adjoint K2
struct AdjConst {
    float C0[ADJ_LCAP];  // Gaussian: C_i about the pair-window centre mA;  exp: K_i
    float C1[ADJ_LCAP];  // Gaussian: C_i (i - mA);                           exp: 1/K_i
    float C2[ADJ_LCAP];  // Gaussian: C_i (i - mA)^2
};

struct Anc {
    float dx2, dy2, dz2;  // 2 * (y_c - x)  (fp32)
    float dx, dy, dz;     // y_c - x
    float rho, rho2, CA;
    int JA;
    int cull;
};

__device__ __forceinline__ float ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float lg2(float x)
{
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// exp(x) for |x| <= 0.5 to ~1 ulp (degree-8 Taylor): the per-voxel ratio p of the recurrence,
// whose rounding would otherwise compound over the window.
__device__ __forceinline__ float exp_small(float x)
{
    float r = __fmaf_rn(x, 1.0f / 8.0f, 1.0f);
    r = __fmaf_rn(x * (1.0f / 7.0f), r, 1.0f);
    r = __fmaf_rn(x * (1.0f / 6.0f), r, 1.0f);
    r = __fmaf_rn(x * (1.0f / 5.0f), r, 1.0f);
    r = __fmaf_rn(x * (1.0f / 4.0f), r, 1.0f);
    r = __fmaf_rn(x * (1.0f / 3.0f), r, 1.0f);
    r = __fmaf_rn(x * 0.5f, r, 1.0f);
    return __fmaf_rn(x, r, 1.0f);
}

__device__ __forceinline__ void elem_pos(const float *__restrict__ poses, const float *__restrict__ tmpl, int f, int e,
                                         double x[3])
{
    const float *P = poses + 12 * f;
    const float *xh = tmpl + 3 * e;
    double x0 = xh[0], x1 = xh[1], x2 = xh[2];
#pragma unroll
    for (int a = 0; a < 3; ++a)
        x[a] = (double)P[3 * a] * x0 + (double)P[3 * a + 1] * x1 + (double)P[3 * a + 2] * x2 + (double)P[9 + a];
}

// Per (tile, element) fp64 anchor (K1/K2 prologue).
__device__ __forceinline__ Anc make_anchor(const Geo &g, const double x[3], int tx, int ty, int tz)
{
    double cx = g.ox + g.h * (TX * tx + 0.5 * (TX - 1));
    double cy = g.oy + g.h * (TY * ty + 0.5 * (TY - 1));
    double cz = g.oz + g.h * (TZ * tz + 0.5 * (TZ - 1));
    double dx = cx - x[0], dy = cy - x[1], dz = cz - x[2];
    double rho = sqrt(dx * dx + dy * dy + dz * dz);
    double D = rho - g.c * g.t0;
    double JA = rint(D * g.inv_a_d);
    double CA = D - JA * g.a_d;
    Anc A;
    A.dx = (float)dx;
    A.dy = (float)dy;
    A.dz = (float)dz;
    A.dx2 = 2.0f * A.dx;
    A.dy2 = 2.0f * A.dy;
    A.dz2 = 2.0f * A.dz;
    A.rho = (float)rho;
    A.rho2 = (float)(rho * rho);
    A.CA = (float)CA;
    A.JA = (int)JA;
    double m = g.rt_d + g.ksig_d + 3.0 * g.a_d;
    A.cull = (D - m > (double)(g.nt - 1) * g.a_d) || (D + m < 0.0);
    return A;
}

struct Pair {
    float drel;   // r - rho
    float inv_r;  // 1/r
    int jlo;      // first in-window sample (unclipped)
    int L;        // window length, clamped to [LMIN, LMIN+1]
};

// The single definition of a (voxel, element) pair's window used by every kernel (R17); LMIN is the
// window length L_min (a compile-time constant in the compiled classes, folded by the compiler).
__device__ __forceinline__ Pair pair(const Geo &g, const Anc &A, float ex, float ey, float ez, float e2, int LMIN)
{
    float num = __fmaf_rn(A.dx2, ex, __fmaf_rn(A.dy2, ey, __fmaf_rn(A.dz2, ez, e2)));
    float r2 = __fadd_rn(A.rho2, num);
    float inv_r = rsqrtf(r2);
    float r = __fmul_rn(r2, inv_r);
    float drel = __fdividef(num, __fadd_rn(r, A.rho));
    float base = __fadd_rn(drel, A.CA);
    float xlo = __fmul_rn(__fsub_rn(base, g.ksig), g.inv_a);
    float xhi = __fmul_rn(__fadd_rn(base, g.ksig), g.inv_a);
    int clo = (int)ceilf(xlo);
    int L = (int)floorf(xhi) - clo + 1;
    L = L < LMIN ? LMIN : (L > LMIN + 1 ? LMIN + 1 : L);
    Pair p;
    p.drel = drel;
    p.inv_r = inv_r;
    p.jlo = A.JA + clo;
    p.L = L;
    return p;
}

__device__ __forceinline__ float warp_sum(float v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int warp_min(int v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// Fixed-order block reduction (blockDim a power of two); red has blockDim entries.
__device__ __forceinline__ double block_sum(double v, double *red)
{
    __syncthreads();
    red[threadIdx.x] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}
__device__ __forceinline__ int warp_max(int v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ============================================================================================
// K1 — forward radiation (a2, Eq. gpu_forward_model), element-stationary.
//
// CTA = one (frame f, element e) row of the output; 4 warps stride over the 8x8x4 voxel
// tiles.  In a tile, lane l owns a 2x2x2 voxel cluster and a register window acc[0..R) of
// samples [J_l, J_l+R), R = LMIN+OMAX, J_l = min jlo over the cluster (jlo spread < OMAX by
// geometry).  Each voxel adds its L in-window terms by the exp recurrence with static
// register indices (only the first OMAX-1 and last OMAX steps are predicated).  The 32
// windows are then summed through shared memory into a warp-private trace (no atomics),
// and the 4 warp traces are summed in fixed order at the end.  Epilogue optionally fuses
// the MSE / NC cotangent (a3) so the trace is never written.
// ============================================================================================
// LMIN = 0: a runtime class — L_min, OMAX and the centre step come from Geo (lmin, omax, mF) and RC is
// the register-window capacity (>= L_min + OMAX); the loops below are written over the whole capacity
// with bounds tests that fold away for the compiled classes.
template <int LMIN, int OMAX, int SPAN, int RC = LMIN + OMAX>
struct FwdCfg {
    static constexpr int R = RC;
    static constexpr int NCOL = R + SPAN;   // columns of the flush buffer (window + tile spread)
    static constexpr int NPH = PA_FWD_PHASES;         // flush phases (rows per phase = 32 / NPH)
    static constexpr int ROWS = 32 / NPH;
    static constexpr int CSTR = ROWS + 4;              // column stride (floats): rows + skew, 16-B aligned
    static constexpr int PADL = (LMIN > 0 ? LMIN : RC) + 2;
    static __host__ __device__ int trace_len(int nt) { return PADL + nt + NCOL + 1; }
    static __host__ __device__ int warp_floats(int nt) { return ((trace_len(nt) + 3) & ~3) + NCOL * CSTR; }
};

enum { FWD_TRACE = 0, FWD_MSE = 1, FWD_NC = 2 };

// K(D) evaluated directly (slow paths)
template <int FAM>
__device__ __forceinline__ float fam_direct(const Geo &g, float D)
{
    if constexpr (FAM == KF_GAUSS) return ex2(-D * D * g.k2);
    else if constexpr (FAM == KF_EXP) return ex2(-fabsf(D) * g.ls);
    else return ex2(-g.nu * lg2(__fmaf_rn(D, D, g.s2)));
}

// Kernel-family values at step i for the generic (non-Gaussian) forward path: packed (i, i+1)
// and scalar.  A, B: exp family per-voxel factors (c folded in); c: amplitude (power law).
template <int FAM>
__device__ __forceinline__ float2 fam_val2(const Geo &g, const FwdConst &fc, int i2, float2 D, float A, float B)
{
    if constexpr (FAM == KF_EXP) {
        const float2 t1 = __fmul2_rn(make_float2(A, A), fc.C2[i2]);
        const float2 t2 = __fmul2_rn(make_float2(B, B), fc.X2[i2]);
        return make_float2(fminf(t1.x, t2.x), fminf(t1.y, t2.y));
    } else {
        const float2 x = __ffma2_rn(D, D, make_float2(g.s2, g.s2));
        return make_float2(A * ex2(-g.nu * lg2(x.x)), A * ex2(-g.nu * lg2(x.y)));
    }
}
template <int FAM>
__device__ __forceinline__ float fam_val1(const Geo &g, const FwdConst &fc, int i, float D, float A, float B)
{
    if constexpr (FAM == KF_EXP) {
        const float K = (i & 1) ? fc.C2[i >> 1].y : fc.C2[i >> 1].x;
        const float Ki = (i & 1) ? fc.X2[i >> 1].y : fc.X2[i >> 1].x;
        return fminf(A * K, B * Ki);
    } else {
        return A * ex2(-g.nu * lg2(__fmaf_rn(D, D, g.s2)));
    }
}

template <int LMIN_, int OMAX_, int SPAN, int FAM, int RC = LMIN_ + OMAX_>
__global__ void __launch_bounds__(FWD_WARPS * 32, (PA_FWD_PHASES == 2 && SPAN <= 64) ? 3 : 2) k_forward(Geo g, FwdConst fc, const float *__restrict__ poses,
                                                            const float *__restrict__ tmpl,
                                                            const float *__restrict__ p0, float *__restrict__ out,
                                                            int mode, const float *__restrict__ meas,
                                                            const uint8_t *__restrict__ row_mask,
                                                            double *__restrict__ rowloss)
{
    using C = FwdCfg<LMIN_, OMAX_, SPAN, RC>;
    constexpr int R = C::R;
    // window length, cluster spread and recurrence centre: compile-time in the compiled classes, from the
    // plan in a runtime class (LMIN_ = 0)
    const int LMIN = LMIN_ > 0 ? LMIN_ : g.lmin;
    const int OMAX = OMAX_ > 0 ? OMAX_ : g.omax;
    const int M = LMIN_ > 0 ? (((LMIN_ + OMAX_) / 2) & ~1) : g.mF;  // centre step (even), host Geo::mF
    const int UPE = M + 2 * ((LMIN - M) / 2);  // upward packed pairs: [M, UPE)
    const int DNE = 2 * (OMAX / 2);            // downward packed pairs: [DNE, M)
    extern __shared__ float sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TL = (C::trace_len(g.nt) + 3) & ~3;
    float *trw = sm + warp * C::warp_floats(g.nt);
    float *cols = trw + TL;  // [NCOL][CSTR]: entry (c, lane) = lane's window value at column c
    for (int i = lane; i < C::warp_floats(g.nt); i += 32) trw[i] = 0.0f;  // trace + rows

    const int fe = blockIdx.x;
    const int f = fe / g.E, e = fe - f * g.E;
    double x[3];
    elem_pos(poses, tmpl, f, e, x);

    const int cx = lane & 3, cy = (lane >> 2) & 3, cz = lane >> 4;
    __syncwarp();

    // tile coordinates advanced incrementally (tile += FWD_WARPS), no integer division
    int tx = warp % g.ntx, ty = (warp / g.ntx) % g.nty, tz = warp / (g.ntx * g.nty);
    for (int tile = warp; tile < g.ntiles; tile += FWD_WARPS) {
        if (tile != warp) {
            tx += FWD_WARPS;
            while (tx >= g.ntx) {
                tx -= g.ntx;
                if (++ty == g.nty) {
                    ty = 0;
                    ++tz;
                }
            }
        }
        const Anc A = make_anchor(g, x, tx, ty, tz);
        if (A.cull) continue;  // warp-uniform

        // cluster geometry: voxel (2cx+vx, 2cy+vy, 2cz+vz) of the tile; offsets from the tile centre
        const int bx = TX * tx + 2 * cx, by = TY * ty + 2 * cy, bz = TZ * tz + 2 * cz;
        const float ex0 = ((float)(2 * cx) - 0.5f * (TX - 1)) * g.hf;
        const float ey0 = ((float)(2 * cy) - 0.5f * (TY - 1)) * g.hf;
        const float ez0 = ((float)(2 * cz) - 0.5f * (TZ - 1)) * g.hf;
        float P[8];
        {
            const float *pb = p0 + ((size_t)bz * g.ny + by) * g.nx + bx;
            const size_t sy = (size_t)g.nx, sz = (size_t)g.nx * g.ny;
            const bool okx1 = bx + 1 < g.nx, oky1 = by + 1 < g.ny, okz1 = bz + 1 < g.nz;
            const bool ok0 = bx < g.nx && by < g.ny && bz < g.nz;
#pragma unroll
            for (int v = 0; v < 8; ++v) {
                const int vx = v & 1, vy = (v >> 1) & 1, vz = v >> 2;
                const bool ok = ok0 && (!vx || okx1) && (!vy || oky1) && (!vz || okz1);
                P[v] = ok ? __ldg(pb + vx + vy * sy + vz * sz) : 0.0f;
            }
        }
        // window base: jlo of the cluster voxel closest to the element (exact minimiser of |d+delta|
        // coordinate-wise); other voxels have jlo >= J (up to rounding, handled by the slow path)
        const int qx = (A.dx + ex0 + 0.5f * g.hf > 0.0f) ? 0 : 1;
        const int qy = (A.dy + ey0 + 0.5f * g.hf > 0.0f) ? 0 : 1;
        const int qz = (A.dz + ez0 + 0.5f * g.hf > 0.0f) ? 0 : 1;
        int J;
        {
            const float exq = ((float)(2 * cx + qx) - 0.5f * (TX - 1)) * g.hf;
            const float eyq = ((float)(2 * cy + qy) - 0.5f * (TY - 1)) * g.hf;
            const float ezq = ((float)(2 * cz + qz) - 0.5f * (TZ - 1)) * g.hf;
            const float e2q = __fmaf_rn(exq, exq, __fmaf_rn(eyq, eyq, __fmul_rn(ezq, ezq)));
            J = pair(g, A, exq, eyq, ezq, e2q, LMIN).jlo;
        }
        J = max(J, -(LMIN + 1));  // windows ending before 0 contribute nothing
        const bool any = J <= g.nt - 1;
        if (!__any_sync(0xffffffffu, any)) continue;
        const int Jmin = warp_min(any ? J : 0x7fffffff);
        if (!any) J = Jmin;

        constexpr int R2 = (R + 1) / 2;
        float2 acc2[R2];  // acc'_i in register pairs (i even -> .x, odd -> .y)
#pragma unroll
        for (int k = 0; k < R2; ++k) acc2[k] = make_float2(0.0f, 0.0f);
#define ACC(i) (((i) & 1) ? acc2[(i) >> 1].y : acc2[(i) >> 1].x)
        unsigned ovf = 0u;  // voxels with jlo outside [J, J+OMAX) (rounding corner cases)
        const float mfa = (float)g.mF * g.af;
        const float jj = -(float)(J - A.JA);
        const float2 af2 = make_float2(g.af, g.af);
        // steps [OMAX-1, LMIN) are in-window for every voxel of the cluster: there the recurrence
        // runs packed on (i, i+1) pairs (FFMA2/FMUL2); the OMAX-1 head and the tail steps are
        // scalar and predicated.  Every loop runs over the register window with static indices; its
        // bounds tests fold away in a compiled class and are warp-uniform branches in a runtime class.
        // NV voxels per pass (independent recurrence chains, ILP NV); the recurrence runs
        // centre-out from step M
        constexpr int NV = PA_FWD_NV;
#pragma unroll 1
        for (int v0 = 0; v0 < 8; v0 += NV) {
            float cq[NV], DJ[NV], pq[NV], qq[NV], um[NV];
            int oq[NV], oLq[NV];
            float2 p2[NV], q2[NV], DJ2[NV], u2[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const int v = v0 + q, vx = v & 1, vy = (v >> 1) & 1, vz = v >> 2;
                const float ex = ex0 + (float)vx * g.hf;
                const float ey = ((float)(2 * cy + vy) - 0.5f * (TY - 1)) * g.hf;
                const float ez = ((float)(2 * cz + vz) - 0.5f * (TZ - 1)) * g.hf;
                const Pair pv = pair(g, A, ex, ey, ez, __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez))), LMIN);
                const bool in = bx + vx < g.nx && by + vy < g.ny && bz + vz < g.nz;
                float c = (in && pv.jlo <= g.nt - 1 && pv.jlo + pv.L - 1 >= 0) ? P[v] * 0.5f * pv.inv_r : 0.0f;
                int o = pv.jlo - J;
                if (c != 0.0f && (o < 0 || o >= OMAX)) {
                    ovf |= 1u << v;
                    c = 0.0f;
                }
                if (c == 0.0f) o = 0;
                cq[q] = c;
                oq[q] = o;
                oLq[q] = o + pv.L;
                DJ[q] = __fmaf_rn(jj, g.af, __fadd_rn(pv.drel, A.CA));
                const float Dm = DJ[q] - mfa;  // D at the centre step M
                DJ2[q] = make_float2(DJ[q], DJ[q]);
                if constexpr (FAM == KF_GAUSS) {
                    // u_M = E(D_m) (C_M = 1); p = exp(a D_m / s^2); walk up with p, down with 1/p
                    um[q] = c * ex2(-g.k2 * Dm * Dm);
                    const float l = 2.0f * g.k2 * g.af * Dm;
                    pq[q] = ex2(l);
                    qq[q] = ex2(-l);
                    p2[q] = make_float2(ex2(2.0f * l), 0.0f);
                    q2[q] = make_float2(ex2(-2.0f * l), 0.0f);
                    u2[q] = make_float2(um[q], um[q] * pq[q]);
                } else if constexpr (FAM == KF_EXP) {
                    // A = c exp(-D_m/s), B = c exp(D_m/s) (exponent clamped: c = 0 rows stay 0)
                    const float l = fminf(fmaxf(g.ls * Dm, -100.0f), 100.0f);
                    um[q] = c * ex2(-l);
                    pq[q] = c * ex2(l);
                } else {
                    um[q] = c;
                    pq[q] = 0.0f;
                }
            }
            if constexpr (FAM == KF_GAUSS) {
                // -- upward, packed
#pragma unroll
                for (int i = 0; i < R - 1; i += 2) {
                    if (i < M) continue;
                    if (i >= UPE) break;
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const float2 D = __ffma2_rn(fc.I2[i >> 1], af2, DJ2[q]);
                        acc2[i >> 1] = __ffma2_rn(u2[q], D, acc2[i >> 1]);
                        u2[q] = __fmul2_rn(u2[q], make_float2(p2[q].x, p2[q].x));
                    }
                }
                // -- upward tail, scalar (predicated on the window end); steps past every lane's
                // window end are skipped with a warp-uniform exit
                int mx = 0, mn = 0x7fffffff;
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    mx = max(mx, oLq[q]);
                    mn = min(mn, oq[q]);
                }
                const int tail_end = (int)__reduce_max_sync(0xffffffffu, (unsigned)mx);
                float us[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) us[q] = u2[q].x;
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    if (i < UPE) continue;
                    if (i >= tail_end) break;
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const float D = __fmaf_rn(-(float)i, g.af, DJ[q]);
                        if (i < LMIN || i < oLq[q]) ACC(i) = __fmaf_rn(us[q], D, ACC(i));
                        us[q] *= pq[q];
                    }
                }
                // -- downward, packed on pairs (i, i+1), i = M-2, M-4, ..., DNE
#pragma unroll
                for (int q = 0; q < NV; ++q) u2[q] = make_float2(um[q] * q2[q].x, um[q] * qq[q]);
#pragma unroll
                for (int i = R - 2 - (R & 1); i >= 0; i -= 2) {
                    if (i > M - 2) continue;
                    if (i < DNE) break;
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const float2 D = __ffma2_rn(fc.I2[i >> 1], af2, DJ2[q]);
                        acc2[i >> 1] = __ffma2_rn(u2[q], D, acc2[i >> 1]);
                        u2[q] = __fmul2_rn(u2[q], make_float2(q2[q].x, q2[q].x));
                    }
                }
                // -- downward head, scalar (predicated on the window start); steps before every
                // lane's window start are skipped with a warp-uniform exit
                const int head_beg = (int)__reduce_min_sync(0xffffffffu, (unsigned)mn);
#pragma unroll
                for (int q = 0; q < NV; ++q) us[q] = u2[q].y;
#pragma unroll
                for (int i = R - 1; i >= 0; --i) {
                    if (i >= DNE) continue;
                    if (i < head_beg) break;
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const float D = __fmaf_rn(-(float)i, g.af, DJ[q]);
                        if (i >= OMAX - 1 || i >= oq[q]) ACC(i) = __fmaf_rn(us[q], D, ACC(i));
                        us[q] *= qq[q];
                    }
                }
            } else {
                // exponential / power law: no recurrence state; packed where every voxel of the
                // pass is in-window, scalar and predicated at the edges (warp-uniform exits)
#pragma unroll
                for (int i = 0; i < R - 1; i += 2) {
                    if (i < DNE) continue;
                    if (i + 1 >= UPE) break;
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const float2 D = __ffma2_rn(fc.I2[i >> 1], af2, DJ2[q]);
                        acc2[i >> 1] = __ffma2_rn(fam_val2<FAM>(g, fc, i >> 1, D, um[q], pq[q]), D, acc2[i >> 1]);
                    }
                }
                int mx = 0, mn = 0x7fffffff;
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    mx = max(mx, oLq[q]);
                    mn = min(mn, oq[q]);
                }
                const int tail_end = (int)__reduce_max_sync(0xffffffffu, (unsigned)mx);
                const int head_beg = (int)__reduce_min_sync(0xffffffffu, (unsigned)mn);
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    if (i < UPE) continue;
                    if (i >= tail_end) break;
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const float D = __fmaf_rn(-(float)i, g.af, DJ[q]);
                        const float Ev = fam_val1<FAM>(g, fc, i, D, um[q], pq[q]);
                        if (i < LMIN || i < oLq[q]) ACC(i) = __fmaf_rn(Ev, D, ACC(i));
                    }
                }
#pragma unroll
                for (int i = R - 1; i >= 0; --i) {
                    if (i >= DNE) continue;
                    if (i < head_beg) break;
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const float D = __fmaf_rn(-(float)i, g.af, DJ[q]);
                        const float Ev = fam_val1<FAM>(g, fc, i, D, um[q], pq[q]);
                        if (i >= OMAX - 1 || i >= oq[q]) ACC(i) = __fmaf_rn(Ev, D, ACC(i));
                    }
                }
            }
        }
        if constexpr (FAM == KF_GAUSS) {
#pragma unroll
            for (int k = 0; k < R2; ++k) acc2[k] = __fmul2_rn(acc2[k], fc.C2[k]);
        }  // acc'_i C_i -> samples

        // ---- flush, in two half-warp phases: lanes (16 ph .. 16 ph + 15) write C_i acc'_i into
        // column (J - Jmin + i), row lane%16, of the column-major buffer (zero between uses);
        // every lane then sums whole columns with 128-bit loads (fixed order) into the warp
        // trace and clears the columns it consumed.
        const int Jmax = warp_max(J);
        if (Jmax - Jmin <= SPAN) {
            const int ncol = Jmax - Jmin + R;
            float *w = cols + (J - Jmin) * C::CSTR + (lane % C::ROWS);
#pragma unroll
            for (int ph = 0; ph < C::NPH; ++ph) {
                if (lane / C::ROWS == ph) {
#pragma unroll
                    for (int i = 0; i < R; ++i) w[i * C::CSTR] = ACC(i);
                }
                __syncwarp();
                for (int c = lane; c < ncol; c += 32) {
                    float4 *col = reinterpret_cast<float4 *>(cols + c * C::CSTR);
                    float4 a = col[0];
#pragma unroll
                    for (int q = 1; q < C::ROWS / 4; ++q) {
                        const float4 t = col[q];
                        a.x += t.x;
                        a.y += t.y;
                        a.z += t.z;
                        a.w += t.w;
                    }
                    trw[C::PADL + Jmin + c] += (a.x + a.y) + (a.z + a.w);
                    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);  // consume-and-clear
#pragma unroll
                    for (int q = 0; q < C::ROWS / 4; ++q) col[q] = z4;
                }
                __syncwarp();
            }
        } else {
            // serialized fallback (not reached for supported geometry)
            for (int l = 0; l < 32; ++l) {
                if (lane == l) {
#pragma unroll
                    for (int i = 0; i < R; ++i) trw[C::PADL + J + i] += ACC(i);
                }
                __syncwarp();
            }
        }
#undef ACC
        // ---- exact slow path for any voxel outside the register window (lane-serialised)
        const unsigned ovm = __ballot_sync(0xffffffffu, ovf != 0u);
        if (ovm) {
            for (int l = 0; l < 32; ++l) {
                if (!((ovm >> l) & 1u)) continue;
                if (lane == l) {
                    for (int v = 0; v < 8; ++v) {
                        if (!((ovf >> v) & 1u)) continue;
                        const int vx = v & 1, vy = (v >> 1) & 1, vz = v >> 2;
                        const float ex = ((float)(2 * cx + vx) - 0.5f * (TX - 1)) * g.hf;
                        const float ey = ((float)(2 * cy + vy) - 0.5f * (TY - 1)) * g.hf;
                        const float ez = ((float)(2 * cz + vz) - 0.5f * (TZ - 1)) * g.hf;
                        const Pair pv = pair(g, A, ex, ey, ez, __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez))), LMIN);
                        const float cv = P[v] * 0.5f * pv.inv_r;
                        for (int i = 0; i < pv.L; ++i) {
                            const int j = pv.jlo + i;
                            const float D = __fmaf_rn(-(float)(j - A.JA), g.af, __fadd_rn(pv.drel, A.CA));
                            if (j >= 0 && j < g.nt) trw[C::PADL + j] += cv * D * fam_direct<FAM>(g, D);
                        }
                    }
                }
                __syncwarp();
            }
        }
    }
    __syncthreads();

    // ---- sum warp traces in fixed order; epilogue
    const int nt = g.nt;
    const size_t rowoff = (size_t)fe * nt;
    const int wf = C::warp_floats(nt);
    const bool masked = row_mask != nullptr && row_mask[fe] == 0;
    __shared__ double red[FWD_WARPS * 32];
    if (mode == FWD_TRACE) {
        for (int j = threadIdx.x; j < nt; j += blockDim.x) {
            float s = 0.0f;
#pragma unroll
            for (int w = 0; w < FWD_WARPS; ++w) s += sm[w * wf + C::PADL + j];
            out[rowoff + j] = s;
        }
        return;
    }
    // y -> warp-0 trace slot (each j owned by one thread; read all warps before writing)
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        float s = 0.0f;
#pragma unroll
        for (int w = 0; w < FWD_WARPS; ++w) s += sm[w * wf + C::PADL + j];
        sm[C::PADL + j] = s;
    }
    __syncthreads();
    const float *y = sm + C::PADL;
    const float *S = meas + rowoff;
    if (mode == FWD_MSE) {
        double part = 0.0;
        for (int j = threadIdx.x; j < nt; j += blockDim.x) {
            const float d = y[j] - __ldg(S + j);
            part += (double)d * (double)d;
            out[rowoff + j] = masked ? 0.0f : 2.0f * d;
        }
        const double tot = block_sum(part, red);
        if (threadIdx.x == 0) rowloss[fe] = masked ? 0.0 : tot;
        return;
    }
    // NC (Eq. 3, population normalisation)
    double sy = 0.0, ss = 0.0;
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        sy += y[j];
        ss += __ldg(S + j);
    }
    const double my = block_sum(sy, red) / nt, ms = block_sum(ss, red) / nt;
    double cv = 0.0, vy = 0.0, vs = 0.0;
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        const double a = y[j] - my, b = (double)__ldg(S + j) - ms;
        cv += a * b;
        vy += a * a;
        vs += b * b;
    }
    const double COV = block_sum(cv, red) / nt, VY = block_sum(vy, red) / nt, VS = block_sum(vs, red) / nt;
    const double sdy = sqrt(VY), sds = sqrt(VS);
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        const double gj = -(((double)__ldg(S + j) - ms) / (sdy * sds) - COV * (y[j] - my) / (sdy * sdy * sdy * sds)) / nt;
        out[rowoff + j] = masked ? 0.0f : (float)gj;
    }
    if (threadIdx.x == 0) rowloss[fe] = masked ? 0.0 : -COV / (sdy * sds);
}

// ============================================================================================
// K2 (+K3 partials) — adjoint back-projection (a4) fused with the element/pose gradient (a5).
//
// Persistent CTAs (grid = 2 x #SM), one thread per voxel of an 8x8x4 tile; static tile
// ownership.  Loop order: frame chunk (Fc frames) > tile > frame > element.  Per (tile,
// frame) all E cotangent segments the tile can touch are staged in shared memory (zero
// padded outside [0, nt)) and all E fp64 anchors are formed once.  Each thread walks its
// voxel's L-sample window with the exp recurrence:
//   A1 = sum g D E   (adjoint: z += A1/(2r))
//   Bq = sum g E (D^2 - s^2)  => sum g h'(D) = -Bq/s^2
//   dL/dr = P/(2r) (-Bq/s^2 - A1/r);  G_fe += dL/dr (x_fe - y_k)/r       (R11)
// G is reduced over the 32 voxels of a warp by shuffles, over the 8 warps in smem (fixed
// order), accumulated over the CTA's tiles for the frame chunk, and written as a per-CTA
// partial [P][F][E][3] reduced by K3 in fixed order.  z stays in a register across the
// frames of a chunk and is read-modified-written once per chunk by its owner thread.
// ============================================================================================
struct AdjCfg {
    static __host__ __device__ size_t smem_floats(int E, int SEG, int Fc, bool pose)
    {
        size_t f = (size_t)E * SEG + (size_t)E * 12 /*anchors*/ + (size_t)E /*jseg*/;
        if (pose) f += (size_t)(ADJ_THREADS / 32) * E * 3 + (size_t)Fc * E * 3;
        return f;
    }
};

struct AncS {  // anchor as stored in shared memory (12 words)
    float dx2, dy2, dz2, dx, dy, dz, rho, rho2, CA;
    int JA, cull, jseg;
};

// LMIN_ = 0: a runtime class (L_min = Geo::lmin, the segment length Geo::seg).
template <int LMIN_, int SEG_, bool POSE, bool ADJ, int FAM>
__global__ void __launch_bounds__(ADJ_THREADS, 2) k_adjoint(Geo g, AdjConst ac, const float *__restrict__ poses,
                                                           const float *__restrict__ tmpl,
                                                           const float *__restrict__ p0,
                                                           const float *__restrict__ cot, float *__restrict__ grad_p0,
                                                           float *__restrict__ partial, int Fc)
{
    const int LMIN = LMIN_ > 0 ? LMIN_ : g.lmin;
    const int SEG = SEG_ > 0 ? SEG_ : g.seg;
    const int LMAX = LMIN + 1;
    constexpr int UNR = LMIN_ > 0 ? 128 : 4;  // full unroll in a compiled class
    extern __shared__ float sm[];
    const int E = g.E, F = g.F;
    float *seg = sm;
    AncS *anc = reinterpret_cast<AncS *>(seg + (size_t)E * SEG);
    float *wred = reinterpret_cast<float *>(anc + E);  // [8][E][3]
    float *gacc = wred + (ADJ_THREADS / 32) * E * 3;  // [Fc][E][3]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int lx = tid & 7, ly = (tid >> 3) & 7, lz = tid >> 6;
    const float ex = ((float)lx - 0.5f * (TX - 1)) * g.hf;
    const float ey = ((float)ly - 0.5f * (TY - 1)) * g.hf;
    const float ez = ((float)lz - 0.5f * (TZ - 1)) * g.hf;
    const float e2 = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez)));

    for (int f0 = 0; f0 < F; f0 += Fc) {
        const int fn = min(Fc, F - f0);
        if (POSE) {
            for (int q = tid; q < Fc * E * 3; q += ADJ_THREADS) gacc[q] = 0.0f;
        }
        for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
            const int tx = tile % g.ntx, ty = (tile / g.ntx) % g.nty, tz = tile / (g.ntx * g.nty);
            const int ix = TX * tx + lx, iy = TY * ty + ly, iz = TZ * tz + lz;
            const bool inside = ix < g.nx && iy < g.ny && iz < g.nz;
            const size_t kidx = ((size_t)iz * g.ny + iy) * g.nx + ix;
            const float P = (POSE && inside) ? __ldg(p0 + kidx) : 0.0f;
            float z = 0.0f;
            for (int fl = 0; fl < fn; ++fl) {
                const int f = f0 + fl;
                __syncthreads();  // previous frame's segments / wred fully consumed
                for (int e = tid; e < E; e += ADJ_THREADS) {
                    double x[3];
                    elem_pos(poses, tmpl, f, e, x);
                    const Anc A = make_anchor(g, x, tx, ty, tz);
                    AncS s;
                    s.dx2 = A.dx2; s.dy2 = A.dy2; s.dz2 = A.dz2;
                    s.dx = A.dx; s.dy = A.dy; s.dz = A.dz;
                    s.rho = A.rho; s.rho2 = A.rho2; s.CA = A.CA;
                    s.JA = A.JA; s.cull = A.cull;
                    s.jseg = A.JA + (int)floorf((A.CA - g.rt - g.ksig) * g.inv_a) - 2;
                    anc[e] = s;
                }
                __syncthreads();
                // stage the E cotangent segments with asynchronous global->shared copies (LDGSTS,
                // zero-filled outside [0, nt) and for culled elements): all loads in flight at once
                const float *cf = cot + (size_t)f * E * g.nt;
                for (int q = tid; q < E * SEG; q += ADJ_THREADS) {
                    const int e = q / SEG, i = q - e * SEG;
                    const int j = anc[e].jseg + i;
                    const bool ok = !anc[e].cull && j >= 0 && j < g.nt;
                    const float *src = ok ? cf + (size_t)e * g.nt + j : cf;
                    const unsigned dst = (unsigned)__cvta_generic_to_shared(seg + q);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src),
                                 "r"(ok ? 4 : 0));
                }
                asm volatile("cp.async.wait_all;\n" ::);
                __syncthreads();
#pragma unroll 1
                for (int e0 = 0; e0 < E; e0 += 4) {
                    float G[4][3];
#pragma unroll
                    for (int q = 0; q < 4; q += 2) {
                        // two elements per pass, packed fp32x2 arithmetic (FFMA2/FMUL2: half the
                        // issue slots for the same FP32-pipe work)
                        const int ea = e0 + q, eb = e0 + q + 1;
                        G[q][0] = G[q][1] = G[q][2] = G[q + 1][0] = G[q + 1][1] = G[q + 1][2] = 0.0f;
                        if (ea >= E) continue;  // uniform
                        const bool hb = eb < E;
                        const AncS sa = anc[ea], sb = anc[hb ? eb : ea];
                        if (sa.cull && (!hb || sb.cull)) continue;  // uniform
                        Anc Aa, Ab;
                        Aa.dx2 = sa.dx2; Aa.dy2 = sa.dy2; Aa.dz2 = sa.dz2; Aa.dx = sa.dx; Aa.dy = sa.dy; Aa.dz = sa.dz;
                        Aa.rho = sa.rho; Aa.rho2 = sa.rho2; Aa.CA = sa.CA; Aa.JA = sa.JA; Aa.cull = 0;
                        Ab.dx2 = sb.dx2; Ab.dy2 = sb.dy2; Ab.dz2 = sb.dz2; Ab.dx = sb.dx; Ab.dy = sb.dy; Ab.dz = sb.dz;
                        Ab.rho = sb.rho; Ab.rho2 = sb.rho2; Ab.CA = sb.CA; Ab.JA = sb.JA; Ab.cull = 0;
                        const Pair pa = pair(g, Aa, ex, ey, ez, e2, LMIN);
                        const Pair pb = pair(g, Ab, ex, ey, ez, e2, LMIN);
                        const bool va = inside && !sa.cull && pa.jlo <= g.nt - 1 && pa.jlo + pa.L - 1 >= 0;
                        const bool vb = inside && hb && !sb.cull && pb.jlo <= g.nt - 1 && pb.jlo + pb.L - 1 >= 0;
                        const int offa = va ? min(max(pa.jlo - sa.jseg, 0), SEG - LMAX) : 0;
                        const int offb = vb ? min(max(pb.jlo - sb.jseg, 0), SEG - LMAX) : 0;
                        const float *gsa = seg + ea * SEG + offa;
                        const float *gsb = seg + (hb ? eb : ea) * SEG + offb;
                        const int MA = (LMIN + 1) / 2;  // == Geo::mA
                        const float Dma = __fmaf_rn(-(float)(pa.jlo - sa.JA), g.af, __fadd_rn(pa.drel, sa.CA)) - (float)MA * g.af;
                        const float Dmb = __fmaf_rn(-(float)(pb.jlo - sb.JA), g.af, __fadd_rn(pb.drel, sb.CA)) - (float)MA * g.af;
                        // A1 = sum g D K (adjoint);  A2 = sum g (K + D K') (pose, d/dr of D K)
                        float A1a, A1b, A2a = 0.0f, A2b = 0.0f;
                        if constexpr (FAM == KF_GAUSS) {
                            // centre-out: u_MA = E(D_m); up with p = exp(a D_m/s^2), down with 1/p
                            const float2 um = make_float2(ex2(-g.k2 * Dma * Dma), ex2(-g.k2 * Dmb * Dmb));
                            const float la = 2.0f * g.k2 * g.af * Dma, lb = 2.0f * g.k2 * g.af * Dmb;
                            const float2 pu = make_float2(ex2(la), ex2(lb)), pd = make_float2(ex2(-la), ex2(-lb));
#if PA_ADJ_HORNER
                            // Moments S_n = sum_i g_i E_i (i - MA)^n with E_i = um C_i x^|i-MA| (x = pu above
                            // MA, pd below) are polynomials in x with coefficients c_k = g C: Horner with
                            // synthetic-division derivatives, b = P(x), d1 = P'(x), d2 = P''(x)/2, from the
                            // outermost step inwards (3 FFMA2 + 1 FMUL2 per step for two elements):
                            //   sum c_k x^k = b, sum k c_k x^k = x d1, sum k^2 c_k x^k = x d1 + 2 x^2 d2.
                            const float2 z2 = make_float2(0.f, 0.f);
                            float2 bu = z2, d1u = z2, d2u = z2, bd = z2, d1d = z2, d2d = z2;
#pragma unroll UNR
                            for (int i = LMAX - 1; i >= MA; --i) {
                                float2 c = __fmul2_rn(make_float2(gsa[i], gsb[i]), make_float2(ac.C0[i], ac.C0[i]));
                                if (i >= LMIN) {
                                    c.x = i < pa.L ? c.x : 0.0f;
                                    c.y = i < pb.L ? c.y : 0.0f;
                                }
                                if (POSE) d2u = __ffma2_rn(d2u, pu, d1u);
                                d1u = __ffma2_rn(d1u, pu, bu);
                                bu = __ffma2_rn(bu, pu, c);
                            }
#pragma unroll UNR
                            for (int i = 0; i <= MA; ++i) {  // k = MA - i; the k = 0 step (i = MA) adds 0
                                const float2 c = i < MA ? __fmul2_rn(make_float2(gsa[i], gsb[i]),
                                                                     make_float2(ac.C0[i], ac.C0[i]))
                                                        : z2;
                                if (POSE) d2d = __ffma2_rn(d2d, pd, d1d);
                                d1d = __ffma2_rn(d1d, pd, bd);
                                bd = __ffma2_rn(bd, pd, c);
                            }
                            const float2 xu1 = __fmul2_rn(pu, d1u), xd1 = __fmul2_rn(pd, d1d);
                            const float2 S0 = __fmul2_rn(um, __fadd2_rn(bu, bd));
                            const float2 S1 = __fmul2_rn(um, make_float2(xu1.x - xd1.x, xu1.y - xd1.y));
                            float2 S2 = z2;
                            if (POSE) {
                                const float2 two = make_float2(2.f, 2.f);
                                const float2 su = __ffma2_rn(__fmul2_rn(two, __fmul2_rn(pu, pu)), d2u, xu1);
                                const float2 sd = __ffma2_rn(__fmul2_rn(two, __fmul2_rn(pd, pd)), d2d, xd1);
                                S2 = __fmul2_rn(um, __fadd2_rn(su, sd));
                            }
#else
                            float2 S0 = make_float2(0.f, 0.f), S1 = S0, S2 = S0;  // sum g E k^n, k = i - MA
                            float2 u = um;
#pragma unroll UNR
                            for (int i = MA; i < LMAX; ++i) {
                                float2 t = __fmul2_rn(make_float2(gsa[i], gsb[i]), u);
                                if (i >= LMIN) {
                                    t.x = i < pa.L ? t.x : 0.0f;
                                    t.y = i < pb.L ? t.y : 0.0f;
                                }
                                S0 = __ffma2_rn(t, make_float2(ac.C0[i], ac.C0[i]), S0);
                                S1 = __ffma2_rn(t, make_float2(ac.C1[i], ac.C1[i]), S1);
                                if (POSE) S2 = __ffma2_rn(t, make_float2(ac.C2[i], ac.C2[i]), S2);
                                u = __fmul2_rn(u, pu);
                            }
                            u = __fmul2_rn(um, pd);
#pragma unroll UNR
                            for (int i = MA - 1; i >= 0; --i) {
                                const float2 t = __fmul2_rn(make_float2(gsa[i], gsb[i]), u);
                                S0 = __ffma2_rn(t, make_float2(ac.C0[i], ac.C0[i]), S0);
                                S1 = __ffma2_rn(t, make_float2(ac.C1[i], ac.C1[i]), S1);
                                if (POSE) S2 = __ffma2_rn(t, make_float2(ac.C2[i], ac.C2[i]), S2);
                                u = __fmul2_rn(u, pd);
                            }
#endif
                            // A1 = sum g D E = Dm S0 - a S1 ;  Bq = sum g E (D^2 - s^2)
                            A1a = __fmaf_rn(-g.af, S1.x, Dma * S0.x);
                            A1b = __fmaf_rn(-g.af, S1.y, Dmb * S0.y);
                            float Bqa = 0.0f, Bqb = 0.0f;
                            if (POSE) {
                                Bqa = (Dma * Dma - g.s2) * S0.x - 2.0f * g.af * Dma * S1.x + g.af * g.af * S2.x;
                                Bqb = (Dmb * Dmb - g.s2) * S0.y - 2.0f * g.af * Dmb * S1.y + g.af * g.af * S2.y;
                                A2a = -Bqa * g.inv_s2;  // sum g (K + D K') = -Bq / s^2
                                A2b = -Bqb * g.inv_s2;
                            }
                        } else {
                            // exponential: K_i = min(A C0_i, B C1_i); power law: K = 2^(-nu lg2(D^2+s^2)).
                            // SX: exp sum t|D|, power law sum t/(D^2+s^2)
                            const float2 Dm2 = make_float2(Dma, Dmb), af2 = make_float2(g.af, g.af);
                            float2 Ae = make_float2(0.f, 0.f), Be = Ae;
                            if constexpr (FAM == KF_EXP) {
                                const float la = fminf(fmaxf(g.ls * Dma, -100.0f), 100.0f);
                                const float lb = fminf(fmaxf(g.ls * Dmb, -100.0f), 100.0f);
                                Ae = make_float2(ex2(-la), ex2(-lb));
                                Be = make_float2(ex2(la), ex2(lb));
                            }
                            float2 SE = make_float2(0.f, 0.f), SD = SE, SX = SE;
#pragma unroll UNR
                            for (int i = 0; i < LMAX; ++i) {
                                const float2 D = __ffma2_rn(make_float2((float)(MA - i), (float)(MA - i)), af2, Dm2);
                                float2 Kv;
                                float2 lx;
                                if constexpr (FAM == KF_EXP) {
                                    const float2 t1 = __fmul2_rn(Ae, make_float2(ac.C0[i], ac.C0[i]));
                                    const float2 t2 = __fmul2_rn(Be, make_float2(ac.C1[i], ac.C1[i]));
                                    Kv = make_float2(fminf(t1.x, t2.x), fminf(t1.y, t2.y));
                                } else {
                                    const float2 x = __ffma2_rn(D, D, make_float2(g.s2, g.s2));
                                    lx = make_float2(lg2(x.x), lg2(x.y));
                                    Kv = make_float2(ex2(-g.nu * lx.x), ex2(-g.nu * lx.y));
                                }
                                float2 t = __fmul2_rn(make_float2(gsa[i], gsb[i]), Kv);
                                if (i >= LMIN) {
                                    t.x = i < pa.L ? t.x : 0.0f;
                                    t.y = i < pb.L ? t.y : 0.0f;
                                }
                                SE = __fadd2_rn(SE, t);
                                SD = __ffma2_rn(t, D, SD);
                                if (POSE) {
                                    if constexpr (FAM == KF_EXP)
                                        SX = __ffma2_rn(t, make_float2(fabsf(D.x), fabsf(D.y)), SX);
                                    else
                                        SX = __ffma2_rn(t, make_float2(ex2(-lx.x), ex2(-lx.y)), SX);
                                }
                            }
                            A1a = SD.x;
                            A1b = SD.y;
                            if (POSE) {
                                if constexpr (FAM == KF_EXP) {
                                    const float inv_s = g.ls * 0.69314718f;  // K + D K' = K (1 - |D|/s)
                                    A2a = SE.x - inv_s * SX.x;
                                    A2b = SE.y - inv_s * SX.y;
                                } else {  // K + D K' = K (1 - 2 nu D^2/x) = K ((1 - 2 nu) + 2 nu s^2 / x)
                                    A2a = (1.0f - 2.0f * g.nu) * SE.x + 2.0f * g.nu * g.s2 * SX.x;
                                    A2b = (1.0f - 2.0f * g.nu) * SE.y + 2.0f * g.nu * g.s2 * SX.y;
                                }
                            }
                        }
                        if (!va) A1a = A2a = 0.0f;
                        if (!vb) A1b = A2b = 0.0f;
                        if (ADJ) z = __fmaf_rn(A1b, 0.5f * pb.inv_r, __fmaf_rn(A1a, 0.5f * pa.inv_r, z));
                        if (POSE) {
                            const float dLa = P * 0.5f * pa.inv_r * (A2a - A1a * pa.inv_r);
                            const float dLb = P * 0.5f * pb.inv_r * (A2b - A1b * pb.inv_r);
                            const float sca = -dLa * pa.inv_r, scb = -dLb * pb.inv_r;  // x - y_k = -(d + delta)
                            G[q][0] = sca * (sa.dx + ex);
                            G[q][1] = sca * (sa.dy + ey);
                            G[q][2] = sca * (sa.dz + ez);
                            G[q + 1][0] = scb * (sb.dx + ex);
                            G[q + 1][1] = scb * (sb.dy + ey);
                            G[q + 1][2] = scb * (sb.dz + ez);
                        }
                    }
                    if (POSE) {
                        // transposed warp reduction of 4 elements x 3 components (54 instr / 4 elements)
                        const bool h16 = (lane & 16) != 0, h8 = (lane & 8) != 0;
                        float r6[6];
#pragma unroll
                        for (int j = 0; j < 6; ++j) {
                            const float lo = G[j / 3][j % 3], hi = G[2 + j / 3][j % 3];
                            const float snd = h16 ? lo : hi, kp = h16 ? hi : lo;
                            r6[j] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
                        }
                        float r3[3];
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            const float lo = r6[c], hi = r6[3 + c];
                            const float snd = h8 ? lo : hi, kp = h8 ? hi : lo;
                            r3[c] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
                        }
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            r3[c] += __shfl_xor_sync(0xffffffffu, r3[c], 4);
                            r3[c] += __shfl_xor_sync(0xffffffffu, r3[c], 2);
                            r3[c] += __shfl_xor_sync(0xffffffffu, r3[c], 1);
                        }
                        const int e = e0 + ((lane >> 3) & 3);
                        if ((lane & 7) == 0 && e < E) {
                            wred[(warp * E + e) * 3 + 0] = r3[0];
                            wred[(warp * E + e) * 3 + 1] = r3[1];
                            wred[(warp * E + e) * 3 + 2] = r3[2];
                        }
                    }
                }
                if (POSE) {
                    __syncthreads();
                    for (int q = tid; q < E * 3; q += ADJ_THREADS) {
                        float s = 0.0f;
#pragma unroll
                        for (int w = 0; w < ADJ_THREADS / 32; ++w) s += wred[w * E * 3 + q];
                        gacc[fl * E * 3 + q] += s;
                    }
                }
            }
            if (ADJ && inside) grad_p0[kidx] = (f0 == 0 ? 0.0f : grad_p0[kidx]) + z;
        }
        if (POSE) {
            __syncthreads();
            for (int q = tid; q < fn * E * 3; q += ADJ_THREADS)
                partial[((size_t)blockIdx.x * F + f0) * E * 3 + q] = gacc[q];
            __syncthreads();
        }
    }
}

// ============================================================================================
// K2 (Gaussian), moment-filter form.  Relative to the voxel's window centre m (index j_m =
// jlo + MA), D_k = D_m - k a and
//   E_k = exp(-D_k^2/2s^2) = u_m C_k e^{lam k},   u_m = e^{-D_m^2/2s^2}, C_k = e^{-k^2 a^2/2s^2},
//   lam = a D_m / s^2.
// By construction of the window (D at its first sample lies in (kappa s - a, kappa s]) D_m lies
// within 1.5 samples of zero, so lam stays within +-(a/s)^2/2 of a per-class constant lam0.  With
// dl = lam - lam0 and C'_k = C_k e^{lam0 k}:
//   S_n = sum_k g[j_m + k] C_k k^n e^{lam k} = sum_{m=0..M} dl^m/m! F_{n+m}[j_m] (+ remainder),
//   F_p[j] = sum_{k=-MA}^{LMIN-MA-1} g[j + k] C'_k k^p          (per (frame, element) row)
// — the exact Taylor series of e^{dl k}, truncated at M where the remainder is below fp32
// rounding (checked on the host for the actual geometry, else the direct kernel runs).  The
// window's optional last sample (L = LMIN + 1, k = LMIN - MA) is added directly.  Then
//   A1 = sum g E D = u_m (D_m S0 - a S1),  Bq = sum g E (D^2 - s^2) = u_m ((D_m^2-s^2) S0 - 2a D_m S1 + a^2 S2)
// exactly as the direct kernel.  K2a computes F for a frame chunk (L2-resident); K2c (below) replaces
// the per-voxel L-sample walk by one filter-record load and three M-term Horner evaluations.
// ============================================================================================
// The window length L_min is a runtime value (Geo::lmin), up to PA_LMAX; the record size NF is a
// template parameter.
//
// The moments as one polynomial: with H_p = F_p / p!, P(x) = sum_{p<NPS} H_p x^p gives
//   S0 = P(dl),  S1 = P'(dl),  S2 = P''(dl)
// (the Taylor series of S_n is sum_m dl^m/m! F_{n+m}), evaluated together by Horner with synthetic
// division — S0, S1, S2 to orders NPS-1, NPS-2, NPS-3 from NPS stored values.
// Filter record of a position (NF floats, one 256-bit load for NF = 8): H_0 .. H_{NPS-1}, NPS = NF - 1,
// and in the last slot the cotangent sample at the position scaled by C_k(k_t)/2 — the window's optional
// last tap — so a pair needs exactly one load.  Orders for NF = 8: 6 / 5 / 4; NF = 12 (short windows):
// 10 / 9 / 8.  The host bounds the remainders: S0, S1 <= 4e-7, the pose moment S2 <= 1e-5 (as K2s's).
// All filters carry the factor 1/2 of D/(2r).  Rows are zero-padded by PADL / PADR positions on both
// sides, so every pair of a non-culled (tile, element) — and every pair of a culled one, through a
// sentinel anchor — addresses a valid position: no per-pair bounds checks (windows outside [0, nt)
// read zeros).
constexpr int PA_LMAX = 512;  // longest window (L_min) of the Gaussian fast path (K1d, K2a/K2c, K2s)
template <int NF_>
struct TayCfg {
    static constexpr int NF = NF_;       // floats per record (32 / 48 B)
    static constexpr int NPS = NF - 1;   // H_0 .. H_{NPS-1} stored
};
constexpr int TAY_MAXNP = 11;  // NF <= 12

struct TayFilt {               // K2a: the filter taps
    float H[PA_LMAX * TAY_MAXNP];  // H[t][p] = C'_k k^p / (2 p!), k = t - MA, t in [0, L_min), p in [0, NPS)
    float gx;                      // C_k(k_t) / 2 at the extra tap k_t = L_min - MA
    int padl;                      // leading zero positions of a row
};
struct TayConst {              // K2c: the series constants
    float lam0;        // series centre (natural units)
    float lam_s;       // a / s^2: lam = lam_s D_m
    float c_a;         // -2 a / s^2   (pose moment Bq / s^2)
    float c_aa;        // 2 a^2 / s^2  (S2 = 2 x the synthetic-division d2)
};

template <int NF>
__global__ void __launch_bounds__(256) k_adj_filter(Geo g, TayFilt tf, const float *__restrict__ cot, int f0, int fn,
                                                    int njp, float *__restrict__ Fg)
{
    using T = TayCfg<NF>;
    __shared__ float s[256 + PA_LMAX];
    const int lmin = g.lmin;
    const int row = blockIdx.y;  // chunk-local row (f - f0) E + e
    const int jp0 = blockIdx.x * 256;
    const int jj0 = jp0 - tf.padl;  // position jj = jp - PADL; j_m = jj + MA - L_min
    const float *gr = cot + ((size_t)f0 * g.E + row) * g.nt;
    // the taps k in [-MA, L_min - MA) read samples jj - L_min + t, t = k + MA; the last tap sample jj
    for (int t = threadIdx.x; t < 256 + lmin; t += 256) {
        const int j = jj0 - lmin + t;
        s[t] = (j >= 0 && j < g.nt) ? __ldg(gr + j) : 0.0f;
    }
    __syncthreads();
    const int jp = jp0 + threadIdx.x;
    if (jp >= njp) return;
    float acc[T::NF];
#pragma unroll
    for (int p = 0; p < T::NF; ++p) acc[p] = 0.0f;
#pragma unroll 2
    for (int t = 0; t < lmin; ++t) {
        const float v = s[threadIdx.x + t];
#pragma unroll
        for (int p = 0; p < T::NPS; ++p) acc[p] = __fmaf_rn(v, tf.H[t * T::NPS + p], acc[p]);
    }
    acc[T::NF - 1] = s[threadIdx.x + lmin] * tf.gx;  // the last tap's sample g[jj] C_k(k_t) / 2
    float4 *o = reinterpret_cast<float4 *>(Fg + ((size_t)row * njp + jp) * T::NF);
#pragma unroll
    for (int q = 0; q < T::NF / 4; ++q) o[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
}

// ============================================================================================
// K1d — forward radiation (a2 + fused a3), Gaussian, deposit form.
//
// Relative to the pair window centre j_m = jlo + MA, every main tap k in [-MA, LMIN-MA) is in
// the window for every pair, and the term at sample j_m + k is
//   c * G(D_m, k),  G(D_m, k) = D_k exp(-D_k^2/2s^2),  D_k = D_m - k a,  c = P/(2r),
// with D_m confined by the window construction to an interval of width a.  On that interval G
// has a separable approximation of rank R (host: Chebyshev fit + one-sided Jacobi SVD, error
// checked on a fine grid):
//   G(D_m, k) ~= sum_{m<R} phi_m(t) psi_m(k),   t = (D_m - Dc)/Dw in [-1, 1],
// phi_m a polynomial of parity m (4 coefficients in t^2).  So a pair deposits R numbers
// c phi_m(t) at ONE position pos = j_m + OFF of a per-row channel accumulator, plus the exact
// optional last tap (L = LMIN + 1) in channel X, and the trace is, once per row,
//   y[j] = sum_{q=1..LMIN} sum_m Q_m[j + q] psi_m(OFF - q) + Q_X[j].
// Deposits are fixed-point integers (red.shared.add: integer addition is associative, so the
// result is deterministic): per-position scale r_lo(pos) <= r removes 1/r, 1/Pmax normalises P,
// and per-channel scales bound |n| <= 2^NB (channel 0 in two words, hi 2^10 + lo).  A round =
// one 8x8x4 tile per warp; after each round the touched range is flushed into fp32 accumulators
// in a fixed order.  Layout [pos][channel] with an odd stride: the R + 2 words of a deposit are
// immediate offsets of one address, and 32 lanes at distinct positions hit distinct banks.
// ============================================================================================
constexpr int DEP_MAXR = 7;  // separable rank 5, 6 or 7 (7 for the shortest windows, L_min < ~21)

// rank per window class: the factorisation error is <= ~2e-8 (L_min 53), 5e-9 (26, rank 6),
// 6e-10 (106) of max|G|
#ifndef PA_DEP_RANK_SHORT
#define PA_DEP_RANK_SHORT 6  // rank for the short-window class (L_min <= 32)
#endif

struct DepConst {
    float psi[DEP_MAXR][PA_LMAX];  // psi[m][q-1] = psi_m(k = OFF - q), q in [1, L_min]
    float2 cf2[DEP_MAXR + 1][4]; // (c, c): phi_m(t) = t^(m%2) (c0 + s c1 + s^2 c2 + s^3 c3), s = t^2, scaled by S_m;
                                 // X (index R): c0 + t c1 + t^2 c2 + t^3 c3, scaled by S_X
    float dec[DEP_MAXR + 1];   // 0.5 / S_m  (x Pmax / r_lo at decode)
    float tA, tB;              // t = tA * bse - clo * tB + tC   (= (D_m - Dc) / Dw)
    float tC;
    float W0;                  // r_lo(pos) = max(r_min, pos * a + W0) <= r of every pair depositing at pos
    int nr;                    // positions of the round accumulator ring (>= the span a round can touch)
    unsigned nrm;              // nr - 1 (nr a power of two), or ~0 when the ring covers the whole row (nr = NJ)
};

#ifndef PA_DEP_CNT
// 1: deposits carry the raw shifter bits (0x4B400000 + n: no subtraction per deposit) and a count word per
// position (one more atomic of the constant 1); the flush removes count x 0x4B400000 (mod 2^32, exact since
// |sum n| < 2^30).  Measured 1% faster at C4 than subtracting per deposit (124.6 vs 125.8 ms per 16 frames).
#define PA_DEP_CNT 1
#endif
#ifndef PA_DEP_UNROLL2
#define PA_DEP_UNROLL2 1  // the slot loop unrolled by 2 (a tile pair: anchor and row offsets fold per half): C4 -2.3%, C2 -2.4%
#endif
#ifndef PA_DEP_LATEPF
#define PA_DEP_LATEPF 1  // 1: the next slot's amplitudes are loaded after this slot's deposits (no register copy): C4 -1.1%, C5 -1.4%
#endif
#ifndef PA_DEP_FASTLOAD
#define PA_DEP_FASTLOAD 1  // K1d: unpredicated 64-bit amplitude loads for tiles inside the grid (even nx): C4 forward 114.2 -> 105.3 ms per 16 frames
#endif
#ifndef PA_DEP_MAP
#define PA_DEP_MAP 2  // lane -> voxel map: 2 = two z-adjacent tiles per warp slot (default); 1 = one tile, 2x4x1 per lane; 0 = 2x2x2 cluster
#endif
// |deposit| <= 2^NB with NW warps x TPR tiles x 256 voxels adding to a word per round: sums < 2^30
constexpr int dep_ilog2(int x) { return x <= 1 ? 0 : 1 + dep_ilog2(x / 2); }
constexpr int dep_nb(int nw, int tpr) { return 22 - dep_ilog2(nw * tpr); }

// G = copies of the round accumulator, interleaved per position; lane l deposits into copy l % G
// (chosen per geometry on the host: Plan::dep_g)
template <int R_, int NW, int G_ = 1, int TPR_ = 4>
struct DepCfg {
    static constexpr int R = R_;                  // separable rank (5 or 6; chosen per geometry on the host)
    static constexpr int NQ = R + 2 + PA_DEP_CNT; // int words per position: R channels, X, low word of channel 0
                                                  // (+ the deposit count, PA_DEP_CNT)
    static constexpr int G = G_;                  // lanes of one deposit instruction at the same position hit
                                                  // G different words (same-address atomics serialise)
    static constexpr int CS = (G * NQ) | 1;       // odd stride
    static constexpr int CF = R + 1;              // fp32 words per position
    static constexpr int TPR = TPR_;              // tiles per warp per round (4 or 8, chosen per geometry on the host)
    static constexpr int NB = dep_nb(NW, TPR);    // a round adds <= 256 NW TPR deposits per word
    static constexpr int NB0 = NB + 10;           // channel 0: hi (<= 2^NB) * 2^10 + lo
    static __host__ __device__ int njp(int nt, int lmin) { return nt + lmin; }
    // ring of nr positions x CS round words + NJ x CF fp32 row accumulators
    static __host__ __device__ size_t smem_bytes(int nt, int lmin, int nr) { return ((size_t)CS * nr + (size_t)CF * njp(nt, lmin)) * 4; }
};

// Row epilogue shared by the forward kernels: y (shared memory, nt floats) -> trace, or the MSE / NC
// cotangent and row loss (a3; Eq. 2, Eq. 3; mask Eq. 4).
__device__ __forceinline__ void fwd_epilogue(const Geo &g, const float *y, int fe, float *__restrict__ out, int mode,
                                             const float *__restrict__ meas, const uint8_t *__restrict__ row_mask,
                                             double *__restrict__ rowloss, double *red)
{
    const int nt = g.nt;
    const size_t rowoff = (size_t)fe * nt;
    if (mode == FWD_TRACE) {
        for (int j = threadIdx.x; j < nt; j += blockDim.x) out[rowoff + j] = y[j];
        return;
    }
    const bool masked = row_mask != nullptr && row_mask[fe] == 0;
    const float *S = meas + rowoff;
    if (mode == FWD_MSE) {
        double part = 0.0;
        for (int j = threadIdx.x; j < nt; j += blockDim.x) {
            const float d = y[j] - __ldg(S + j);
            part += (double)d * (double)d;
            out[rowoff + j] = masked ? 0.0f : 2.0f * d;
        }
        const double tot = block_sum(part, red);
        if (threadIdx.x == 0) rowloss[fe] = masked ? 0.0 : tot;
        return;
    }
    double sy = 0.0, ss = 0.0;
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        sy += y[j];
        ss += __ldg(S + j);
    }
    const double my = block_sum(sy, red) / nt, ms = block_sum(ss, red) / nt;
    double cv = 0.0, vy = 0.0, vs = 0.0;
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        const double a = y[j] - my, b = (double)__ldg(S + j) - ms;
        cv += a * b;
        vy += a * a;
        vs += b * b;
    }
    const double COV = block_sum(cv, red) / nt, VY = block_sum(vy, red) / nt, VS = block_sum(vs, red) / nt;
    const double sdy = sqrt(VY), sds = sqrt(VS);
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        const double gj = -(((double)__ldg(S + j) - ms) / (sdy * sds) - COV * (y[j] - my) / (sdy * sdy * sdy * sds)) / nt;
        out[rowoff + j] = masked ? 0.0f : (float)gj;
    }
    if (threadIdx.x == 0) rowloss[fe] = masked ? 0.0 : -COV / (sdy * sds);
}

// (Pairs of channels as one 64-bit shared-memory add — red.shared.add.u64, exact with a borrow-aware split —
// measured 2.9x slower on B200: 368 vs 126 ms per 16 C4 frames.  Not taken.)
// Unpredicated shared-memory integer add (ATOMS.ADD, no return value) at addr + OFF: a predicated
// red is turned into a branch per atomic by ptxas, so lanes without a deposit add 0 to a per-lane
// dummy word instead.
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
// one 256-bit read-only global load (LDG.E.ENL2.256, sm_100): 8 consecutive floats, 32-B aligned
__device__ __forceinline__ void ldg256(const float *p, float v[8])
{
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p));
}
__device__ __forceinline__ float rcp_approx(float x)  // the reciprocal of __fdividef (div.approx = a * rcp(b))
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int OFF>
__device__ __forceinline__ void red_s32(unsigned addr, int v)
{
    asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(addr), "r"(v), "n"(OFF) : "memory");
}
template <int OFF>
__device__ __forceinline__ void red_one(unsigned addr)  // the deposit count (PA_DEP_CNT)
{
    asm volatile("red.shared.add.u32 [%0+%1], 1;" ::"r"(addr), "n"(OFF) : "memory");
}
#if PA_DEP_CNT
#define DEPV(x) __float_as_int(x)  // raw shifter bits; the flush subtracts count x 0x4B400000
#else
#define DEPV(x) (__float_as_int(x) - 0x4B400000)
#endif

#ifndef PA_DEP_MINB
#define PA_DEP_MINB 3  // resident CTAs per SM of the 8-warp K1d (<= 80 registers, no spills; 2: 128 registers, 4.5% slower at C4)
#endif
template <int RK, int NW, int NG, int TPR_>
__global__ void __launch_bounds__(NW * 32, NW == 8 ? PA_DEP_MINB : 1) k_fwd_dep(Geo g, DepConst dc, const float *__restrict__ poses,
                                                                       const float *__restrict__ tmpl,
                                                                       const float *__restrict__ p0,
                                                                       const unsigned *__restrict__ pmax_bits,
                                                                       float *__restrict__ out, int mode,
                                                                       const float *__restrict__ meas,
                                                                       const uint8_t *__restrict__ row_mask,
                                                                       double *__restrict__ rowloss)
{
    using C = DepCfg<RK, NW, NG, TPR_>;
    constexpr int R = C::R, CS = C::CS, CF = C::CF, NQ = C::NQ, G = C::G;
    extern __shared__ int smi[];
    const int LMIN = g.lmin;  // runtime window length L_min
    const int NJ = C::njp(g.nt, LMIN), NR = dc.nr;
    const unsigned nrm = dc.nrm;
    int *Qi = smi;                                         // [NR][CS] fixed-point round accumulators (ring: pos & nrm)
    float *Qf = reinterpret_cast<float *>(smi + CS * NR);  // [NJ][CF] fp32 row accumulators
    __shared__ int rng[2][2];
    __shared__ double red[NW * 32];
    __shared__ int dummy[32 + C::CS];  // target of lanes without a deposit (adds 0)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < CS * NR + CF * NJ; i += blockDim.x) smi[i] = 0;
    if (tid < 2) {
        rng[tid][0] = 0x7fffffff;
        rng[tid][1] = -1;
    }
    const int fe = blockIdx.x;
    const int f = fe / g.E, e = fe - f * g.E;
    double x[3];
    elem_pos(poses, tmpl, f, e, x);
    // r_min: distance from the element to the nearest voxel centre (nearest lattice point, clamped)
    float rmin;
    {
        const double o[3] = {g.ox, g.oy, g.oz};
        const int n[3] = {g.nx, g.ny, g.nz};
        double d2 = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            double i = rint((x[q] - o[q]) / g.h);
            i = i < 0.0 ? 0.0 : (i > n[q] - 1 ? (double)(n[q] - 1) : i);
            const double d = x[q] - (o[q] + g.h * i);
            d2 += d * d;
        }
        rmin = (float)(sqrt(d2) * (1.0 - 1e-6));
    }
    const float pm = __uint_as_float(__ldg(pmax_bits));
    const float invP = pm > 0.0f ? 1.0f / pm : 0.0f;
    // lane l's voxels of a tile: (bx + vx, by + dyv(v), bz + dzv(v)), v = 0..7, vx = v & 1 (the packed pair).
    // PA_DEP_MAP 1 puts the 32 lanes of one deposit instruction on all 4 z planes of the tile (8 lanes
    // each) instead of 2 (16 each): more distinct window positions per instruction, fewer same-word atomics.
    // PA_DEP_MAP 2: a warp slot covers two z-adjacent tiles (lanes 0-15: tile 2 tzp, 16-31: 2 tzp + 1)
    // and half of their y rows (hh = slot parity): 8 z planes, 4 lanes each, per deposit instruction;
    // the anchor of a tile is computed once for both halves.
    constexpr bool PAIR = PA_DEP_MAP == 2;
#if PA_DEP_MAP == 2
    const int bx = 2 * (lane & 3), by = 0, bz = (lane >> 2) & 3, half = lane >> 4;
    auto dyv = [](int v) { return v >> 1; };
    auto dzv = [](int) { return 0; };
#elif PA_DEP_MAP == 1
    const int bx = 2 * (lane & 3), by = 4 * ((lane >> 2) & 1), bz = lane >> 3, half = 0;
    auto dyv = [](int v) { return v >> 1; };
    auto dzv = [](int) { return 0; };
#else
    const int bx = 2 * (lane & 3), by = 2 * ((lane >> 2) & 3), bz = 2 * (lane >> 4), half = 0;
    auto dyv = [](int v) { return (v >> 1) & 1; };
    auto dzv = [](int v) { return v >> 2; };
#endif
    // rounds: NW tiles in a 2 x 2 x (NW/4) tile block, x fastest
    // a round = TPR tiles per warp: NW TPR tiles in a 2 x 2 x (NW TPR / 4) tile block, x fastest
    constexpr int TPR = C::TPR, BZ = NW / 4;
    constexpr int TPRT = PAIR ? TPR / 2 : TPR;  // tiles (pairs) per warp per round
    static_assert(!PAIR || TPR % 2 == 0, "paired tiles need an even slot count per round");
    const int ntzu = PAIR ? (g.ntz + 1) >> 1 : g.ntz;  // z units (tile pairs)
    const int nbx = (g.ntx + 1) >> 1, nby = (g.nty + 1) >> 1, nbz = (ntzu + BZ * TPRT - 1) / (BZ * TPRT);
    const int nb = nbx * nby * nbz, nslot = nb * TPR;
    const int spanlo = (int)floorf((-g.rt - g.ksig) * g.inv_a) - 2, spanhi = (int)ceilf((g.rt - g.ksig) * g.inv_a) + 3;
    const unsigned qbase = (unsigned)__cvta_generic_to_shared(Qi) + 4u * NQ * (unsigned)(lane % G);  // this lane's copy
    const unsigned dbase = (unsigned)__cvta_generic_to_shared(dummy) + 4u * lane;
    __syncthreads();

    // the next tile of this warp, advanced incrementally (slot q: round b = q / TPR, k = q % TPR;
    // rounds run over 2 x 2 x (BZ TPR) tile blocks, x fastest) — no integer division per tile
    int nk = 0, nbx_ = 0, nby_ = 0, nbz_ = 0, hh_ = 0, ptx = 0, pty = 0, ptz = 0;
    auto next_tile = [&](int &tx, int &ty, int &tz, int &hh) {
        if (!PAIR || hh_ == 0) {
            ptx = 2 * nbx_ + (warp & 1);
            pty = 2 * nby_ + ((warp >> 1) & 1);
            ptz = BZ * (TPRT * nbz_ + nk) + (warp >> 2);
            if (++nk == TPRT) {
                nk = 0;
                if (++nbx_ == nbx) {
                    nbx_ = 0;
                    if (++nby_ == nby) {
                        nby_ = 0;
                        ++nbz_;
                    }
                }
            }
        }
        tx = ptx;
        ty = pty;
        tz = PAIR ? 2 * ptz + half : ptz;  // this lane's tile
        hh = PAIR ? hh_ : 0;
        if (PAIR) hh_ ^= 1;
        return tx < g.ntx && ty < g.nty && tz < g.ntz;
    };
    // the lane's voxel amplitudes of a tile (0 outside the grid): one 64-bit base per tile (volumes of
    // >= 2^31 voxels), 32-bit in-tile offsets (a z-plane of < 2^30 voxels, checked on the host), the tile's
    // edge tests once
    const int sy = g.nx, sz = g.nx * g.ny;
    auto load_p = [&](int tx, int ty, int tz, int hh, bool ok, float P[8]) {
        const int ix0 = TX * tx + bx, iy0 = TY * ty + by + 4 * hh, iz0 = TZ * tz + bz;
        const bool ok0 = ok && ix0 < g.nx && iy0 < g.ny && iz0 < g.nz;
        const bool okx1 = ix0 + 1 < g.nx, okz1 = iz0 + 1 < g.nz;
        const int ny_left = g.ny - iy0;  // rows of the lane's y run inside the grid
        const float *pb = p0 + (ok0 ? ((size_t)iz0 * (size_t)sz + (size_t)(iy0 * sy + ix0)) : (size_t)0);
#if PA_DEP_MAP == 2 && PA_DEP_FASTLOAD
        // the common case: all 8 voxels inside and an even row pitch (the x-pair 8-B aligned: ix0 is even) ->
        // four unpredicated 64-bit loads along the lane's 4 rows
        if (ok0 && okx1 && ny_left >= 4 && (sy & 1) == 0) {
            const float2 *q = reinterpret_cast<const float2 *>(pb);
            const int s2 = sy >> 1;
            const float2 v0 = __ldg(q), v1 = __ldg(q + s2), v2 = __ldg(q + 2 * s2), v3 = __ldg(q + 3 * s2);
            P[0] = v0.x; P[1] = v0.y; P[2] = v1.x; P[3] = v1.y;
            P[4] = v2.x; P[5] = v2.y; P[6] = v3.x; P[7] = v3.y;
            return;
        }
#endif
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            const int vx = v & 1, vy = dyv(v), vz = dzv(v);
            const bool in = ok0 && (vx == 0 || okx1) && vy < ny_left && (vz == 0 || okz1);
            P[v] = in ? __ldg(pb + (vx + vy * sy + vz * sz)) : 0.0f;
        }
    };
    int ntx_ = 0, nty_ = 0, ntz_ = 0, nhh_ = 0;
    bool nok = nslot > 0 && next_tile(ntx_, nty_, ntz_, nhh_);
    float Pn[8];
    load_p(ntx_, nty_, ntz_, nhh_, nok, Pn);
    Anc A;  // the lane's tile anchor (PAIR: kept for the second half of the tile pair)
#if PA_DEP_UNROLL2 == 4
#pragma unroll 4
#elif PA_DEP_UNROLL2
#pragma unroll 2
#endif
    for (int q = 0; q < nslot; ++q) {
        const int b = q / TPR;
        const int tx = ntx_, ty = nty_, tz = ntz_, hh = nhh_;
        const bool tok = nok;
#if PA_DEP_LATEPF
        float *P = Pn;  // this slot's amplitudes; the next slot's are loaded after its deposits (no copy)
#else
        float P[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) P[v] = Pn[v];
        // software pipeline: the next tile's amplitudes are in flight during this one
        nok = q + 1 < nslot && next_tile(ntx_, nty_, ntz_, nhh_);
        load_p(ntx_, nty_, ntz_, nhh_, nok, Pn);
#endif
        if (PAIR ? __any_sync(0xffffffffu, tok) : tok) {
            if (hh == 0) A = make_anchor(g, x, tx, ty, tok ? tz : 0);
            const bool live = tok && !A.cull;
            if (PAIR ? __any_sync(0xffffffffu, live) : live) {
                const int base = A.JA + LMIN + (int)floorf(A.CA * g.inv_a);
                const bool leader = PAIR ? (lane & 15) == 0 : lane == 0;  // one lane per tile
                if (leader && live && hh == 0) {
                    atomicMin(&rng[b & 1][0], max(base + spanlo, 0));
                    atomicMax(&rng[b & 1][1], min(base + spanhi, NJ - 1));
                }
                // voxel offsets from the tile centre: the same expression as every other kernel (R17)
                const float2 ex = make_float2(((float)bx - 0.5f * (TX - 1)) * g.hf, ((float)(bx + 1) - 0.5f * (TX - 1)) * g.hf);
                const float posA = (float)(A.JA + LMIN);
                const float2 tCA = f2(__fmaf_rn(A.CA, dc.tA, dc.tC));
                // two voxels (vx = 0, 1) per pass in packed fp32x2 (FFMA2/FMUL2/FADD2: half the issue
                // slots); every scalar step below is the same operation as pair() (R17)
                const int pbase = A.JA + LMIN - 0x4B400000;  // position = pbase + bits(ceil shifter)
#pragma unroll
                for (int v = 0; v < 8; v += 2) {
                    const float2 Pv = make_float2(P[v], P[v + 1]);
                    const float ey = ((float)(by + 4 * hh + dyv(v)) - 0.5f * (TY - 1)) * g.hf;
                    const float ez = ((float)(bz + dzv(v)) - 0.5f * (TZ - 1)) * g.hf;
                    const float2 e2 = __ffma2_rn(ex, ex, f2(__fmaf_rn(ey, ey, __fmul_rn(ez, ez))));
                    const float2 num = __ffma2_rn(f2(A.dx2), ex, __ffma2_rn(f2(A.dy2), f2(ey), __ffma2_rn(f2(A.dz2), f2(ez), e2)));
                    const float2 r2 = __fadd2_rn(f2(A.rho2), num);
                    const float2 inv_r = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
                    const float2 den = __fadd2_rn(__fmul2_rn(r2, inv_r), f2(A.rho));
                    const float2 drel = __fmul2_rn(num, make_float2(rcp_approx(den.x), rcp_approx(den.y)));
                    const float2 bse = __fadd2_rn(drel, f2(A.CA));
                    const float2 xlo = __fmul2_rn(__fadd2_rn(bse, f2(-g.ksig)), f2(g.inv_a));
                    const float2 xhi = __fmul2_rn(__fadd2_rn(bse, f2(g.ksig)), f2(g.inv_a));
                    // ceil(xlo) = the round-up sum with the 1.5 2^23 shifter (exact for |xlo| < 2^22; == ceilf)
                    const float shx = __fadd_ru(xlo.x, 12582912.0f), shy = __fadd_ru(xlo.y, 12582912.0f);
                    const float2 clof = __fadd2_rn(make_float2(shx, shy), f2(-12582912.0f));
                    const float2 cl2 = __fadd2_rn(clof, f2((float)LMIN));
                    const bool Lxx = xhi.x >= cl2.x, Lxy = xhi.y >= cl2.y;  // floor(xhi) - clo + 1 >= LMIN + 1
                    const int posx = pbase + __float_as_int(shx), posy = pbase + __float_as_int(shy);  // j_m + OFF = jlo + LMIN
                    // (a zero amplitude deposits zeros: no test; a window outside the row deposits nowhere)
                    const bool vax = live && (unsigned)posx < (unsigned)NJ;
                    const bool vay = live && (unsigned)posy < (unsigned)NJ;
                    // t = (D_m - Dc)/Dw, D_m = bse - clo a - MA a
                    const float2 t = __ffma2_rn(clof, f2(-dc.tB), __ffma2_rn(drel, f2(dc.tA), tCA));
                    const float2 s2 = __fmul2_rn(t, t);
                    float2 rlo = __ffma2_rn(__fadd2_rn(clof, f2(posA)), f2(g.af), f2(dc.W0));
                    rlo.x = fmaxf(rmin, rlo.x);
                    rlo.y = fmaxf(rmin, rlo.y);
                    float2 ct = __fmul2_rn(__fmul2_rn(__fmul2_rn(Pv, f2(invP)), rlo), inv_r);
                    ct.x = vax ? ct.x : 0.0f;
                    ct.y = vay ? ct.y : 0.0f;
                    const float2 o0 = __fmul2_rn(ct, t);  // odd channels: c t phi_m(t) = (c t) (c0 + s c1 + s^2 c2 + s^3 c3)
                    // a lane without a deposit (ct = 0: every word 0) adds to its dummy words
                    const unsigned sax = vax ? qbase + ((unsigned)posx & nrm) * (CS * 4) : dbase;
                    const unsigned say = vay ? qbase + ((unsigned)posy & nrm) * (CS * 4) : dbase;
                    // phi_m by Horner in s = t^2 (3 FFMA2), then x (c or c t) with the 1.5 2^23 shifter riding in
                    // the last FFMA2: each deposit rounds to an integer (quantisation <= 2 units on a channel <= 8%
                    // of the trace)
                    auto poly = [&](int m) {
                        return __ffma2_rn(__ffma2_rn(__ffma2_rn(dc.cf2[m][3], s2, dc.cf2[m][2]), s2, dc.cf2[m][1]), s2, dc.cf2[m][0]);
                    };
                    {  // channel 0: two words, |x| <= 2^NB0 = hi 2^10 + lo, quantum far below fp32 rounding
                        const float2 xm = __fmul2_rn(poly(0), ct);
                        const float2 hs = __ffma2_rn(xm, f2(1.0f / 1024.0f), f2(12582912.0f));
                        const float2 ls = __fadd2_rn(__ffma2_rn(__fadd2_rn(hs, f2(-12582912.0f)), f2(-1024.0f), xm), f2(12582912.0f));
                        red_s32<0>(sax, DEPV(hs.x));
                        red_s32<0>(say, DEPV(hs.y));
                        red_s32<4 * (R + 1)>(sax, DEPV(ls.x));
                        red_s32<4 * (R + 1)>(say, DEPV(ls.y));
#if PA_DEP_CNT
                        red_one<4 * (R + 2)>(sax);
                        red_one<4 * (R + 2)>(say);
#endif
                    }
                    auto chan = [&](auto mc) {
                        constexpr int m = decltype(mc)::value;
                        const float2 xm = __ffma2_rn(poly(m), (m & 1) ? o0 : ct, f2(12582912.0f));
                        red_s32<4 * m>(sax, DEPV(xm.x));
                        red_s32<4 * m>(say, DEPV(xm.y));
                    };
                    chan(std::integral_constant<int, 1>{});
                    chan(std::integral_constant<int, 2>{});
                    chan(std::integral_constant<int, 3>{});
                    if constexpr (R > 4) chan(std::integral_constant<int, 4>{});
                    if constexpr (R > 5) chan(std::integral_constant<int, 5>{});
                    if constexpr (R > 6) chan(std::integral_constant<int, 6>{});
                    static_assert(R >= 4 && R <= 7, "rank 4 to 7");
                    {  // X: the optional last tap (L = LMIN + 1), a cubic in t by Horner
                        const float2 cx = make_float2(Lxx ? ct.x : 0.0f, Lxy ? ct.y : 0.0f);
                        const float2 px = __ffma2_rn(__ffma2_rn(__ffma2_rn(dc.cf2[R][3], t, dc.cf2[R][2]), t, dc.cf2[R][1]), t, dc.cf2[R][0]);
                        const float2 xm = __ffma2_rn(px, cx, f2(12582912.0f));
                        red_s32<4 * R>(sax, DEPV(xm.x));
                        red_s32<4 * R>(say, DEPV(xm.y));
                    }
                }
            }
        }
#if PA_DEP_LATEPF
        nok = q + 1 < nslot && next_tile(ntx_, nty_, ntz_, nhh_);
        load_p(ntx_, nty_, ntz_, nhh_, nok, Pn);
#endif
        if (q - b * TPR != TPR - 1) continue;  // flush after the round's last tile
        __syncthreads();
        {
            const int lo = rng[b & 1][0], hi = rng[b & 1][1];  // lo > hi when every tile was culled
            for (int p = (lo <= hi ? lo : hi + 1) + tid; p <= hi; p += blockDim.x) {
                int *qi = Qi + (int)((unsigned)p & nrm) * CS;
                float *qf = Qf + p * CF;
                int n[NQ];
#pragma unroll
                for (int c = 0; c < NQ; ++c) n[c] = qi[c];
#pragma unroll
                for (int k = 1; k < G; ++k)
#pragma unroll
                    for (int c = 0; c < NQ; ++c) n[c] += qi[k * NQ + c];  // all copies together < 2^30: no overflow
#if PA_DEP_CNT
#pragma unroll
                for (int c = 0; c < R + 2; ++c) n[c] = (int)((unsigned)n[c] - (unsigned)n[R + 2] * 0x4B400000u);
#endif
                qf[0] += __fmaf_rn((float)n[0], 1024.0f, (float)n[R + 1]);
#pragma unroll
                for (int c = 1; c <= R; ++c) qf[c] += (float)n[c];
#pragma unroll
                for (int c = 0; c < G * NQ; ++c) qi[c] = 0;
            }
            if (tid < 1) {
                rng[(b + 1) & 1][0] = 0x7fffffff;
                rng[(b + 1) & 1][1] = -1;
            }
        }
        __syncthreads();
    }
    // decode: Q_m[pos] = Qf * (0.5 / S_m) * Pmax / r_lo(pos)
    for (int p = tid; p < NJ; p += blockDim.x) {
        const float rr = pm / fmaxf(rmin, __fmaf_rn((float)p, g.af, dc.W0));
#pragma unroll
        for (int m = 0; m < CF; ++m) Qf[p * CF + m] = (Qf[p * CF + m] * dc.dec[m]) * rr;  // no denormal intermediate for tiny Pmax
    }
    __syncthreads();
    float *y = reinterpret_cast<float *>(Qi);  // the round accumulators are free now
    for (int j = tid; j < g.nt; j += blockDim.x) {
        float acc = Qf[j * CF + R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const float *qm = Qf + j * CF + m;
            float am = 0.0f;
#pragma unroll 8
            for (int q = 1; q <= LMIN; ++q) am = __fmaf_rn(qm[q * CF], dc.psi[m][q - 1], am);  // runtime L_min
            acc += am;
        }
        y[j] = acc;
    }
    __syncthreads();
    fwd_epilogue(g, y, fe, out, mode, meas, row_mask, rowloss, red);
}

// ============================================================================================
// K2c — the moment-filter adjoint (a4 + a5) with two voxels per thread in packed fp32x2.
//
// Per (voxel, element): the window of pair() (every step bit-identical; ceil by a round-up add of the
// 1.5 2^23 shifter; L_min is the runtime Geo::lmin), the Taylor moments S_n = sum_m dl^m/m! F_{n+m}[j_m]
// from the L2-resident per-row filter records (one 256-bit load per voxel, the last tap included),
// A1 = u_m (D_m S0 - a S1) and Bq / s^2 = u_m ((D_m^2/s^2 - 1) S0 - (2a/s^2) D_m S1 + (a^2/s^2) S2) (the
// filters carry the 1/2 of D/(2r)).  A thread owns voxels z and z + 2 of an 8x8x4 anchor tile (a CTA =
// one tile of 128 threads, or two stacked in z: PA_ADJ_TPC), so the geometry, the series and the gradient terms of the
// two voxels run as FFMA2/FMUL2/FADD2, the anchor is read once for both, and their element-gradient
// terms are summed before the warp reduction.  No per-pair validity logic: zero-padded filter rows, a
// sentinel anchor for culled / padding elements, amplitude 0 for voxels outside the grid.
// ============================================================================================
struct AncT {  // anchor of K2c / K2s in shared memory (8 words: two 128-bit loads)
    float dx, dy, dz, rho, rho2, CA;
    int JAp;   // JA + L_min + PADL: the record index of the window is JAp + clo
    int pad;
};

// the shared anchor of (tile, element), or the sentinel of a culled / padding element whose record
// index lands in the leading zero padding of the row
__device__ __forceinline__ AncT make_anct(const Geo &g, const Anc &A, bool culled, int padl, int sentinel)
{
    AncT s;
    s.dx = A.dx;
    s.dy = A.dy;
    s.dz = A.dz;
    s.rho = A.rho;
    s.rho2 = A.rho2;
    s.CA = A.CA;
    s.JAp = culled ? sentinel : A.JA + g.lmin + padl;
    s.pad = 0;
    return s;
}

template <int NF>
struct Tay2A {
    float Fa[NF], Fb[NF];  // records of voxel a (.x) and voxel b (.y), straight from the loads
    float2 Dm, inv_r, dz;
    float dx, dy;
    bool La, Lb;  // the window has the last tap (L = L_min + 1)
};

template <int NF>
__device__ __forceinline__ Tay2A<NF> tay2_stage_a(const Geo &g, const AncT *anc, int e, float ex2x, float ey2x,
                                                  float2 ez2x, float2 e2, float2 ez, const float *__restrict__ Frow)
{
    Tay2A<NF> o;
    const AncT sa = anc[e];
    // num = 2 d.delta + |delta|^2 exactly as pair(): fma(2dx, ex, ...) == fma(dx, 2ex, ...) (exact doubling)
    const float2 num = __ffma2_rn(f2(sa.dx), f2(ex2x), __ffma2_rn(f2(sa.dy), f2(ey2x), __ffma2_rn(f2(sa.dz), ez2x, e2)));
    const float2 r2 = __fadd2_rn(f2(sa.rho2), num);
    const float2 inv_r = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
    const float2 den = __fadd2_rn(__fmul2_rn(r2, inv_r), f2(sa.rho));
    const float2 drel = __fmul2_rn(num, make_float2(rcp_approx(den.x), rcp_approx(den.y)));
    const float2 bse = __fadd2_rn(drel, f2(sa.CA));
    const float2 xlo = __fmul2_rn(__fadd2_rn(bse, f2(-g.ksig)), f2(g.inv_a));
    const float2 xhi = __fmul2_rn(__fadd2_rn(bse, f2(g.ksig)), f2(g.inv_a));
    // ceil(xlo) = the round-up sum with the 1.5 2^23 shifter (exact for |xlo| < 2^22; == ceilf)
    const float sha = __fadd_ru(xlo.x, 12582912.0f), shb = __fadd_ru(xlo.y, 12582912.0f);
    const float2 clof = __fadd2_rn(make_float2(sha, shb), f2(-12582912.0f));
    // record indices; the unsigned clamp only guards memory against non-finite (degenerate, R10) geometry
    const unsigned ja = min((unsigned)(sa.JAp + (__float_as_int(sha) - 0x4B400000)), g.njp_m1);
    const unsigned jb = min((unsigned)(sa.JAp + (__float_as_int(shb) - 0x4B400000)), g.njp_m1);
    const float2 cl2 = __fadd2_rn(clof, f2((float)g.lmin));
    o.La = xhi.x >= cl2.x;  // floor(xhi) - clo + 1 >= L_min + 1
    o.Lb = xhi.y >= cl2.y;
    if constexpr (NF == 8) {  // one 256-bit load per voxel (32-B records)
        ldg256(Frow + (size_t)ja * NF, o.Fa);
        ldg256(Frow + (size_t)jb * NF, o.Fb);
    } else {  // 48-B records: 128-bit loads
#pragma unroll
        for (int r = 0; r < NF / 4; ++r) {
            const float4 u4 = __ldg(reinterpret_cast<const float4 *>(Frow + (size_t)ja * NF) + r);
            const float4 w4 = __ldg(reinterpret_cast<const float4 *>(Frow + (size_t)jb * NF) + r);
            o.Fa[4 * r] = u4.x; o.Fa[4 * r + 1] = u4.y; o.Fa[4 * r + 2] = u4.z; o.Fa[4 * r + 3] = u4.w;
            o.Fb[4 * r] = w4.x; o.Fb[4 * r + 1] = w4.y; o.Fb[4 * r + 2] = w4.z; o.Fb[4 * r + 3] = w4.w;
        }
    }
    o.Dm = __fadd2_rn(__ffma2_rn(clof, f2(-g.af), bse), f2(-(float)g.mA * g.af));
    o.inv_r = inv_r;
    o.dx = sa.dx + 0.5f * ex2x;  // d + delta (x, y shared by the two voxels)
    o.dy = sa.dy + 0.5f * ey2x;
    o.dz = __fadd2_rn(f2(sa.dz), ez);
    return o;
}

// A1 / 2 and Bq / (2 s^2) of the two voxels
template <int NF, bool POSE>
__device__ __forceinline__ void tay2_stage_b(const Geo &g, const TayConst &tc, const Tay2A<NF> &a, float2 &A1,
                                             float2 &Bq)
{
    constexpr int NPS = TayCfg<NF>::NPS;
    const float KT = (float)(g.lmin - g.mA);  // the optional last tap k_t = L_min - MA
    const float2 Dm = a.Dm;
    const float2 dl = __ffma2_rn(f2(tc.lam_s), Dm, f2(-tc.lam0));
    // P, P', P''/2 at dl by Horner with synthetic division, in scalar FFMAs straight on the loaded
    // registers (packing the two voxels' values would cost a register move per value)
    float ba = a.Fa[NPS - 1], bb = a.Fb[NPS - 1], d1a = 0.0f, d1b = 0.0f, d2a = 0.0f, d2b = 0.0f;
#pragma unroll
    for (int p = NPS - 2; p >= 0; --p) {
        if (POSE) {
            if (p <= NPS - 4) {
                d2a = __fmaf_rn(d2a, dl.x, d1a);
                d2b = __fmaf_rn(d2b, dl.y, d1b);
            } else if (p == NPS - 3) {
                d2a = d1a;
                d2b = d1b;
            }
        }
        if (p <= NPS - 3) {
            d1a = __fmaf_rn(d1a, dl.x, ba);
            d1b = __fmaf_rn(d1b, dl.y, bb);
        } else {
            d1a = ba;
            d1b = bb;
        }
        ba = __fmaf_rn(ba, dl.x, a.Fa[p]);
        bb = __fmaf_rn(bb, dl.y, a.Fb[p]);
    }
    float2 S[3] = {make_float2(ba, bb), make_float2(d1a, d1b), make_float2(d2a, d2b)};  // S[2] = S2 / 2
    // the last tap (record slot NF - 1 = g C_k(k_t) / 2), in the window iff L = L_min + 1
    const float2 ea = __fmul2_rn(Dm, f2(g.two_a_k2 * KT));
    const float2 gx = make_float2(a.La ? a.Fa[NF - 1] : 0.0f, a.Lb ? a.Fb[NF - 1] : 0.0f);
    const float2 w = __fmul2_rn(gx, make_float2(ex2(ea.x), ex2(ea.y)));
    S[0] = __fadd2_rn(S[0], w);
    S[1] = __ffma2_rn(w, f2(KT), S[1]);
    const float2 q = __fmul2_rn(Dm, Dm);
    const float2 kq = __fmul2_rn(f2(-g.k2), q);
    const float2 um = make_float2(ex2(kq.x), ex2(kq.y));
    A1 = __fmul2_rn(um, __ffma2_rn(f2(-g.af), S[1], __fmul2_rn(Dm, S[0])));
    Bq = f2(0.0f);
    if (POSE) {
        S[2] = __ffma2_rn(w, f2(0.5f * KT * KT), S[2]);
        // (D^2/s^2 - 1) S0 - (2a/s^2) D S1 + (a^2/s^2) S2, with S[2] = S2 / 2 and c_aa = 2 a^2/s^2
        const float2 b = __ffma2_rn(f2(tc.c_aa), S[2],
                                    __ffma2_rn(__fmul2_rn(f2(tc.c_a), Dm), S[1], __fmul2_rn(__ffma2_rn(q, f2(g.inv_s2), f2(-1.0f)), S[0])));
        Bq = __fmul2_rn(um, b);
    }
}

#ifndef PA_TAY_EUNROLL
#define PA_TAY_EUNROLL 2  // K2c element-loop unroll (32-B records)
#endif
#ifndef PA_ADJ_TPC
// K2c tiles per CTA: 1 (128 threads, 4 CTAs/SM at 128 registers: C4 105.8 ms per 16 frames) or 2 (256
// threads, 2 CTAs/SM: 107.2 ms).  Measured with 1 tile per CTA: 5 CTAs/SM (96 registers, 16 B spills)
// 106.3 ms, 6 CTAs/SM (80 registers) 106.4 ms — more resident warps do not pay.
#define PA_ADJ_TPC 1
#endif
#ifndef PA_ADJ_MINB
#define PA_ADJ_MINB (PA_ADJ_TPC == 2 ? 2 : 4)  // resident CTAs per SM of K2c
#endif
constexpr int TAY_NT = 128 * PA_ADJ_TPC;  // K2c threads per CTA
template <int NF, bool POSE, bool ADJ>
__global__ void __launch_bounds__(TAY_NT, PA_ADJ_MINB) k_adjoint_tay2(Geo g, TayConst tc, const float *__restrict__ poses,
                                                                const float *__restrict__ tmpl,
                                                                const float *__restrict__ p0,
                                                                const float *__restrict__ Fg,
                                                                float *__restrict__ grad_p0,
                                                                float *__restrict__ partial, int f0, int fn, int njp,
                                                                int padl, int sentinel)
{
    extern __shared__ float sm[];
    const int E = g.E, F = g.F;
    const int E4 = (E + 3) & ~3;                           // elements padded to the unroll of 4 (sentinels)
    constexpr int TPC = PA_ADJ_TPC, NT = TAY_NT;
    AncT *anc = reinterpret_cast<AncT *>(sm);               // [TPC][E4]: the tiles of the CTA
    float *wred = reinterpret_cast<float *>(anc + TPC * E4); // [NT/32][E][3]
    float *gacc = wred + (NT / 32) * E * 3;                  // [fn][E][3]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int half = TPC == 2 ? tid >> 7 : 0, u = tid & 127;
    const int lx = u & 7, ly = (u >> 3) & 7, lzp = u >> 6;  // voxels (lx, ly, lzp) and (lx, ly, lzp + 2)
    const float ex = ((float)lx - 0.5f * (TX - 1)) * g.hf;
    const float ey = ((float)ly - 0.5f * (TY - 1)) * g.hf;
    const float2 ez = make_float2(((float)lzp - 0.5f * (TZ - 1)) * g.hf, ((float)(lzp + 2) - 0.5f * (TZ - 1)) * g.hf);
    // e2 exactly as pair(): fma(ex, ex, fma(ey, ey, ez * ez))
    const float2 e2 = __ffma2_rn(f2(ex), f2(ex), __ffma2_rn(f2(ey), f2(ey), __fmul2_rn(ez, ez)));
    const float ex2x = 2.0f * ex, ey2x = 2.0f * ey;
    const float2 ez2x = __fmul2_rn(f2(2.0f), ez);
    const AncT *anch = anc + half * E4;
    const int ntzp = TPC == 2 ? (g.ntz + 1) >> 1 : g.ntz, ntp = g.ntx * g.nty * ntzp;

    if (POSE) {
        for (int q = tid; q < fn * E * 3; q += NT) gacc[q] = 0.0f;
    }
    for (int tp = blockIdx.x; tp < ntp; tp += gridDim.x) {
        const int tx = tp % g.ntx, ty = (tp / g.ntx) % g.nty, tzp = tp / (g.ntx * g.nty);
        const int tz = TPC * tzp + half;
        const int ix = TX * tx + lx, iy = TY * ty + ly, iza = TZ * tz + lzp, izb = iza + 2;
        const bool ina = ix < g.nx && iy < g.ny && iza < g.nz, inb = ix < g.nx && iy < g.ny && izb < g.nz;
        const size_t ka = ((size_t)iza * g.ny + iy) * g.nx + ix, kb = ka + 2 * (size_t)g.nx * g.ny;
        // amplitude 0 outside the grid: those voxels add nothing to the element gradient
        const float2 P = make_float2((POSE && ina) ? __ldg(p0 + ka) : 0.0f, (POSE && inb) ? __ldg(p0 + kb) : 0.0f);
        float2 z = f2(0.0f);
        for (int fl = 0; fl < fn; ++fl) {
            const int f = f0 + fl;
            __syncthreads();  // previous frame's anchors / wred consumed
            for (int q = tid; q < TPC * E4; q += NT) {
                const int hh = q / E4, e = q - hh * E4;
                const int tzh = TPC * tzp + hh;
                Anc A;
                bool culled = true;
                if (e < E) {
                    double x[3];
                    elem_pos(poses, tmpl, f, e, x);
                    A = make_anchor(g, x, tx, ty, tzh < g.ntz ? tzh : 0);
                    culled = A.cull || tzh >= g.ntz;
                } else {
                    A.dx = A.dy = A.dz = A.rho = A.rho2 = A.CA = 0.0f;
                    A.rho2 = 1.0f;  // finite geometry for the padding sentinels
                    A.rho = 1.0f;
                    A.JA = 0;
                }
                anc[q] = make_anct(g, A, culled, padl, sentinel);
            }
            __syncthreads();
            // per-element record rows advanced incrementally (stage A runs one element ahead; rows past
            // E - 1 stay on the last row, their sentinel anchors read its zero padding)
            const float *Frow = Fg + (size_t)fl * E * njp * NF;
            const size_t fstep = (size_t)njp * NF;
            Tay2A<NF> cur = tay2_stage_a<NF>(g, anch, 0, ex2x, ey2x, ez2x, e2, ez, Frow);
            // two 4-element batches per iteration for the 32-B records (C4 -2.2%, C2 -2.0%; 48-B records: +1.2%, one)
            constexpr int EU = NF == 8 ? PA_TAY_EUNROLL : 1;
#pragma unroll EU
            for (int e0 = 0; e0 < E; e0 += 4) {
                float G[4][3];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = e0 + q;
                    if (e + 1 < E) Frow += fstep;
                    const Tay2A<NF> nxt = tay2_stage_a<NF>(g, anch, min(e + 1, E4 - 1), ex2x, ey2x, ez2x, e2, ez, Frow);
                    float2 A1, Bq;
                    tay2_stage_b<NF, POSE>(g, tc, cur, A1, Bq);
                    const float2 ir = cur.inv_r;
                    if (ADJ) z = __ffma2_rn(A1, ir, z);
                    if (POSE) {
                        // dL/dr = P/(2r) (-Bq/s^2 - A1/r);  G += -dL/dr (d + delta)/r  (x - y_k = -(d + delta)):
                        // with the halved moments, -dL/dr / r = P ir^2 (Bq'/s^2 + A1' ir)
                        const float2 sc = __fmul2_rn(__fmul2_rn(P, __fmul2_rn(ir, ir)), __ffma2_rn(A1, ir, Bq));
                        const float sxy = sc.x + sc.y;  // both voxels share x and y
                        G[q][0] = sxy * cur.dx;
                        G[q][1] = sxy * cur.dy;
                        G[q][2] = __fmaf_rn(sc.x, cur.dz.x, sc.y * cur.dz.y);
                    }
                    cur = nxt;
                }
                if (POSE) {
                    // transposed warp reduction of 4 elements x 3 components
                    const bool h16 = (lane & 16) != 0, h8 = (lane & 8) != 0;
                    float r6[6];
#pragma unroll
                    for (int j = 0; j < 6; ++j) {
                        const float lo = G[j / 3][j % 3], hi = G[2 + j / 3][j % 3];
                        const float snd = h16 ? lo : hi, kp = h16 ? hi : lo;
                        r6[j] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
                    }
                    float r3[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float lo = r6[c], hi = r6[3 + c];
                        const float snd = h8 ? lo : hi, kp = h8 ? hi : lo;
                        r3[c] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
                    }
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        r3[c] += __shfl_xor_sync(0xffffffffu, r3[c], 4);
                        r3[c] += __shfl_xor_sync(0xffffffffu, r3[c], 2);
                        r3[c] += __shfl_xor_sync(0xffffffffu, r3[c], 1);
                    }
                    const int e = e0 + ((lane >> 3) & 3);
                    if ((lane & 7) == 0 && e < E) {
                        wred[(warp * E + e) * 3 + 0] = r3[0];
                        wred[(warp * E + e) * 3 + 1] = r3[1];
                        wred[(warp * E + e) * 3 + 2] = r3[2];
                    }
                }
            }
            if (POSE) {
                __syncthreads();
                for (int q = tid; q < E * 3; q += NT) {
                    float s = 0.0f;
#pragma unroll
                    for (int w = 0; w < NT / 32; ++w) s += wred[w * E * 3 + q];
                    gacc[fl * E * 3 + q] += s;
                }
            }
        }
        if (ADJ) {
            if (ina) grad_p0[ka] = (f0 == 0 ? 0.0f : grad_p0[ka]) + z.x;
            if (inb) grad_p0[kb] = (f0 == 0 ? 0.0f : grad_p0[kb]) + z.y;
        }
    }
    if (POSE) {
        __syncthreads();
        for (int q = tid; q < fn * E * 3; q += NT)
            partial[((size_t)blockIdx.x * F + f0) * E * 3 + q] = gacc[q];
    }
}

// ============================================================================================
// K2s — the adjoint (a4 + a5) in the basis of the forward's factorisation (R24): per (voxel,
// element) pair with pos = j_m + OFF,
//   A1 = sum_k g[j_m + k] G(t, k) ~= sum_m phi_m(t) F_m[pos] + [L = LMIN+1] g[pos] phi_X(t),
//   F_m[pos] = sum_{q=1..LMIN} g[pos - q] psi_m(OFF - q)          (K2s-a, per row, L2-resident)
// and the pose moment sum_k g (K + D K') = dA1/dD_m = (1/Dw) dA1/dt (the derivative of the same
// smooth approximation; the window indicator held constant, R11).  The record of a position is
// [F_0 .. F_{R-1}, g[pos], 0...] (8 floats, one 256-bit load).  With b_r = sum_{m even} F_m c_{m,r},
// o_r = sum_{m odd} F_m c_{m,r}:  A1 = E(s) + t O(s),  dA1/dt = 2t E'(s) + O(s) + 2s O'(s),  s = t^2.
// No exp, no Taylor series, no scattered load for the last tap; the window, geometry, tiling and
// pose reduction are K2c's.
// ============================================================================================
struct SvdConst {
    float psi[DEP_MAXR][PA_LMAX];  // as DepConst::psi
    float c[DEP_MAXR + 1][4];   // unscaled phi_m coefficients (index R: the last-tap cubic in t)
    float tA, tB, tC;           // t = (D_m - Dc)/Dw as in K1d
    float invDw;                // dt/dD_m
};
constexpr int SVD_NF = 8;  // floats per position record

template <int R>
__global__ void __launch_bounds__(256) k_adj_svd_filter(Geo g, SvdConst sc, const float *__restrict__ cot, int f0,
                                                        int fn, float *__restrict__ Fg)
{
    __shared__ float sg[256 + PA_LMAX];
    const int LMIN = g.lmin;  // runtime window length
    const int NJ = g.nt + LMIN;
    const int row = blockIdx.y;  // chunk-local row (f - f0) E + e
    const int p0 = blockIdx.x * 256;
    const float *gr = cot + ((size_t)f0 * g.E + row) * g.nt;
    // positions p0 .. p0+255 read samples p - q, q in [1, LMIN], and g[p]: samples [p0 - LMIN, p0 + 255]
    for (int t = threadIdx.x; t < 256 + LMIN; t += 256) {
        const int j = p0 - LMIN + t;
        sg[t] = (j >= 0 && j < g.nt) ? __ldg(gr + j) : 0.0f;
    }
    __syncthreads();
    const int pos = p0 + threadIdx.x;
    if (pos >= NJ) return;
    float acc[R];
#pragma unroll
    for (int m = 0; m < R; ++m) acc[m] = 0.0f;
#pragma unroll 4
    for (int q = 1; q <= LMIN; ++q) {  // runtime L_min
        const float v = sg[threadIdx.x + LMIN - q];
#pragma unroll
        for (int m = 0; m < R; ++m) acc[m] = __fmaf_rn(v, sc.psi[m][q - 1], acc[m]);
    }
    float rec[SVD_NF];
#pragma unroll
    for (int r = 0; r < SVD_NF; ++r) rec[r] = 0.0f;
#pragma unroll
    for (int m = 0; m < R; ++m) rec[m] = acc[m];
    rec[R] = sg[threadIdx.x + LMIN];  // g[pos]
    float4 *o = reinterpret_cast<float4 *>(Fg + ((size_t)row * NJ + pos) * SVD_NF);
    o[0] = make_float4(rec[0], rec[1], rec[2], rec[3]);
    o[1] = make_float4(rec[4], rec[5], rec[6], rec[7]);
}

struct SvdA {
    float Fa[SVD_NF], Fb[SVD_NF];  // records of voxel a (.x) and voxel b (.y)
    float2 t, inv_r, dz;
    float dx, dy;
    bool va, vb, xa, xb;  // valid; last tap in-window
};

__device__ __forceinline__ SvdA svd_stage_a(const Geo &g, const SvdConst &sc, const AncS *anc, int e, int E, bool ina,
                                            bool inb, float ex, float ey, float2 ez, float2 e2,
                                            const float *__restrict__ Frow)
{
    SvdA o;
    const int LMIN = g.lmin;  // runtime window length
    const int ec = min(e, E - 1);
    const AncS sa = anc[ec];
    const float2 num = __ffma2_rn(f2(sa.dx2), f2(ex), __ffma2_rn(f2(sa.dy2), f2(ey), __ffma2_rn(f2(sa.dz2), ez, e2)));
    const float2 r2 = __fadd2_rn(f2(sa.rho2), num);
    const float2 inv_r = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
    const float2 den = __fadd2_rn(__fmul2_rn(r2, inv_r), f2(sa.rho));
    const float2 drel = __fmul2_rn(num, make_float2(rcp_approx(den.x), rcp_approx(den.y)));
    const float2 bse = __fadd2_rn(drel, f2(sa.CA));
    const float2 xlo = __fmul2_rn(__fadd2_rn(bse, f2(-g.ksig)), f2(g.inv_a));
    const float2 xhi = __fmul2_rn(__fadd2_rn(bse, f2(g.ksig)), f2(g.inv_a));
    const float2 sh = __fadd2_rn(xlo, f2(12582912.0f));
    float2 clof = __fadd2_rn(sh, f2(-12582912.0f));
    const bool upx = clof.x < xlo.x, upy = clof.y < xlo.y;
    clof.x = upx ? clof.x + 1.0f : clof.x;
    clof.y = upy ? clof.y + 1.0f : clof.y;
    const int jla = sa.JA + __float_as_int(sh.x) - 0x4B400000 + (upx ? 1 : 0);
    const int jlb = sa.JA + __float_as_int(sh.y) - 0x4B400000 + (upy ? 1 : 0);
    const float2 cl2 = __fadd2_rn(clof, f2((float)LMIN));
    const bool Lxa = xhi.x >= cl2.x, Lxb = xhi.y >= cl2.y;  // L = LMIN + 1
    const bool ok = e < E && !sa.cull;
    o.va = ok && ina && jla <= g.nt - 1 && jla + LMIN + (Lxa ? 0 : -1) >= 0;
    o.vb = ok && inb && jlb <= g.nt - 1 && jlb + LMIN + (Lxb ? 0 : -1) >= 0;
    o.xa = Lxa;
    o.xb = Lxb;
    const int pa = o.va ? jla + LMIN : 0, pb = o.vb ? jlb + LMIN : 0;  // pos = j_m + OFF
    ldg256(Frow + pa * SVD_NF, o.Fa);
    ldg256(Frow + pb * SVD_NF, o.Fb);
    // t = (D_m - Dc)/Dw, D_m = bse - clo a - MA a  (as K1d)
    o.t = __ffma2_rn(clof, f2(-sc.tB), __ffma2_rn(drel, f2(sc.tA), f2(__fmaf_rn(sa.CA, sc.tA, sc.tC))));
    o.inv_r = inv_r;
    o.dx = sa.dx;
    o.dy = sa.dy;
    o.dz = __fadd2_rn(f2(sa.dz), ez);
    return o;
}

// A1 and dA1/dt of one voxel from its record
template <int R, bool POSE>
__device__ __forceinline__ void svd_eval(const SvdConst &sc, const float F[SVD_NF], float t, bool lx, float &A1,
                                         float &dA1)
{
    const float s = t * t;
    float e[4], o[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        e[r] = F[0] * sc.c[0][r];
        o[r] = F[1] * sc.c[1][r];
#pragma unroll
        for (int m = 2; m < R; ++m) {
            if (m & 1) o[r] = __fmaf_rn(F[m], sc.c[m][r], o[r]);
            else e[r] = __fmaf_rn(F[m], sc.c[m][r], e[r]);
        }
    }
    const float E0 = __fmaf_rn(__fmaf_rn(__fmaf_rn(e[3], s, e[2]), s, e[1]), s, e[0]);
    const float O0 = __fmaf_rn(__fmaf_rn(__fmaf_rn(o[3], s, o[2]), s, o[1]), s, o[0]);
    const float gx = lx ? F[R] : 0.0f;  // the last tap, in-window iff L = LMIN + 1
    const float X0 = __fmaf_rn(__fmaf_rn(__fmaf_rn(sc.c[R][3], t, sc.c[R][2]), t, sc.c[R][1]), t, sc.c[R][0]);
    A1 = __fmaf_rn(gx, X0, __fmaf_rn(t, O0, E0));
    dA1 = 0.0f;
    if (POSE) {
        const float E1 = __fmaf_rn(__fmaf_rn(3.0f * e[3], s, 2.0f * e[2]), s, e[1]);  // E'(s)
        const float O1 = __fmaf_rn(__fmaf_rn(3.0f * o[3], s, 2.0f * o[2]), s, o[1]);  // O'(s)
        const float X1 = __fmaf_rn(__fmaf_rn(3.0f * sc.c[R][3], t, 2.0f * sc.c[R][2]), t, sc.c[R][1]);
        const float d = __fmaf_rn(2.0f * s, O1, __fmaf_rn(2.0f * t, E1, O0));  // dA/dt = 2t E' + O + 2s O'
        dA1 = __fmaf_rn(gx, X1, d) * sc.invDw;                                 // d/dD_m
    }
}

template <int R, bool POSE, bool ADJ>
__global__ void __launch_bounds__(ADJ_THREADS, 2) k_adjoint_svd(Geo g, SvdConst sc, const float *__restrict__ poses,
                                                               const float *__restrict__ tmpl,
                                                               const float *__restrict__ p0,
                                                               const float *__restrict__ Fg,
                                                               float *__restrict__ grad_p0,
                                                               float *__restrict__ partial, int f0, int fn)
{
    extern __shared__ float sm[];
    const int E = g.E, F = g.F, NJ = g.nt + g.lmin;
    AncS *anc = reinterpret_cast<AncS *>(sm);             // [2][E]: the two tiles of the CTA
    float *wred = reinterpret_cast<float *>(anc + 2 * E);  // [8][E][3]
    float *gacc = wred + (ADJ_THREADS / 32) * E * 3;       // [fn][E][3]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int half = tid >> 7, u = tid & 127;
    const int lx = u & 7, ly = (u >> 3) & 7, lzp = u >> 6;  // voxels (lx, ly, lzp) and (lx, ly, lzp + 2)
    const float ex = ((float)lx - 0.5f * (TX - 1)) * g.hf;
    const float ey = ((float)ly - 0.5f * (TY - 1)) * g.hf;
    const float2 ez = make_float2(((float)lzp - 0.5f * (TZ - 1)) * g.hf, ((float)(lzp + 2) - 0.5f * (TZ - 1)) * g.hf);
    const float2 e2 = __ffma2_rn(f2(ex), f2(ex), __ffma2_rn(f2(ey), f2(ey), __fmul2_rn(ez, ez)));
    const AncS *anch = anc + half * E;
    const int ntzp = (g.ntz + 1) >> 1, ntp = g.ntx * g.nty * ntzp;

    if (POSE) {
        for (int q = tid; q < fn * E * 3; q += ADJ_THREADS) gacc[q] = 0.0f;
    }
    for (int tp = blockIdx.x; tp < ntp; tp += gridDim.x) {
        const int tx = tp % g.ntx, ty = (tp / g.ntx) % g.nty, tzp = tp / (g.ntx * g.nty);
        const int tz = 2 * tzp + half;
        const int ix = TX * tx + lx, iy = TY * ty + ly, iza = TZ * tz + lzp, izb = iza + 2;
        const bool ina = ix < g.nx && iy < g.ny && iza < g.nz, inb = ix < g.nx && iy < g.ny && izb < g.nz;
        const size_t ka = ((size_t)iza * g.ny + iy) * g.nx + ix, kb = ka + 2 * (size_t)g.nx * g.ny;
        const float2 P = make_float2((POSE && ina) ? __ldg(p0 + ka) : 0.0f, (POSE && inb) ? __ldg(p0 + kb) : 0.0f);
        const float2 hP = __fmul2_rn(f2(0.5f), P);
        float2 z = f2(0.0f);
        for (int fl = 0; fl < fn; ++fl) {
            const int f = f0 + fl;
            __syncthreads();  // previous frame's anchors / wred consumed
            for (int q = tid; q < 2 * E; q += ADJ_THREADS) {
                const int hh = q / E, e = q - hh * E;
                double x[3];
                elem_pos(poses, tmpl, f, e, x);
                const int tzh = 2 * tzp + hh;
                const Anc A = make_anchor(g, x, tx, ty, tzh < g.ntz ? tzh : 0);
                AncS sa;
                sa.dx2 = A.dx2; sa.dy2 = A.dy2; sa.dz2 = A.dz2;
                sa.dx = A.dx; sa.dy = A.dy; sa.dz = A.dz;
                sa.rho = A.rho; sa.rho2 = A.rho2; sa.CA = A.CA;
                sa.JA = A.JA; sa.cull = A.cull || tzh >= g.ntz; sa.jseg = 0;
                anc[q] = sa;
            }
            __syncthreads();
            const float *Frow = Fg + (size_t)fl * E * NJ * SVD_NF;
            const size_t fstep = (size_t)NJ * SVD_NF;
            SvdA cur = svd_stage_a(g, sc, anch, 0, E, ina, inb, ex, ey, ez, e2, Frow);
#pragma unroll 1
            for (int e0 = 0; e0 < E; e0 += 4) {
                float G[4][3];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = e0 + q;
                    if (e + 1 < E) Frow += fstep;
                    const SvdA nxt = svd_stage_a(g, sc, anch, e + 1, E, ina, inb, ex, ey, ez, e2, Frow);
                    float a1x, a1y, d1x = 0.0f, d1y = 0.0f;
                    svd_eval<R, POSE>(sc, cur.Fa, cur.t.x, cur.xa, a1x, d1x);
                    svd_eval<R, POSE>(sc, cur.Fb, cur.t.y, cur.xb, a1y, d1y);
                    float2 A1 = make_float2(cur.va ? a1x : 0.0f, cur.vb ? a1y : 0.0f);
                    const float2 ir = cur.inv_r;
                    const float2 hir = __fmul2_rn(f2(0.5f), ir);
                    if (ADJ) z = __ffma2_rn(A1, hir, z);
                    if (POSE) {
                        const float2 A2 = make_float2(cur.va ? d1x : 0.0f, cur.vb ? d1y : 0.0f);
                        // dL/dr = P/(2r) (A2 - A1/r);  G += -dL/dr (d + delta)/r
                        const float2 dL = __fmul2_rn(__fmul2_rn(hP, ir), __ffma2_rn(__fmul2_rn(f2(-1.0f), A1), ir, A2));
                        const float2 scv = __fmul2_rn(__fmul2_rn(f2(-1.0f), dL), ir);
                        const float sxy = scv.x + scv.y;  // both voxels share x and y
                        G[q][0] = sxy * (cur.dx + ex);
                        G[q][1] = sxy * (cur.dy + ey);
                        G[q][2] = scv.x * cur.dz.x + scv.y * cur.dz.y;
                    }
                    cur = nxt;
                }
                if (POSE) {
                    const bool h16 = (lane & 16) != 0, h8 = (lane & 8) != 0;
                    float r6[6];
#pragma unroll
                    for (int j = 0; j < 6; ++j) {
                        const float lo = G[j / 3][j % 3], hi = G[2 + j / 3][j % 3];
                        const float snd = h16 ? lo : hi, kp = h16 ? hi : lo;
                        r6[j] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
                    }
                    float r3[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float lo = r6[c], hi = r6[3 + c];
                        const float snd = h8 ? lo : hi, kp = h8 ? hi : lo;
                        r3[c] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
                    }
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        r3[c] += __shfl_xor_sync(0xffffffffu, r3[c], 4);
                        r3[c] += __shfl_xor_sync(0xffffffffu, r3[c], 2);
                        r3[c] += __shfl_xor_sync(0xffffffffu, r3[c], 1);
                    }
                    const int e = e0 + ((lane >> 3) & 3);
                    if ((lane & 7) == 0 && e < E) {
                        wred[(warp * E + e) * 3 + 0] = r3[0];
                        wred[(warp * E + e) * 3 + 1] = r3[1];
                        wred[(warp * E + e) * 3 + 2] = r3[2];
                    }
                }
            }
            if (POSE) {
                __syncthreads();
                for (int q = tid; q < E * 3; q += ADJ_THREADS) {
                    float s = 0.0f;
#pragma unroll
                    for (int w = 0; w < ADJ_THREADS / 32; ++w) s += wred[w * E * 3 + q];
                    gacc[fl * E * 3 + q] += s;
                }
            }
        }
        if (ADJ) {
            if (ina) grad_p0[ka] = (f0 == 0 ? 0.0f : grad_p0[ka]) + z.x;
            if (inb) grad_p0[kb] = (f0 == 0 ? 0.0f : grad_p0[kb]) + z.y;
        }
    }
    if (POSE) {
        __syncthreads();
        for (int q = tid; q < fn * E * 3; q += ADJ_THREADS)
            partial[((size_t)blockIdx.x * F + f0) * E * 3 + q] = gacc[q];
    }
}

// max |p0| as float bits (non-negative floats order like unsigned integers): the 1/Pmax
// normalisation of the fixed-point deposits of K1d.
static __global__ void k_absmax(const float *__restrict__ p, long long n, unsigned *__restrict__ out)
{
    unsigned m = 0u;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        m = max(m, __float_as_uint(fabsf(__ldg(p + i))));
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace pa

#ifdef PA_API_TU  // the TGV kernels are launched from pa_api.cu only
#include <cuda.h>  // CUtensorMap
namespace pa {

// ============================================================================================
// K7 — TGV^2 regulariser of Eq. 2 (reading R20): value and gradients
//   L = a1 sum_O phi(grad P - w) + a0 sum_O phi(E w),  phi(v) = sqrt(|v|^2 + eps^2) - eps,
//   forward differences, O = {x : x_d <= n_d - 2}, and
//   dL/dP(k)   = a1/h sum_d [n_d(k - e_d) - n_d(k)]
//   dL/dw_b(k) = -a1 n_b(k) + a0/h sum_a [m_ab(k - e_a) - m_ab(k)]      (m symmetric)
// with the dphi fields n = g/|g|_eps (g = grad P - w) and m = E/|E|_eps (E = sym grad w).
// 2.5-D streaming: a CTA owns a 32 x 8 column of (x, y) outputs and walks z through a slab; thread q owns the
// raw point (x0 - 1 + q % 34, y0 - 1 + q / 34) of a 34 x 10 region.  Per plane z, the 33 x 9 halo points form
// n and m from raw plane z (own value, x + 1 and y + 1 neighbours) and their own plane-(z + 1) value, keep
// n and m in registers and publish only what a neighbour's gradient reads: the x-row (n_x, m_xx, m_xy, m_xz)
// and the y-row (n_y, m_xy, m_yy, m_yz); the gradient of plane z at the owned points takes the -e_x / -e_y
// rows from shared memory and the -e_z row (n_z, m_xz, m_yz, m_zz of plane z - 1) from the registers of the
// previous plane.  The value is reduced per block in fp64 (fixed order) into `part`, summed by k_sum_parts.
// Two variants move the raw planes:
//   k_tgv_tma (nx % 4 == 0, 16-B aligned): TMA (cp.async.bulk.tensor) copies each raw plane (40 x 10 box of
//     P and 40 x 10 x 3 of w, x from x0 - 4: TMA needs a 16-B aligned innermost start; zero-filled outside the volume) into a ring of TGV_STAGES shared-memory stages
//     on an mbarrier, issued TGV_STAGES - 1 planes ahead — the kernel is HBM-latency-bound, and the ring keeps
//     ~4x more bytes in flight per SM than registers can; double-buffered field rows, one barrier per plane;
//   k_tgv (any shape): each thread streams its column through four register buffers (rotated by name) and
//     publishes raw plane z in shared memory; two barriers per plane.
// ============================================================================================
struct TgvArgs {
    int nx, ny, nz;
    float inv_h, a1, a0, eps;
    float gs;  // scale of both gradients (lambda of Eq. 2 inside pa_step, 1 for pa_tgv)
};

#ifndef TGV_BYM
#define TGV_BYM 8
#endif
#ifndef TGV_ZSM
#define TGV_ZSM 32
#endif
constexpr int TGV_BX = 32, TGV_BY = TGV_BYM, TGV_ZS = TGV_ZSM;
constexpr int TGV_RX = TGV_BX + 2, TGV_RY = TGV_BY + 2;               // raw region 34 x 10
constexpr int TGV_NT = (TGV_RX * TGV_RY + 31) / 32 * 32;              // 352 threads
constexpr int TGV_PX = TGV_BX + 1, TGV_PY = TGV_BY + 1;               // halo (field) points 33 x 9
#ifndef TGV_MINB
#define TGV_MINB 2  // resident k_tgv_tma CTAs per SM (18 warps each at 16 rows)
#endif

// The dphi fields at a halo point of plane z (zero outside O): c = (P, w) at the point, rx / ry at its
// x + 1 / y + 1 neighbours, c1 at z + 1.  Publishes the x- and y-rows; returns n, m and this point's value
// terms a1 phi(g) + a0 phi(E) (0 outside O).
struct TgvF {
    float n0, n1, n2, mxx, myy, mzz, mxy, mxz, myz;
};
__device__ __forceinline__ TgvF tgv_fields(const TgvArgs &t, bool in, const float c[4], const float rx[4],
                                           const float ry[4], const float c1[4], float &v)
{
    TgvF F = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    v = 0.0f;
    if (!in) return F;
    const float h1 = t.inv_h, ee = t.eps * t.eps;
    const float g0 = __fmaf_rn(rx[0] - c[0], h1, -c[1]);
    const float g1 = __fmaf_rn(ry[0] - c[0], h1, -c[2]);
    const float g2 = __fmaf_rn(c1[0] - c[0], h1, -c[3]);
    // D[a][b] = d_a w_b
    const float dxx = (rx[1] - c[1]) * h1, dxy = (rx[2] - c[2]) * h1, dxz = (rx[3] - c[3]) * h1;
    const float dyx = (ry[1] - c[1]) * h1, dyy = (ry[2] - c[2]) * h1, dyz = (ry[3] - c[3]) * h1;
    const float dzx = (c1[1] - c[1]) * h1, dzy = (c1[2] - c[2]) * h1, dzz = (c1[3] - c[3]) * h1;
    const float sg = __fmaf_rn(g0, g0, __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, ee)));
    const float ig = rsqrtf(sg);  // |v|_eps and 1/|v|_eps from one MUFU.RSQ
    F.n0 = g0 * ig;
    F.n1 = g1 * ig;
    F.n2 = g2 * ig;
    const float exy = 0.5f * (dxy + dyx), exz = 0.5f * (dxz + dzx), eyz = 0.5f * (dyz + dzy);
    const float se = __fmaf_rn(dxx, dxx, __fmaf_rn(dyy, dyy, __fmaf_rn(dzz, dzz,
                     __fmaf_rn(2.0f * exy, exy, __fmaf_rn(2.0f * exz, exz, __fmaf_rn(2.0f * eyz, eyz, ee))))));
    const float ie = rsqrtf(se);
    F.mxx = dxx * ie;
    F.myy = dyy * ie;
    F.mzz = dzz * ie;
    F.mxy = exy * ie;
    F.mxz = exz * ie;
    F.myz = eyz * ie;
    v = t.a1 * (sg * ig - t.eps) + t.a0 * (se * ie - t.eps);
    return F;
}

// the gradient at an owned point k from its fields F, the -e_x / -e_y rows and the -e_z row pz
__device__ __forceinline__ void tgv_grad(const TgvArgs &t, const TgvF &F, float4 fx, float4 fy, const float pz[4],
                                         int k, int nv, float *__restrict__ gP, float *__restrict__ gw)
{
    const float ga = t.gs * t.a1 * t.inv_h, gb = t.gs * t.a0 * t.inv_h, gc = t.gs * t.a1;
    gP[k] = ga * ((fx.x - F.n0) + (fy.x - F.n1) + (pz[0] - F.n2));
    gw[k] = __fmaf_rn(-gc, F.n0, gb * ((fx.y - F.mxx) + (fy.y - F.mxy) + (pz[1] - F.mxz)));
    gw[nv + k] = __fmaf_rn(-gc, F.n1, gb * ((fx.z - F.mxy) + (fy.z - F.myy) + (pz[2] - F.myz)));
    gw[2 * nv + k] = __fmaf_rn(-gc, F.n2, gb * ((fx.w - F.mxz) + (fy.w - F.myz) + (pz[3] - F.mzz)));
}

// fixed-order block sum of the value: shuffle tree per warp, then the warp partials in order
__device__ __forceinline__ void tgv_block_value(double val, double *red, double *__restrict__ part)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) val += __shfl_down_sync(0xffffffffu, val, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = val;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s2 = 0.0;
        for (int q = 0; q < TGV_NT / 32; ++q) s2 += red[q];
        part[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s2;
    }
}

__global__ void __launch_bounds__(TGV_NT, 2) k_tgv(TgvArgs t, const float *__restrict__ P,
                                                const float *__restrict__ w, float *__restrict__ gP,
                                                float *__restrict__ gw, double *__restrict__ part)
{
    __shared__ float raw[4][TGV_RY][TGV_RX];  // raw plane z: P, w_x, w_y, w_z at (x - 1 .. x + 32, y - 1 .. y + 8)
    __shared__ float4 fxr[TGV_PY][TGV_PX];    // x-row of the fields: (n_x, m_xx, m_xy, m_xz)
    __shared__ float4 fyr[TGV_PY][TGV_PX];    // y-row of the fields: (n_y, m_xy, m_yy, m_yz)
    __shared__ double red[TGV_NT / 32];
    const int i = threadIdx.x % TGV_RX, j = threadIdx.x / TGV_RX;  // this thread's raw point
    const int x0 = blockIdx.x * TGV_BX, y0 = blockIdx.y * TGV_BY, z0 = blockIdx.z * TGV_ZS;
    const int x = x0 - 1 + i, y = y0 - 1 + j;
    const bool rp = threadIdx.x < TGV_RX * TGV_RY;           // a raw point
    const bool pt = rp && i < TGV_PX && j < TGV_PY;          // a halo point (computes fields)
    const int sz = t.nx * t.ny, nv = sz * t.nz;              // 3 nv < 2^31 (tgv_args)
    const bool own = pt && i >= 1 && j >= 1 && x < t.nx && y < t.ny;  // owns output voxel (x, y)
    const bool inxy = rp && x >= 0 && y >= 0 && x < t.nx && y < t.ny;
    const bool fxy = x >= 0 && y >= 0 && x <= t.nx - 2 && y <= t.ny - 2;  // interior in x, y
    const int kxy = inxy ? y * t.nx + x : 0;
    const int zbeg = z0 - 1, zend = min(z0 + TGV_ZS, t.nz);
    double val = 0.0;
    auto ld = [&](int z, float v[4]) {  // this column's raw values at plane z (0 outside the volume / past the slab)
        const bool ok = inxy && z >= 0 && z < t.nz && z <= zend;
        const int k = z * sz + kxy;
        v[0] = ok ? __ldg(P + k) : 0.0f;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[1 + c] = ok ? __ldg(w + c * nv + k) : 0.0f;
    };
    float pz[4] = {0.f, 0.f, 0.f, 0.f};  // n_z, m_xz, m_yz, m_zz of the previous plane at this point
    auto plane = [&](int z, const float cz[4], const float c1[4]) {
        if (rp) {
#pragma unroll
            for (int c = 0; c < 4; ++c) raw[c][j][i] = cz[c];
        }
        __syncthreads();  // raw plane z published (and the previous plane's field rows consumed)
        TgvF F = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (pt) {
            const bool in = fxy && z >= 0 && z <= t.nz - 2;
            float rx[4], ry[4], v;
            if (in) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    rx[c] = raw[c][j][i + 1];
                    ry[c] = raw[c][j + 1][i];
                }
            }
            F = tgv_fields(t, in, cz, rx, ry, c1, v);
            if (own && z >= z0) val += (double)v;  // counted once, by the owner, in its own slab
            fxr[j][i] = make_float4(F.n0, F.mxx, F.mxy, F.mxz);
            fyr[j][i] = make_float4(F.n1, F.mxy, F.myy, F.myz);
        }
        __syncthreads();  // field rows of plane z published (and raw plane z consumed)
        if (own && z >= z0) tgv_grad(t, F, fxr[j][i - 1], fyr[j - 1][i], pz, z * sz + kxy, nv, gP, gw);
        pz[0] = F.n2;
        pz[1] = F.mxz;
        pz[2] = F.myz;
        pz[3] = F.mzz;
    };
    // four column buffers rotated by name (unrolled by 4: no register move waits on a load in flight), each
    // refilled right after its plane is done — planes z + 1 .. z + 3 are in flight during plane z
    float b0[4], b1[4], b2[4], b3[4];
    ld(zbeg, b0);
    ld(zbeg + 1, b1);
    ld(zbeg + 2, b2);
    ld(zbeg + 3, b3);
    for (int z = zbeg; z < zend; z += 4) {
        plane(z, b0, b1);
        ld(z + 4, b0);
        if (z + 1 >= zend) break;
        plane(z + 1, b1, b2);
        ld(z + 5, b1);
        if (z + 2 >= zend) break;
        plane(z + 2, b2, b3);
        ld(z + 6, b2);
        if (z + 3 >= zend) break;
        plane(z + 3, b3, b0);
        ld(z + 7, b3);
    }
    tgv_block_value(val, red, part);
}

// ---- TMA-staged variant ------------------------------------------------------------------------------
#ifndef TGV_STAGES
#define TGV_STAGES 6
#endif
// TMA box: x0 - 4 .. x0 + 35 (the innermost start coordinate must be a multiple of 16 B, so not x0 - 1;
// raw column i of the thread grid is box column i + 3), y0 - 1 .. y0 + 8
constexpr int TGV_BOXX = 40, TGV_BOX0 = 3;
#ifndef TGV_TBYM
#define TGV_TBYM 16  // 32 x 16 outputs per CTA (256^3: 0.151 ms; 8 rows 0.158, 12 rows 0.163, 24 rows 0.171)
#endif
constexpr int TGV_TBY = TGV_TBYM;                               // k_tgv_tma: outputs per CTA in y (>= TGV_BY)
constexpr int TGV_TRY = TGV_TBY + 2, TGV_TPY = TGV_TBY + 1;     // box rows, halo (field) rows
constexpr int TGV_PLN = TGV_BOXX * TGV_TRY;                     // floats of one channel plane (400 at 8 rows)
constexpr int TGV_WOFF = (TGV_PLN + 31) / 32 * 32;              // w boxes after the P box (padded to 128 B)
constexpr int TGV_STAGE_F = TGV_WOFF + (3 * TGV_PLN + 31) / 32 * 32;  // + the w boxes (padded): 6528 B per stage at BY = 8
constexpr unsigned TGV_TX_BYTES = 4u * 4u * TGV_PLN;            // bytes a stage receives (6400)
constexpr size_t tgv_tma_smem() { return (size_t)TGV_STAGES * TGV_STAGE_F * 4 + 2 * 2 * TGV_TPY * TGV_PX * 16 + 128; }

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TGV_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TGV_WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_3d(float *dst, const void *tm, int x, int y, int z, uint64_t *b)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)), "l"(tm), "r"(x), "r"(y), "r"(z), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void tma_4d(float *dst, const void *tm, int x, int y, int z, int c, uint64_t *b)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(smem_u32(dst)), "l"(tm), "r"(x), "r"(y), "r"(z), "r"(c), "r"(smem_u32(b))
        : "memory");
}

// tmP: P as {nx, ny, nz} fp32, box {40, 10, 1};  tmW: w as {nx, ny, nz, 3}, box {40, 10, 1, 3}.
// Threads only for the 33 x (TBY + 1) halo points (the raw planes arrive by TMA): warp w <= TBY is halo row
// j = w, lanes columns i = 1..32 (uniform per warp: no divergent halo / ownership tests inside a row); warp
// TBY + 1, lanes 0..TBY, is column i = 0.  32 x 16 outputs per CTA (halo rows 6%), 2 CTAs per SM.
// Measured (256^3 / 512^3): one thread per raw point (352 threads, 8 rows) 0.179 / 1.295 ms; halo-point
// threads at 8 rows 0.158 / 1.148, 12 rows 0.163 / 1.125, 16 rows 0.151 / 1.084, 24 rows 0.171 / 1.232;
// 16-, 24-, 48-plane slabs 0.157 / 0.155 / 0.163 at 256^3; 4 stages 0.155; two raw rows per thread 0.19.
constexpr int TGV2_NT = (TGV_TPY + 1) * 32;  // 576 at 16 rows
__global__ void __launch_bounds__(TGV2_NT, TGV_MINB) k_tgv_tma(TgvArgs t, const __grid_constant__ CUtensorMap tmP,
                                                     const __grid_constant__ CUtensorMap tmW,
                                                     float *__restrict__ gP, float *__restrict__ gw,
                                                     double *__restrict__ part)
{
    extern __shared__ __align__(128) float tsm_[];
    // TMA destinations 128-B aligned whatever the dynamic base (tgv_tma_smem() has 128 B of slack)
    float *tsm = tsm_ + ((128u - (smem_u32(tsm_) & 127u)) & 127u) / 4;
    float *stg = tsm;                                                          // [S][TGV_STAGE_F]
    float4 *frows = reinterpret_cast<float4 *>(tsm + TGV_STAGES * TGV_STAGE_F); // [2 planes][X, Y][PY][PX]
    __shared__ __align__(8) uint64_t full[TGV_STAGES];
    __shared__ double red[TGV2_NT / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = warp < TGV_TPY ? lane + 1 : 0, j = warp < TGV_TPY ? warp : lane;
    const bool pt = warp < TGV_TPY || lane < TGV_TPY;                // a halo point (computes fields)
    const int x0 = blockIdx.x * TGV_BX, y0 = blockIdx.y * TGV_TBY, z0 = blockIdx.z * TGV_ZS;
    const int x = x0 - 1 + i, y = y0 - 1 + j;
    const int sz = t.nx * t.ny, nv = sz * t.nz;
    const bool own = pt && i >= 1 && j >= 1 && x < t.nx && y < t.ny;
    const bool fxy = x >= 0 && y >= 0 && x <= t.nx - 2 && y <= t.ny - 2;
    const int zbeg = z0 - 1, zend = min(z0 + TGV_ZS, t.nz), nq = zend - zbeg;  // planes zbeg .. zend (nq + 1)
    const int o = j * TGV_BOXX + i + TGV_BOX0;                                   // this point in a box plane
    const int fo = j * TGV_PX + i;                                               // ... in a field-row plane
    auto issue = [&](int q) {  // plane zbeg + q into stage q % S (one thread)
        float *d = stg + (q % TGV_STAGES) * TGV_STAGE_F;
        uint64_t *b = &full[q % TGV_STAGES];
        mbar_expect_tx(b, TGV_TX_BYTES);
        tma_3d(d, &tmP, x0 - 4, y0 - 1, zbeg + q, b);
        tma_4d(d + TGV_WOFF, &tmW, x0 - 4, y0 - 1, zbeg + q, 0, b);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < TGV_STAGES; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int q = 0; q < TGV_STAGES && q <= nq; ++q) issue(q);
    double val = 0.0;
    float pz[4] = {0.f, 0.f, 0.f, 0.f};
    int k = zbeg * sz + ((x >= 0 && y >= 0) ? y * t.nx + x : 0);  // global index of (x, y, z), advanced per plane
    for (int q = 0; q < nq; ++q, k += sz) {
        const int z = zbeg + q;
        const float *s0 = stg + (q % TGV_STAGES) * TGV_STAGE_F, *s1 = stg + ((q + 1) % TGV_STAGES) * TGV_STAGE_F;
        float4 *fx = frows + (q & 1) * 2 * TGV_TPY * TGV_PX, *fy = fx + TGV_TPY * TGV_PX;
        mbar_wait(&full[q % TGV_STAGES], (unsigned)(q / TGV_STAGES) & 1u);
        mbar_wait(&full[(q + 1) % TGV_STAGES], (unsigned)((q + 1) / TGV_STAGES) & 1u);
        TgvF F = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (pt) {
            const bool in = fxy && z >= 0 && z <= t.nz - 2;
            float c[4], c1[4], rx[4], ry[4], v;
            if (in) {
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const int co = cc == 0 ? 0 : TGV_WOFF + (cc - 1) * TGV_PLN;
                    const float *a = s0 + co, *a1 = s1 + co;
                    c[cc] = a[o];
                    rx[cc] = a[o + 1];
                    ry[cc] = a[o + TGV_BOXX];
                    c1[cc] = a1[o];
                }
            }
            F = tgv_fields(t, in, c, rx, ry, c1, v);
            if (own && z >= z0) val += (double)v;  // counted once, by the owner, in its own slab
            fx[fo] = make_float4(F.n0, F.mxx, F.mxy, F.mxz);
            fy[fo] = make_float4(F.n1, F.mxy, F.myy, F.myz);
        }
        __syncthreads();  // field rows of plane z published; stage q consumed by every thread
        if (threadIdx.x == 0 && q + TGV_STAGES <= nq) issue(q + TGV_STAGES);
        if (own && z >= z0) tgv_grad(t, F, fx[fo - 1], fy[fo - TGV_PX], pz, k, nv, gP, gw);
        pz[0] = F.n2;
        pz[1] = F.mxz;
        pz[2] = F.myz;
        pz[3] = F.mzz;
    }
    // fixed-order block sum (10 warps)
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) val += __shfl_down_sync(0xffffffffu, val, o2);
    if (lane == 0) red[warp] = val;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s2 = 0.0;
        for (int w = 0; w < TGV2_NT / 32; ++w) s2 += red[w];
        part[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s2;
    }
}

}  // namespace pa
#endif  // PA_API_TU
