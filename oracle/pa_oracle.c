/*
 * pa_oracle.c — plain, slow, obviously-correct fp64 CPU oracle for the PA-SFM
 * differentiable acoustic radiation operator (arXiv 2604.09643).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code
 * with the CUDA path (paper_2604_09643_b200/csrc) and includes none of its headers.
 *
 * Citation convention: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * DESIGN.md "R<k>" = a reading of the paper listed in DESIGN.md §3.
 *
 * Units: mm, µs, mm/µs.  Every function evaluates in double precision, loops in a
 * fixed order, and each OpenMP thread owns the outputs it writes (deterministic).
 *
 * Definitions:
 *   voxel k = i + nx*(j + ny*l), centre y_k = origin + pitch*(i, j, l)         (R7)
 *   element position x_fe = R_f * tmpl_e + t_f, poses[f] = R row-major, t
 *   sample j at time t_j = t0 + j*dt                                           (R5)
 *   r = |x_fe - y_k|,  D = r - c*t_j
 *   traces[f,e,j] = sum_k p0[k] * D/(2r) * K(|D|) * [|D| <= kappa*sigma]
 *                                                   (Eq. gpu_forward_model P:341-345,
 *                                                    cutoff R4 / S:141; kappa <= 0 => dense)
 *   K = "the designated kernel function"; sigma is its scale s (R23):
 *     kernel 0  Gaussian     K(D) = exp(-D^2 / 2 s^2)      (Eq. gaussian_far_field)
 *     kernel 1  exponential  K(D) = exp(-|D| / s)          (Eq. exponential_solution, P:313-316,
 *                                                           outgoing term, far field P:325-329)
 *     kernel 2  power law    K(D) = (D^2 + s^2)^(-nu)      (Eq. power_law_solution, P:318-322,
 *                                                           outgoing term, nu > 1/2)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef struct {
    int32_t nx, ny, nz;
    double origin[3];
    double pitch;
} og_grid;

typedef struct {
    double c, t0, dt;
    int32_t nt;
    double sigma, kappa; /* kappa <= 0 : dense (no cutoff), documentation/FD mode (R11) */
    int32_t kernel;      /* 0 Gaussian, 1 exponential, 2 power law (R23) */
    double nu;           /* power-law exponent (kernel 2 only) */
} og_acq;

/* ---------------------------------------------------------------------------
 * a1: rigid placement x_fe = R_f x^_e + t_f  (Stage 4; Alg. 1)
 * ------------------------------------------------------------------------- */
void oracle_place(const double *tmpl, int32_t E, const double *poses, int32_t F, double *pos)
{
    for (int f = 0; f < F; ++f) {
        const double *R = poses + 12 * f, *t = poses + 12 * f + 9;
        for (int e = 0; e < E; ++e) {
            const double *xh = tmpl + 3 * e;
            for (int a = 0; a < 3; ++a)
                pos[(f * E + e) * 3 + a] = R[3 * a + 0] * xh[0] + R[3 * a + 1] * xh[1] + R[3 * a + 2] * xh[2] + t[a];
        }
    }
}

static void voxel_centre(const og_grid *g, int64_t k, double y[3])
{
    int64_t i = k % g->nx, j = (k / g->nx) % g->ny, l = k / ((int64_t)g->nx * g->ny);
    y[0] = g->origin[0] + g->pitch * (double)i;
    y[1] = g->origin[1] + g->pitch * (double)j;
    y[2] = g->origin[2] + g->pitch * (double)l;
}

static double dist3(const double x[3], const double y[3])
{
    double dx = x[0] - y[0], dy = x[1] - y[1], dz = x[2] - y[2];
    return sqrt(dx * dx + dy * dy + dz * dz);
}

/* The window predicate |r - c (t0 + j dt)| <= kappa sigma, evaluated literally. */
static int in_window(const og_acq *a, double r, int j)
{
    if (a->kappa <= 0.0) return 1;
    double D = r - a->c * (a->t0 + (double)j * a->dt);
    return fabs(D) <= a->kappa * a->sigma;
}

/* Support [jlo, jhi] (clipped to [0, nt-1]) of the predicate for distance r.
 * First guess by solving the inequality, then corrected against the literal
 * predicate so that the support is exactly {j : in_window(j)}.  Returns 0 if empty. */
static int window(const og_acq *a, double r, int *jlo_out, int *jhi_out)
{
    int jlo, jhi;
    if (a->kappa <= 0.0) {
        jlo = 0;
        jhi = a->nt - 1;
    } else {
        double cdt = a->c * a->dt, w = a->kappa * a->sigma;
        double lo = ceil((r - w - a->c * a->t0) / cdt), hi = floor((r + w - a->c * a->t0) / cdt);
        if (hi < 0.0 || lo > (double)(a->nt - 1)) return 0;
        jlo = lo < 0.0 ? 0 : (int)lo;
        jhi = hi > (double)(a->nt - 1) ? a->nt - 1 : (int)hi;
        while (jlo > 0 && in_window(a, r, jlo - 1)) --jlo;
        while (jlo <= jhi && !in_window(a, r, jlo)) ++jlo;
        while (jhi < a->nt - 1 && in_window(a, r, jhi + 1)) ++jhi;
        while (jhi >= jlo && !in_window(a, r, jhi)) --jhi;
        if (jhi < jlo) return 0;
    }
    *jlo_out = jlo;
    *jhi_out = jhi;
    return 1;
}

/* The designated kernel K(D) and D K'(D) / K(D), by family (R23). */
static double kfun(const og_acq *a, double D)
{
    double s = a->sigma;
    if (a->kernel == 1) return exp(-fabs(D) / s);
    if (a->kernel == 2) return pow(D * D + s * s, -a->nu);
    return exp(-D * D / (2.0 * s * s));
}

static double dlogk_times_D(const og_acq *a, double D)
{
    double s = a->sigma;
    if (a->kernel == 1) return -fabs(D) / s;                      /* d/dD e^{-|D|/s} = -sgn(D)/s K */
    if (a->kernel == 2) return -2.0 * a->nu * D * D / (D * D + s * s);
    return -D * D / (s * s);
}

/* N-shaped kernel h(D)/(2r) = D/(2r) K(|D|)   (Eq. gpu_forward_model) */
static double kern(const og_acq *a, double r, int j)
{
    double D = r - a->c * (a->t0 + (double)j * a->dt);
    return D / (2.0 * r) * kfun(a, D);
}

/* d/dr [D K(D)/(2r)] = K(D)/(2r) * [(1 + D K'/K) - D/r];
 * Gaussian: 1 + D K'/K = 1 - D^2/s^2 */
static double dkern_dr(const og_acq *a, double r, int j)
{
    double D = r - a->c * (a->t0 + (double)j * a->dt);
    return kfun(a, D) / (2.0 * r) * ((1.0 + dlogk_times_D(a, D)) - D / r);
}

/* OpenMP threads of the oracle's parallel loops (the cpu_baseline's 1-thread and all-core rates). */
void oracle_set_threads(int32_t n) { omp_set_num_threads(n > 0 ? n : 1); }
int32_t oracle_get_threads(void) { return omp_get_max_threads(); }

/* ---------------------------------------------------------------------------
 * a2: forward radiation (Eq. gpu_forward_model; Eq. 1)
 * traces[F][E][nt] are overwritten.
 * ------------------------------------------------------------------------- */
void oracle_forward(const og_grid *g, const og_acq *a, const double *tmpl, int32_t E, const double *poses,
                    int32_t F, const double *p0, double *traces)
{
    int64_t nvox = (int64_t)g->nx * g->ny * g->nz;
    double *pos = (double *)malloc(sizeof(double) * 3 * (size_t)F * E);
    oracle_place(tmpl, E, poses, F, pos);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t fe = 0; fe < (int64_t)F * E; ++fe) {
        double *out = traces + fe * a->nt;
        for (int j = 0; j < a->nt; ++j) out[j] = 0.0;
        for (int64_t k = 0; k < nvox; ++k) {
            double y[3];
            voxel_centre(g, k, y);
            double r = dist3(pos + 3 * fe, y);
            int jlo, jhi;
            if (!window(a, r, &jlo, &jhi)) continue;
            for (int j = jlo; j <= jhi; ++j) out[j] += p0[k] * kern(a, r, j);
        }
    }
    free(pos);
}

/* ---------------------------------------------------------------------------
 * a4: adjoint back-projection, the exact transpose of a2
 * grad_p0[k] = sum_f sum_e sum_j cot[f,e,j] * h(D)/(2r) * [window].  Overwritten.
 * ------------------------------------------------------------------------- */
void oracle_adjoint(const og_grid *g, const og_acq *a, const double *tmpl, int32_t E, const double *poses,
                    int32_t F, const double *cot, double *grad_p0)
{
    int64_t nvox = (int64_t)g->nx * g->ny * g->nz;
    double *pos = (double *)malloc(sizeof(double) * 3 * (size_t)F * E);
    oracle_place(tmpl, E, poses, F, pos);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nvox; ++k) {
        double y[3], z = 0.0;
        voxel_centre(g, k, y);
        for (int64_t fe = 0; fe < (int64_t)F * E; ++fe) {
            double r = dist3(pos + 3 * fe, y);
            int jlo, jhi;
            if (!window(a, r, &jlo, &jhi)) continue;
            const double *gfe = cot + fe * a->nt;
            for (int j = jlo; j <= jhi; ++j) z += gfe[j] * kern(a, r, j);
        }
        grad_p0[k] = z;
    }
    free(pos);
}

/* Error scale of a4 per voxel (test infrastructure, not part of the operator): the sum of the
 * magnitudes of the terms a4 adds, sum_f sum_e sum_j |cot[f,e,j]| |h(D)/(2r)| [window].  A per-voxel
 * parity bound |z_gpu - z| <= tol * grad_abs[k] judges each voxel against its own terms (the fp32
 * rounding of a sum scales with the sum of its |terms|, not with its value). */
void oracle_adjoint_abs(const og_grid *g, const og_acq *a, const double *tmpl, int32_t E, const double *poses,
                        int32_t F, const double *cot, double *grad_abs)
{
    int64_t nvox = (int64_t)g->nx * g->ny * g->nz;
    double *pos = (double *)malloc(sizeof(double) * 3 * (size_t)F * E);
    oracle_place(tmpl, E, poses, F, pos);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nvox; ++k) {
        double y[3], z = 0.0;
        voxel_centre(g, k, y);
        for (int64_t fe = 0; fe < (int64_t)F * E; ++fe) {
            double r = dist3(pos + 3 * fe, y);
            int jlo, jhi;
            if (!window(a, r, &jlo, &jhi)) continue;
            const double *gfe = cot + fe * a->nt;
            for (int j = jlo; j <= jhi; ++j) z += fabs(gfe[j]) * fabs(kern(a, r, j));
        }
        grad_abs[k] = z;
    }
    free(pos);
}

/* ---------------------------------------------------------------------------
 * a5: element-position gradient ("sensor spatial coordinates")
 * grad_elem[f,e,:] = sum_k p0[k] sum_j cot[f,e,j] d/dr[h/(2r)] * (x_fe - y_k)/r.
 * The window indicator is held constant (R11).
 * ------------------------------------------------------------------------- */
void oracle_elem_grad(const og_grid *g, const og_acq *a, const double *tmpl, int32_t E, const double *poses,
                      int32_t F, const double *p0, const double *cot, double *grad_elem)
{
    int64_t nvox = (int64_t)g->nx * g->ny * g->nz;
    double *pos = (double *)malloc(sizeof(double) * 3 * (size_t)F * E);
    oracle_place(tmpl, E, poses, F, pos);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t fe = 0; fe < (int64_t)F * E; ++fe) {
        const double *x = pos + 3 * fe, *gfe = cot + fe * a->nt;
        double G[3] = {0.0, 0.0, 0.0};
        for (int64_t k = 0; k < nvox; ++k) {
            double y[3];
            voxel_centre(g, k, y);
            double r = dist3(x, y);
            int jlo, jhi;
            if (!window(a, r, &jlo, &jhi)) continue;
            double dLdr = 0.0;
            for (int j = jlo; j <= jhi; ++j) dLdr += gfe[j] * dkern_dr(a, r, j);
            dLdr *= p0[k];
            for (int c = 0; c < 3; ++c) G[c] += dLdr * (x[c] - y[c]) / r;
        }
        for (int c = 0; c < 3; ++c) grad_elem[3 * fe + c] = G[c];
    }
    free(pos);
}

/* ---------------------------------------------------------------------------
 * a6: pose chain rule (Stage 4 P:109): x_fe = R_f x^_e + t_f
 * dL/dt_f = sum_e G_fe ;  dL/dR_f[a][b] = sum_e G_fe[a] x^_e[b].
 * grad_pose[F][12] = dL/dR (row-major) then dL/dt.
 * ------------------------------------------------------------------------- */
void oracle_pose_grad_from_elem(const double *tmpl, int32_t E, int32_t F, const double *grad_elem, double *grad_pose)
{
    for (int f = 0; f < F; ++f) {
        double *gp = grad_pose + 12 * f;
        for (int i = 0; i < 12; ++i) gp[i] = 0.0;
        for (int e = 0; e < E; ++e) {
            const double *G = grad_elem + 3 * ((int64_t)f * E + e), *xh = tmpl + 3 * e;
            for (int r = 0; r < 3; ++r) {
                for (int c = 0; c < 3; ++c) gp[3 * r + c] += G[r] * xh[c];
                gp[9 + r] += G[r];
            }
        }
    }
}

/* ---------------------------------------------------------------------------
 * Unit of work (SURVEY §8 d): number of (voxel, element, sample) terms with
 * |D| <= kappa sigma, j in [0, nt).  per_frame (nullable) receives per-frame counts.
 * ------------------------------------------------------------------------- */
int64_t oracle_count(const og_grid *g, const og_acq *a, const double *tmpl, int32_t E, const double *poses,
                     int32_t F, int64_t *per_frame)
{
    int64_t nvox = (int64_t)g->nx * g->ny * g->nz, total = 0;
    double *pos = (double *)malloc(sizeof(double) * 3 * (size_t)F * E);
    int64_t *pf = (int64_t *)calloc((size_t)F * E, sizeof(int64_t));
    oracle_place(tmpl, E, poses, F, pos);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t fe = 0; fe < (int64_t)F * E; ++fe) {
        int64_t n = 0;
        for (int64_t k = 0; k < nvox; ++k) {
            double y[3];
            voxel_centre(g, k, y);
            int jlo, jhi;
            if (window(a, dist3(pos + 3 * fe, y), &jlo, &jhi)) n += jhi - jlo + 1;
        }
        pf[fe] = n;
    }
    for (int f = 0; f < F; ++f) {
        int64_t s = 0;
        for (int e = 0; e < E; ++e) s += pf[(int64_t)f * E + e];
        if (per_frame) per_frame[f] = s;
        total += s;
    }
    free(pf);
    free(pos);
    return total;
}

/* ---------------------------------------------------------------------------
 * a3: losses.  MSE (Eq. 2 data term): L = sum (y - S)^2, g = 2 (y - S).
 * ------------------------------------------------------------------------- */
double oracle_mse(const double *y, const double *S, int64_t n, double *cot)
{
    double L = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double d = y[i] - S[i];
        L += d * d;
        if (cot) cot[i] = 2.0 * d;
    }
    return L;
}

/* NC loss per row (Eq. 3, population normalisation): rows of
 * length n; L_row = -cov(y,S)/(sd_y sd_S); cot = dL/dy.  mask (nullable, per row):
 * rows with mask 0 contribute neither loss nor cotangent (Eq. 4 inlier mask). */
double oracle_nc(const double *y, const double *S, int64_t rows, int32_t n, const uint8_t *mask, double *cot)
{
    double Ltot = 0.0;
    for (int64_t r = 0; r < rows; ++r) {
        const double *yr = y + r * n, *sr = S + r * n;
        double *gr = cot ? cot + r * n : NULL;
        if (mask && !mask[r]) {
            if (gr) for (int j = 0; j < n; ++j) gr[j] = 0.0;
            continue;
        }
        double my = 0.0, ms = 0.0;
        for (int j = 0; j < n; ++j) { my += yr[j]; ms += sr[j]; }
        my /= n; ms /= n;
        double cov = 0.0, vy = 0.0, vs = 0.0;
        for (int j = 0; j < n; ++j) {
            cov += (yr[j] - my) * (sr[j] - ms);
            vy += (yr[j] - my) * (yr[j] - my);
            vs += (sr[j] - ms) * (sr[j] - ms);
        }
        cov /= n; vy /= n; vs /= n;
        double sy = sqrt(vy), ss = sqrt(vs);
        Ltot += -cov / (sy * ss);
        if (gr)
            for (int j = 0; j < n; ++j)
                gr[j] = -((sr[j] - ms) / (sy * ss) - cov * (yr[j] - my) / (sy * sy * sy * ss)) / n;
    }
    return Ltot;
}

/* ---------------------------------------------------------------------------
 * a8: Adam ("Adam optimizer"), step t >= 1:
 *   m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2 ; x -= lr * mhat / (sqrt(vhat) + eps)
 * lr is per-element (lr[i] if lr_vec != NULL else lr_scalar); clamp_lo applied if clamp != 0.
 * ------------------------------------------------------------------------- */
void oracle_adam(double *x, double *m, double *v, const double *grad, int64_t n, double lr_scalar,
                 const double *lr_vec, double b1, double b2, double eps, int32_t t, int32_t clamp, double clamp_lo)
{
    double bc1 = 1.0 - pow(b1, t), bc2 = 1.0 - pow(b2, t);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * grad[i];
        v[i] = b2 * v[i] + (1.0 - b2) * grad[i] * grad[i];
        double lr = lr_vec ? lr_vec[i] : lr_scalar;
        x[i] -= lr * (m[i] / bc1) / (sqrt(v[i] / bc2) + eps);
        if (clamp && x[i] < clamp_lo) x[i] = clamp_lo;
    }
}

/* ---------------------------------------------------------------------------
 * Euler ZYX intrinsic (R8): R = Rz(a) Ry(b) Rx(c), euler = (a, b, c).
 * dR[3][9] = dR/da, dR/db, dR/dc (nullable).
 * ------------------------------------------------------------------------- */
static void mat3_mul(const double *A, const double *B, double *C)
{
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += A[3 * i + k] * B[3 * k + j];
            C[3 * i + j] = s;
        }
}

void oracle_euler_zyx(const double *euler, double *R, double *dR)
{
    double a = euler[0], b = euler[1], c = euler[2];
    double Rz[9] = {cos(a), -sin(a), 0, sin(a), cos(a), 0, 0, 0, 1};
    double Ry[9] = {cos(b), 0, sin(b), 0, 1, 0, -sin(b), 0, cos(b)};
    double Rx[9] = {1, 0, 0, 0, cos(c), -sin(c), 0, sin(c), cos(c)};
    double dRz[9] = {-sin(a), -cos(a), 0, cos(a), -sin(a), 0, 0, 0, 0};
    double dRy[9] = {-sin(b), 0, cos(b), 0, 0, 0, -cos(b), 0, -sin(b)};
    double dRx[9] = {0, 0, 0, 0, -sin(c), -cos(c), 0, cos(c), -sin(c)};
    double T[9];
    mat3_mul(Rz, Ry, T);
    mat3_mul(T, Rx, R);
    if (dR) {
        mat3_mul(dRz, Ry, T); mat3_mul(T, Rx, dR + 0);
        mat3_mul(Rz, dRy, T); mat3_mul(T, Rx, dR + 9);
        mat3_mul(Rz, Ry, T); mat3_mul(T, dRx, dR + 18);
    }
}

/* ---------------------------------------------------------------------------
 * One SfM iteration on the given frames (Alg. 1 Stages 1/4/5 objective, P:134-170;
 * SURVEY §3 call stack 3; DESIGN.md §2 "pa_step"):
 *   poses <- Euler(euler_t); y = forward(p0); L, g = loss(y, meas);
 *   gp0 = adjoint(g); G = elem_grad(p0, g); dL/dR, dL/dt; dL/dEuler = <dL/dR, dR/dEuler>_F;
 *   Adam(p0; clamp >= 0) if update_p0; Adam(euler_t) if update_pose.
 * adam_p0 = [m(nvox), v(nvox)], adam_pose = [m(F*6), v(F*6)].
 * loss_kind 0 = MSE, 1 = NC (per row, mask nullable).
 * out_grad_p0 (nvox) / out_grad_pose (F*12) / out_grad_euler (F*6) are nullable diagnostics.
 * Returns the loss.
 * ------------------------------------------------------------------------- */
double oracle_step(const og_grid *g, const og_acq *a, const double *tmpl, int32_t E, int32_t F, const double *meas,
                   double *p0, double *euler_t, double *adam_p0, double *adam_pose, double lr_p0, double lr_rot,
                   double lr_trans, double b1, double b2, double eps, int32_t t, int32_t loss_kind,
                   const uint8_t *mask, int32_t update_p0, int32_t update_pose, double *out_grad_p0,
                   double *out_grad_pose, double *out_grad_euler)
{
    int64_t nvox = (int64_t)g->nx * g->ny * g->nz, ntr = (int64_t)F * E * a->nt;
    double *poses = (double *)malloc(sizeof(double) * 12 * (size_t)F);
    double *dR = (double *)malloc(sizeof(double) * 27 * (size_t)F);
    for (int f = 0; f < F; ++f) {
        oracle_euler_zyx(euler_t + 6 * f, poses + 12 * f, dR + 27 * f);
        for (int i = 0; i < 3; ++i) poses[12 * f + 9 + i] = euler_t[6 * f + 3 + i];
    }
    double *y = (double *)malloc(sizeof(double) * ntr), *cot = (double *)malloc(sizeof(double) * ntr);
    oracle_forward(g, a, tmpl, E, poses, F, p0, y);
    double L = loss_kind == 1 ? oracle_nc(y, meas, (int64_t)F * E, a->nt, mask, cot) : oracle_mse(y, meas, ntr, cot);
    double *gp0 = (double *)malloc(sizeof(double) * nvox);
    double *gel = (double *)malloc(sizeof(double) * 3 * (size_t)F * E);
    double *gpose = (double *)malloc(sizeof(double) * 12 * (size_t)F);
    double *geul = (double *)malloc(sizeof(double) * 6 * (size_t)F);
    oracle_adjoint(g, a, tmpl, E, poses, F, cot, gp0);
    oracle_elem_grad(g, a, tmpl, E, poses, F, p0, cot, gel);
    oracle_pose_grad_from_elem(tmpl, E, F, gel, gpose);
    for (int f = 0; f < F; ++f) {
        for (int q = 0; q < 3; ++q) {
            double s = 0.0;
            for (int i = 0; i < 9; ++i) s += gpose[12 * f + i] * dR[27 * f + 9 * q + i];
            geul[6 * f + q] = s;
            geul[6 * f + 3 + q] = gpose[12 * f + 9 + q];
        }
    }
    if (out_grad_p0) memcpy(out_grad_p0, gp0, sizeof(double) * nvox);
    if (out_grad_pose) memcpy(out_grad_pose, gpose, sizeof(double) * 12 * F);
    if (out_grad_euler) memcpy(out_grad_euler, geul, sizeof(double) * 6 * F);
    if (update_p0) oracle_adam(p0, adam_p0, adam_p0 + nvox, gp0, nvox, lr_p0, NULL, b1, b2, eps, t, 1, 0.0);
    if (update_pose) {
        double *lrv = (double *)malloc(sizeof(double) * 6 * (size_t)F);
        for (int f = 0; f < F; ++f)
            for (int q = 0; q < 6; ++q) lrv[6 * f + q] = q < 3 ? lr_rot : lr_trans;
        oracle_adam(euler_t, adam_pose, adam_pose + 6 * (int64_t)F, geul, 6 * (int64_t)F, 0.0, lrv, b1, b2, eps, t, 0,
                    0.0);
        free(lrv);
    }
    free(poses); free(dR); free(y); free(cot); free(gp0); free(gel); free(gpose); free(geul);
    return L;
}
