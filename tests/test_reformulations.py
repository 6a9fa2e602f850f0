"""CPU pins (fp64 numpy, no CUDA) of the two reformulations the Gaussian kernels evaluate (DESIGN.md §6,
reading R24), each checked against the oracle's plain definition on small seeded cases:

* deposit form of the forward (K1d): every main tap k in [-MA, L_min-MA) of a pair's window (centre
  j_m = jlo + MA) is in-window, so the pair's contribution is c * G(D_m, k); with a rank-R basis of the
  pulse family, the pair deposits c * phi_m(D_m) at position pos = j_m + OFF and the trace is the per-row
  correlation y[j] = sum_q sum_m Q_m[j+q] psi_m(OFF-q) + Q_X[j] (the optional last tap, L = L_min + 1);
* moment-filter form of the adjoint (K2a/K2c): sum_k g[j_m+k] D_k E_k = u_m (D_m S0 - a S1) with
  S_n = sum_m dl^m/m! F_{n+m}[j_m], F_p[j] = sum_k g[j+k] C_k e^{lam0 k} k^p (+ the optional last tap).

These pin the window construction, the centre/offset bookkeeping, the last-tap handling and the
truncation orders independently of the CUDA code (which shares nothing with this file)."""
import math

import numpy as np
import pytest

import oracle
from paper_2604_09643_b200 import gen

A_MM = 1.5 * 0.025  # c dt


def scene(seed, sigma=0.2, nt=260, t0=0.4):
    grid = gen.make_grid((8, 7, 6), sigma)
    acq = gen.make_acq(nt, sigma, t0=t0)
    rng = np.random.default_rng(seed)
    E, F = 3, 2
    tmpl = rng.normal(size=(E, 3)) * 1.0
    e = np.zeros((F, 6))
    e[:, :3] = rng.normal(scale=0.3, size=(F, 3))
    e[:, 3:5] = rng.normal(scale=0.5, size=(F, 2))
    e[:, 5] = grid["origin"][2] - 2.5 - rng.uniform(0, 1, size=F)
    poses = gen.poses_from_euler(e)
    p0 = gen.random_volume(grid, seed + 1)
    return grid, acq, tmpl, poses, p0


def pairs(grid, acq, tmpl, poses):
    """Per (frame, element, voxel): r and the literal window [jlo, jlo + L) of |r - c t_j| <= kappa sigma."""
    nx, ny, nz = grid["nx"], grid["ny"], grid["nz"]
    o, h = np.asarray(grid["origin"], float), grid["pitch"]
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    y = o + h * np.stack([ii, jj, kk], -1).reshape(-1, 3)
    vid = (kk * ny * nx + jj * nx + ii).reshape(-1)
    x = oracle.place(tmpl, poses)  # [F][E][3]
    ks = acq["kappa"] * acq["sigma"]
    out = []
    for f in range(x.shape[0]):
        for e in range(x.shape[1]):
            r = np.linalg.norm(y - x[f, e], axis=1)
            base = r - acq["c"] * acq["t0"]
            jlo = np.ceil((base - ks) / A_MM).astype(int)
            jhi = np.floor((base + ks) / A_MM).astype(int)
            out.append((f, e, r, jlo, jhi - jlo + 1, vid))
    return out


def pulse(D, s):
    return D * np.exp(-D * D / (2 * s * s))


@pytest.mark.parametrize("sigma", [0.2, 0.1])
def test_deposit_form_forward_equals_definition(sigma):
    grid, acq, tmpl, poses, p0 = scene(3, sigma=sigma, t0=0.6)
    nt, s, ks = acq["nt"], sigma, acq["kappa"] * sigma
    lmin = int(math.floor(2 * ks / A_MM))
    ma, off = (lmin + 1) // 2, lmin - (lmin + 1) // 2
    k = np.arange(-ma, lmin - ma)
    # rank-R orthonormal basis psi_m(k) of the pulse family over the D_m interval (numpy SVD)
    dm_grid = np.linspace(ks - (ma + 1) * A_MM, ks - ma * A_MM, 801)
    Gm = pulse(dm_grid[:, None] - k[None, :] * A_MM, s)
    psi = np.linalg.svd(Gm, full_matrices=False)[2][:7]  # rank 7: below the oracle's fp64 noise here
    nj = nt + lmin
    F = poses.shape[0]
    y = np.zeros((F, tmpl.shape[0], nt))
    p = p0.reshape(-1)
    for f, e, r, jlo, L, vid in pairs(grid, acq, tmpl, poses):
        L = np.clip(L, lmin, lmin + 1)
        Q = np.zeros((nj, 8))
        c = p[vid] / (2 * r)
        jm = jlo + ma
        Dm = (r - acq["c"] * acq["t0"]) - jm * A_MM
        pos = jm + off
        ok = (pos >= 0) & (pos < nj)
        # main taps: every k in [-ma, lmin - ma) is in-window (the window construction)
        Dk = Dm[:, None] - k[None, :] * A_MM
        assert np.all(np.abs(Dk) <= ks * (1 + 1e-12))
        coef = pulse(Dk, s) @ psi.T  # phi_m(D_m): projection on the basis
        np.add.at(Q[:, :7], pos[ok], (c[:, None] * coef)[ok])
        # the optional last tap (L = lmin + 1) at j = jlo + lmin = pos
        Dx = Dm - (lmin - ma) * A_MM
        np.add.at(Q[:, 7], pos[ok], np.where(L[ok] == lmin + 1, c[ok] * pulse(Dx[ok], s), 0.0))
        for j in range(nt):
            qs = np.arange(1, lmin + 1)
            y[f, e, j] = np.sum(Q[j + qs, :7] * psi[:, lmin - qs].T) + Q[j, 7]  # column = k + MA, k = OFF - q
    yo = oracle.forward(grid, acq, tmpl, poses, p0)
    err = np.linalg.norm(y - yo) / np.linalg.norm(yo)
    print("deposit-form rel err", err)
    assert err < 1e-9, err


@pytest.mark.parametrize("sigma,M", [(0.2, 5), (0.1, 7)])
def test_moment_filter_adjoint_equals_definition(sigma, M):
    grid, acq, tmpl, poses, _ = scene(5, sigma=sigma, t0=0.6)
    nt, s, ks = acq["nt"], sigma, acq["kappa"] * sigma
    lmin = int(math.floor(2 * ks / A_MM))
    ma = (lmin + 1) // 2
    kt = lmin - ma
    cot = gen.random_cotangent((poses.shape[0], tmpl.shape[0], nt), 6)
    lam_s = A_MM / (s * s)
    lam0 = lam_s * A_MM * (ks / A_MM - ma - 0.5)
    k = np.arange(-ma, lmin - ma)
    Ck = np.exp(-k * k * A_MM * A_MM / (2 * s * s))
    z = np.zeros(grid["nx"] * grid["ny"] * grid["nz"])
    for f, e, r, jlo, L, vid in pairs(grid, acq, tmpl, poses):
        L = np.clip(L, lmin, lmin + 1)
        g = np.zeros(nt + 2 * lmin + 2)
        g[lmin + 1:lmin + 1 + nt] = cot[f, e]  # zero-padded: index j -> j + lmin + 1
        jm = jlo + ma
        valid = (jlo <= nt - 1) & (jlo + L - 1 >= 0)
        jm_c = np.clip(jm, -ma, nt + ma)
        # per-row filters F_p[j_m] = sum_k g[j_m + k] C_k e^{lam0 k} k^p
        W = g[(jm_c[:, None] + k[None, :]) + lmin + 1]
        Fp = np.stack([(W * (Ck * np.exp(lam0 * k) * k.astype(float) ** p)).sum(1) for p in range(M + 2)], 1)
        Dm = (r - acq["c"] * acq["t0"]) - jm * A_MM
        dl = lam_s * Dm - lam0
        S = [sum(dl ** m / math.factorial(m) * Fp[:, n + m] for m in range(M + 1)) for n in range(2)]
        um = np.exp(-Dm * Dm / (2 * s * s))
        A1 = um * (Dm * S[0] - A_MM * S[1])
        # the optional last tap
        jx = jlo + lmin
        gx = np.where((L == lmin + 1) & (jx >= 0) & (jx < nt), g[np.clip(jx, -lmin - 1, nt + lmin) + lmin + 1], 0.0)
        A1 = A1 + gx * pulse(Dm - kt * A_MM, s)
        np.add.at(z, vid[valid], (A1 / (2 * r))[valid])
    zo = oracle.adjoint(grid, acq, tmpl, poses, cot).reshape(-1)
    err = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    print("moment-filter rel err", err)
    assert err < 5e-7, err
