"""Thin host code for rigid-body constraints (Stage 3; Alg. 1) — numpy.

The north star keeps the geometric-consistency check and the rigid-body outlier rejection on the
host; they are O(E) per frame and never on the data path.

* `kabsch`          — least-squares R, t with det R = +1 from corresponded points.
* `ransac_rigid`    — modified RANSAC: minimal samples are pre-checked by their pairwise edge
                      lengths against the template before any SVD, then Kabsch;
                      returns (R, t, inlier mask) (Stage 3 output X_B^corr and I).
* `trajectory_outliers` — geometric consistency of a freehand sweep: frames whose pose departs
                      from a robust local fit of their neighbours (R14: every frame is a view of the
                      same rigid array, and the hand moves smoothly).
* `reinit_from_neighbours` — rigid re-initialisation of outlier frames from inlier neighbours
                      (translation: local linear fit; rotation: chordal mean = SVD projection).
"""
from __future__ import annotations

import math

import numpy as np


def kabsch(A: np.ndarray, B: np.ndarray, w: np.ndarray | None = None):
    """R, t minimising sum_i w_i |R A_i + t - B_i|^2 with R in SO(3) (reflections excluded)."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    w = np.ones(len(A)) if w is None else np.asarray(w, dtype=np.float64)
    ws = w.sum()
    ca = (w[:, None] * A).sum(0) / ws
    cb = (w[:, None] * B).sum(0) / ws
    H = ((A - ca) * w[:, None]).T @ (B - cb)
    U, _, Vt = np.linalg.svd(H)
    d = np.sign(np.linalg.det(Vt.T @ U.T))
    D = np.diag([1.0, 1.0, d if d != 0 else 1.0])
    R = Vt.T @ D @ U.T
    t = cb - R @ ca
    return R, t


def ransac_rigid(X: np.ndarray, tmpl: np.ndarray, thr: float, edge_tol: float, iters: int = 200,
                 seed: int = 0, min_inliers: int = 3):
    """Modified RANSAC of Stage 3: X (n,3) noisy positions, tmpl (n,3) template (same order).
    A random minimal triple is rejected before SVD unless its three pairwise distances match the
    template's within `edge_tol` (geometric-consistency pre-check).  Returns
    (R, t, inliers) refined by Kabsch on the best consensus set, or (None, None, mask) if none."""
    X = np.asarray(X, dtype=np.float64)
    T = np.asarray(tmpl, dtype=np.float64)
    n = len(X)
    rng = np.random.default_rng(seed)
    best = None
    best_n = -1
    if n < 3:
        return None, None, np.zeros(n, bool)
    for _ in range(iters):
        idx = rng.choice(n, 3, replace=False)
        ok = True
        for a, b in ((0, 1), (0, 2), (1, 2)):
            dx = np.linalg.norm(X[idx[a]] - X[idx[b]])
            dt = np.linalg.norm(T[idx[a]] - T[idx[b]])
            if abs(dx - dt) > edge_tol:
                ok = False
                break
        if not ok:
            continue
        # degenerate (collinear) triples carry no roll information; Kabsch still gives a valid
        # least-squares rotation, the consensus step decides
        R, t = kabsch(T[idx], X[idx])
        res = np.linalg.norm(T @ R.T + t - X, axis=1)
        inl = res < thr
        if inl.sum() > best_n:
            best_n = int(inl.sum())
            best = inl
    if best is None or best_n < min_inliers:
        return None, None, np.zeros(n, bool)
    R, t = kabsch(T[best], X[best])
    res = np.linalg.norm(T @ R.T + t - X, axis=1)
    inl = res < thr
    R, t = kabsch(T[inl], X[inl])
    return R, t, inl


def rot_angle(Ra: np.ndarray, Rb: np.ndarray) -> float:
    c = (np.trace(Ra.T @ Rb) - 1.0) / 2.0
    return float(math.acos(max(-1.0, min(1.0, c))))


def euler_to_R(e) -> np.ndarray:
    a, b, c = e[0], e[1], e[2]
    Rz = np.array([[math.cos(a), -math.sin(a), 0], [math.sin(a), math.cos(a), 0], [0, 0, 1.0]])
    Ry = np.array([[math.cos(b), 0, math.sin(b)], [0, 1.0, 0], [-math.sin(b), 0, math.cos(b)]])
    Rx = np.array([[1.0, 0, 0], [0, math.cos(c), -math.sin(c)], [0, math.sin(c), math.cos(c)]])
    return Rz @ Ry @ Rx


def R_to_euler(R: np.ndarray) -> np.ndarray:
    """Inverse of Rz(a) Ry(b) Rx(c) (ZYX intrinsic, R8), away from gimbal lock (|b| < pi/2)."""
    b = -math.asin(max(-1.0, min(1.0, R[2, 0])))
    a = math.atan2(R[1, 0], R[0, 0])
    c = math.atan2(R[2, 1], R[2, 2])
    return np.array([a, b, c])


def element_positions(euler_t: np.ndarray, tmpl: np.ndarray) -> np.ndarray:
    """[F][E][3] = R_f tmpl_e + t_f."""
    out = np.zeros((euler_t.shape[0], tmpl.shape[0], 3))
    for f in range(euler_t.shape[0]):
        out[f] = tmpl @ euler_to_R(euler_t[f, :3]).T + euler_t[f, 3:]
    return out


def _local_residuals(X: np.ndarray, excl: np.ndarray, half: int) -> np.ndarray:
    """Mean element distance of each frame from a local linear fit (over frame index) of its
    non-excluded neighbours within +-half frames (the frame itself never included)."""
    F = X.shape[0]
    res = np.zeros(F)
    for f in range(F):
        nb = [g for g in range(max(0, f - half), min(F, f + half + 1)) if g != f and not excl[g]]
        if len(nb) < 2:
            continue
        s = np.asarray(nb, dtype=np.float64) - f
        A = np.stack([np.ones_like(s), s], 1)
        coef, *_ = np.linalg.lstsq(A, X[nb], rcond=None)
        res[f] = np.linalg.norm((coef[0] - X[f]).reshape(-1, 3), axis=1).mean()
    return res


def trajectory_outliers(euler_t: np.ndarray, tmpl: np.ndarray, half: int = 3, k: float = 6.0,
                        floor_mm: float = 0.3, max_frac: float = 0.3) -> np.ndarray:
    """Geometric consistency of the sweep: a frame is inconsistent if its element positions depart
    from a local linear fit of its consistent neighbours by more than
    max(median + k * 1.4826 MAD, floor_mm).  Greedy: the worst frame is flagged, excluded from its
    neighbours' fits, and the residuals recomputed, until none exceeds the threshold."""
    X = element_positions(euler_t, tmpl).reshape(euler_t.shape[0], -1)
    F = X.shape[0]
    bad = np.zeros(F, bool)
    for _ in range(int(max_frac * F) + 1):
        res = _local_residuals(X, bad, half)
        ok = res[~bad]
        med = np.median(ok)
        mad = np.median(np.abs(ok - med)) + 1e-12
        thr = max(med + k * 1.4826 * mad, floor_mm)
        cand = np.where(~bad & (res > thr), res, -1.0)
        f = int(np.argmax(cand))
        if cand[f] < 0:
            break
        bad[f] = True
    return bad


def rotation_mean(Rs) -> np.ndarray:
    """Chordal L2 mean of rotations: the SO(3) projection (Kabsch/SVD) of their arithmetic mean."""
    M = np.sum(np.asarray(Rs, dtype=np.float64), axis=0)
    U, _, Vt = np.linalg.svd(M)
    D = np.diag([1.0, 1.0, np.sign(np.linalg.det(U @ Vt)) or 1.0])
    return U @ D @ Vt


def reinit_from_neighbours(euler_t: np.ndarray, bad: np.ndarray, half: int = 3) -> np.ndarray:
    """Rigid re-initialisation of every `bad` frame from its good neighbours: translation from a
    local linear fit over frame index, rotation = chordal mean of the neighbours' rotations (a
    Kabsch-style SO(3) projection, which also fixes the roll a linear array cannot observe)."""
    out = euler_t.copy()
    F = euler_t.shape[0]
    good = ~bad
    gidx = np.nonzero(good)[0]
    if len(gidx) < 2:
        return out
    for f in np.nonzero(bad)[0]:
        nb = [g for g in range(max(0, f - half), min(F, f + half + 1)) if good[g]]
        if len(nb) < 2:
            nb = list(gidx[np.argsort(np.abs(gidx - f))[:2]])
        s = np.asarray(nb, dtype=np.float64) - f
        A = np.stack([np.ones_like(s), s], 1)
        coef, *_ = np.linalg.lstsq(A, euler_t[nb, 3:], rcond=None)
        out[f, 3:] = coef[0]
        out[f, :3] = R_to_euler(rotation_mean([euler_to_R(euler_t[g, :3]) for g in nb]))
    return out
