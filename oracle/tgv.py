"""TGV^2 regulariser of Eq. 2 — fp64 numpy oracle.  TEST INFRASTRUCTURE ONLY.

The paper names "Total Generalized Variation (TGV)" with no order, weights, discretisation or
smoothing.  Reading R20: second-order TGV with an auxiliary vector field w
(SPEC S:201-209):

    L(P, w) = a1 * sum_{x in O} phi(grad P(x) - w(x))  +  a0 * sum_{x in O} phi(E w(x))
    phi(v)  = sqrt(|v|^2 + eps^2) - eps                 (smoothed norm, phi(0) = 0)
    (grad P)_d(x) = (P(x + e_d) - P(x)) / h             (forward differences)
    (E w)_{ab}(x) = ((d_a w_b)(x) + (d_b w_a)(x)) / 2    (symmetrised gradient, forward diffs)
    |E w|^2 = sum_{a,b} (E w)_{ab}^2                     (Frobenius; off-diagonals twice)
    O = {x : 0 <= x_d <= n_d - 2}                        (all forward differences defined)

so affine P with w = grad P (constant) is in the null space exactly.  Arrays: P [nz][ny][nx],
w [3][nz][ny][nx] (component d = x, y, z).  Returns the value and the analytic gradients; the
gradients are pinned by central finite differences of the value in tests.
"""
from __future__ import annotations

import numpy as np


def _fd(A: np.ndarray, d: int, h: float) -> np.ndarray:
    """forward difference along axis d of a [nz][ny][nx] array, restricted to O."""
    ax = {0: 2, 1: 1, 2: 0}[d]  # component x -> array axis 2
    lo = [slice(0, -1)] * 3      # x over O (O trims the last index of every axis)
    sl_hi = [slice(0, -1)] * 3   # x + e_d over O
    sl_hi[ax] = slice(1, None)
    return (A[tuple(sl_hi)] - A[tuple(lo)]) / h


def tgv(P: np.ndarray, w: np.ndarray, h: float, a1: float, a0: float, eps: float):
    P = np.asarray(P, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    nz, ny, nx = P.shape
    if min(nz, ny, nx) < 2:
        return 0.0, np.zeros_like(P), np.zeros_like(w)
    Ocut = (slice(0, -1),) * 3
    # first-order term
    g = np.stack([_fd(P, d, h) - w[d][Ocut] for d in range(3)])          # [3][O]
    ng = np.sqrt((g * g).sum(0) + eps * eps)
    val1 = float((ng - eps).sum())
    n = g / ng                                                            # dphi/dg
    # second-order term: D[a][b] = d_a w_b over O
    D = np.stack([np.stack([_fd(w[b], a, h) for b in range(3)]) for a in range(3)])   # [a][b][O]
    Ew = 0.5 * (D + D.transpose(1, 0, 2, 3, 4))
    ne = np.sqrt((Ew * Ew).sum((0, 1)) + eps * eps)
    val0 = float((ne - eps).sum())
    m = Ew / ne                                                           # dphi/dEw [a][b][O]
    # gradients by the adjoint of the forward difference
    gP = np.zeros_like(P)
    gw = np.zeros_like(w)
    for d in range(3):
        ax = {0: 2, 1: 1, 2: 0}[d]
        hi = [slice(0, -1)] * 3
        hi[ax] = slice(1, None)
        gP[tuple(hi)] += a1 * n[d] / h
        gP[Ocut] -= a1 * n[d] / h
        gw[d][Ocut] -= a1 * n[d]
    # d/dw_b of sum phi(Ew): dEw_ab/d(d_a w_b) = 1/2 and dEw_ba/d(d_a w_b) = 1/2 -> m_ab (symmetric)
    for a in range(3):
        ax = {0: 2, 1: 1, 2: 0}[a]
        hi = [slice(0, -1)] * 3
        hi[ax] = slice(1, None)
        for b in range(3):
            coef = a0 * m[a][b] / h
            gw[b][tuple(hi)] += coef
            gw[b][Ocut] -= coef
    return a1 * val1 + a0 * val0, gP, gw
