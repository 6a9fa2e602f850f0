"""Pins for the TGV^2 oracle (reading R20 of Eq. 2's regulariser) — CPU."""
import numpy as np

from oracle.tgv import tgv


def grid_coords(n, h):
    z, y, x = np.meshgrid(np.arange(n[0]), np.arange(n[1]), np.arange(n[2]), indexing="ij")
    return x * h, y * h, z * h


def test_null_space_constant_and_affine():
    h = 0.2
    P = np.full((5, 6, 7), 0.3)
    v, gP, gw = tgv(P, np.zeros((3, 5, 6, 7)), h, 1.0, 2.0, 1e-6)
    assert v == 0.0 and np.abs(gP).max() == 0 and np.abs(gw).max() == 0
    X, Y, Z = grid_coords((5, 6, 7), h)
    P = 0.7 * X - 0.4 * Y + 0.1 * Z + 2.0
    w = np.stack([np.full(P.shape, 0.7), np.full(P.shape, -0.4), np.full(P.shape, 0.1)])
    v, gP, gw = tgv(P, w, h, 1.0, 2.0, 1e-6)
    # the smoothed norm has gradient g/eps at rounding-level residuals g ~ 1e-16: bound it by 1e-6
    assert abs(v) < 1e-12 and np.abs(gP).max() < 1e-6 and np.abs(gw).max() < 1e-6


def test_infinitesimal_rotation_field_has_zero_symmetric_gradient():
    h = 0.25
    X, Y, Z = grid_coords((4, 5, 6), h)
    w = np.stack([-Y, X, np.zeros_like(X)])  # d_x w_y = 1, d_y w_x = -1 -> E w = 0
    P = np.zeros(X.shape)
    v0 = tgv(P, w, h, 0.0, 1.0, 1e-9)[0]
    assert abs(v0) < 1e-12


def test_step_edge_closed_form():
    h, eps, a1 = 0.2, 1e-3, 1.5
    n = (6, 5, 8)
    P = np.zeros(n)
    P[:, :, 4:] = 1.0  # jump between x = 3 and x = 4
    v, _, _ = tgv(P, np.zeros((3,) + n), h, a1, 2.0, eps)
    want = a1 * (n[0] - 1) * (n[1] - 1) * (np.sqrt(1.0 / h ** 2 + eps ** 2) - eps)
    assert abs(v - want) <= 1e-12 * want


def test_gradients_vs_central_differences():
    rng = np.random.default_rng(0)
    n = (4, 5, 6)
    h, a1, a0, eps = 0.3, 1.2, 0.7, 5e-2
    P = rng.normal(size=n)
    w = rng.normal(size=(3,) + n)
    v, gP, gw = tgv(P, w, h, a1, a0, eps)
    d = 1e-6
    for idx in [(0, 0, 0), (1, 2, 3), (3, 4, 5), (2, 0, 5)]:
        Pp, Pm = P.copy(), P.copy()
        Pp[idx] += d
        Pm[idx] -= d
        fd = (tgv(Pp, w, h, a1, a0, eps)[0] - tgv(Pm, w, h, a1, a0, eps)[0]) / (2 * d)
        assert abs(fd - gP[idx]) <= 1e-6 * max(1.0, abs(gP[idx]))
    for c in range(3):
        for idx in [(0, 0, 0), (1, 2, 3), (3, 4, 5)]:
            wp, wm = w.copy(), w.copy()
            wp[(c,) + idx] += d
            wm[(c,) + idx] -= d
            fd = (tgv(P, wp, h, a1, a0, eps)[0] - tgv(P, wm, h, a1, a0, eps)[0]) / (2 * d)
            assert abs(fd - gw[(c,) + idx]) <= 1e-6 * max(1.0, abs(gw[(c,) + idx]))
