"""Pins for the fp64 oracle (runs on CPU, -m "not gpu").

Each test pins the oracle to something other than itself: a closed form printed in
the paper, an invariant of the mathematics, finite differences, or a brute-force
third implementation.  P:n = /root/reference/PAPER.md line n (citations only; nothing
here reads that file).  Pin ids (P1..P11) follow SURVEY.md §8(c) / DESIGN.md §5.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import closed_forms as cf
from paper_2604_09643_b200 import gen

C = 1.5
DT = 0.025


def grid_of(n, pitch, origin=None):
    nx, ny, nz = n
    if origin is None:
        origin = [-(nx - 1) / 2 * pitch, -(ny - 1) / 2 * pitch, -(nz - 1) / 2 * pitch]
    return dict(nx=nx, ny=ny, nz=nz, origin=list(origin), pitch=pitch)


def acq_of(nt, sigma, t0=0.0, kappa=5.0):
    return dict(c=C, t0=t0, dt=DT, nt=nt, sigma=sigma, kappa=kappa)


def ident_pose(t=(0, 0, 0)):
    p = np.zeros((1, 12))
    p[0, :9] = np.eye(3).reshape(-1)
    p[0, 9:] = t
    return p


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def times(acq):
    return acq["t0"] + acq["dt"] * np.arange(acq["nt"])


# --------------------------------------------------------------------------- P1 single blob
@pytest.mark.parametrize("kappa", [0.0, 5.0])
def test_P1_single_blob_equals_gaussian_far_field(kappa):
    """One voxel of amplitude A reproduces Eq. gaussian_far_field exactly,
    with the 1/2r factor and the sign (positive before t=r/c); with kappa=5 it is the
    same closed form multiplied by the window indicator (R4)."""
    A, sigma = 0.7, 0.2
    g = grid_of((1, 1, 1), 0.2, origin=[0.3, -0.2, 0.1])
    a = acq_of(512, sigma, kappa=kappa)
    x = np.array([[0.0, 0.0, 0.0]])
    pose = ident_pose(t=(2.0, 5.0, -6.0))
    y = oracle.forward(g, a, x, pose, np.array([A]))[0, 0]
    r = math.dist((2.0, 5.0, -6.0), (0.3, -0.2, 0.1))
    t = times(a)
    want = cf.gaussian_far_field(r, t, A, sigma, C)
    if kappa > 0:
        want = np.where(np.abs(r - C * t) <= kappa * sigma, want, 0.0)
    assert np.max(np.abs(y - want)) <= 1e-12 * np.max(np.abs(want))
    # zero crossing at t = r/c: positive just before, negative just after
    j0 = int(r / (C * DT))
    assert y[j0] > 0 and y[j0 + 1] < 0


# --------------------------------------------------------------------------- P2 Gaussian ball
def gaussian_ball_amplitudes(grid, c0, s, sigma, A):
    """P_k = B exp(-|y_k - c0|^2 / 2 tau^2), tau^2 = s^2 - sigma^2,
    B = A s^3 h^3 / ((2 pi)^{3/2} tau^3 sigma^3)  (R2: blob-lattice amplitudes)."""
    h = grid["pitch"]
    tau = math.sqrt(s * s - sigma * sigma)
    B = A * s ** 3 * h ** 3 / ((2 * math.pi) ** 1.5 * tau ** 3 * sigma ** 3)
    xs = grid["origin"][0] + h * np.arange(grid["nx"])
    ys = grid["origin"][1] + h * np.arange(grid["ny"])
    zs = grid["origin"][2] + h * np.arange(grid["nz"])
    d2 = ((zs[:, None, None] - c0[2]) ** 2 + (ys[None, :, None] - c0[1]) ** 2 + (xs[None, None, :] - c0[0]) ** 2)
    return B * np.exp(-d2 / (2 * tau * tau))


def test_P2_gaussian_ball_trace_matches_gaussian_solution():
    """A blob lattice sampling a Gaussian ball of total width s reproduces Eq.
    gaussian_solution with sigma -> s (dense mode)."""
    sigma, s, A = 0.2, 0.55, 1.3
    g = grid_of((32, 32, 32), 0.2)
    a = acq_of(512, sigma, kappa=0.0)
    c0 = np.array([0.05, -0.03, 0.02])
    P = gaussian_ball_amplitudes(g, c0, s, sigma, A)
    tmpl = np.array([[0.0, 0.0, 0.0], [2.0, 1.0, 0.5], [-3.0, 0.5, 1.0]])
    pose = ident_pose(t=(0.5, 0.2, -9.0))
    y = oracle.forward(g, a, tmpl, pose, P)[0]
    pos = oracle.place(tmpl, pose)[0]
    t = times(a)
    for e in range(3):
        Re = np.linalg.norm(pos[e] - c0)
        want = cf.gaussian_solution(Re, t, A, s, C)
        assert np.max(np.abs(y[e] - want)) <= 3e-6 * np.max(np.abs(want))


def test_P2_gaussian_ball_element_gradient_closed_form():
    """Element gradient of L = <g, y> against the radial derivative of Eq. gaussian_solution's
    outgoing term: dL/dx_e = sum_j g_j d/dR[A/(2R)(R-ct)e^{-(R-ct)^2/2s^2}] (x_e-c0)/R."""
    sigma, s, A = 0.2, 0.55, 1.3
    g = grid_of((32, 32, 32), 0.2)
    a = acq_of(512, sigma, kappa=0.0)
    c0 = np.array([0.05, -0.03, 0.02])
    P = gaussian_ball_amplitudes(g, c0, s, sigma, A)
    tmpl = np.array([[0.0, 0.0, 0.0], [2.0, 1.0, 0.5]])
    pose = ident_pose(t=(0.5, 0.2, -9.0))
    pos = oracle.place(tmpl, pose)[0]
    t = times(a)
    # a residual-like cotangent (the trace itself) and a white one; the white one cancels
    # heavily in the sum over j, so its error is measured against sum_j |g_j dp/dR|.
    for cot, tol in ((oracle.forward(g, a, tmpl, pose, P), 1e-7), (gen.random_cotangent((1, 2, 512), seed=3), 1e-5)):
        G = oracle.elem_grad(g, a, tmpl, pose, P, cot)[0]
        for e in range(2):
            u = pos[e] - c0
            R = np.linalg.norm(u)
            D = R - C * t
            dpdR = A * np.exp(-D * D / (2 * s * s)) / (2 * R) * ((1 - D * D / (s * s)) - D / R)
            want = np.sum(cot[0, e] * dpdR) * u / R
            scale = np.sum(np.abs(cot[0, e] * dpdR))
            assert np.linalg.norm(G[e] - want) <= tol * scale


# --------------------------------------------------------------------------- P3 uniform sphere
def test_P3_uniform_sphere_north_star_pin():
    """Partial-volume uniform ball (R=2 mm, sigma=h) against the boxed Eq. applied to
    the sigma-smoothed ball, and in the interior against the uniform-sphere N-pulse
    p = p0 (r - ct)/(2r).  Coarse pin: catches factor-2, c, t0 and sign errors."""
    h = sigma = 0.2
    Rb, p0v = 2.0, 1.0
    g = grid_of((32, 32, 32), h)
    a = acq_of(512, sigma, kappa=5.0)
    frac = gen.sphere_fraction(g, (0.0, 0.0, 0.0), Rb, ss=4)
    P = p0v * frac * h ** 3 / ((2 * math.pi) ** 1.5 * sigma ** 3)
    tmpl = np.array([[0.0, 0.0, 0.0], [4.0, 3.0, 0.0]])
    pose = ident_pose(t=(0.0, 0.0, -9.0))
    y = oracle.forward(g, a, tmpl, pose, P)[0]
    pos = oracle.place(tmpl, pose)[0]
    t = times(a)
    for e in range(2):
        r = np.linalg.norm(pos[e])
        want = cf.boxed(r, t, lambda rho: cf.smoothed_ball_profile(rho, Rb, p0v, sigma), C)
        band = np.abs(r - C * t) < Rb + 6 * sigma
        assert rel(y[e][band], want[band]) <= 1.5e-2
        interior = np.abs(r - C * t) < Rb - 4 * sigma
        sphere = cf.uniform_sphere(r, t, p0v, Rb, C)
        peak = np.max(np.abs(sphere))
        assert np.max(np.abs(y[e][interior] - sphere[interior])) <= 6e-3 * peak


# --------------------------------------------------------------------------- P4 closed-form pins
def test_P4_boxed_vs_far_field_and_quadrature():
    """The closed forms used as pins are themselves pinned: boxed vs far field at r >= 20 s
    (P:325-329), Gaussian/exponential/power-law boxed expressions vs a numerical shell
    integral of Eq. pressure_simplified, uniform sphere zero outside support."""
    s = 0.2
    for r in (20 * s, 40 * s, 100 * s):
        t = np.linspace((r - 5 * s) / C, (r + 5 * s) / C, 101)
        full = cf.gaussian_solution(r, t, 1.0, s, C)
        ff = cf.gaussian_far_field(r, t, 1.0, s, C)
        assert np.max(np.abs(full - ff)) <= 1e-6 * np.max(np.abs(full))
        assert np.allclose(cf.boxed(r, t, lambda x: np.exp(-x * x / (2 * s * s)), C), full, rtol=0, atol=1e-14)
        assert np.allclose(cf.far_field(r, t, lambda x: np.exp(-x * x / (2 * s * s)), C), ff, rtol=0, atol=1e-14)
    r = 1.5
    for tt in (0.6, 0.95, 1.2):
        q = cf.shell_integral_pressure(r, tt, lambda x: np.exp(-x * x / (2 * 0.4 ** 2)), C)
        assert abs(q - cf.gaussian_solution(r, tt, 1.0, 0.4, C)) <= 1e-4 * 1.0
        q = cf.shell_integral_pressure(r, tt, lambda x: np.exp(-x / 0.3), C)
        assert abs(q - cf.exponential_solution(r, tt, 1.0, 0.3, C)) <= 1e-4
        q = cf.shell_integral_pressure(r, tt, lambda x: 1.0 / (x * x + 0.25) ** 1.5, C)
        assert abs(q - cf.power_law_solution(r, tt, 1.0, 0.5, 1.5, C)) <= 1e-3
    rr = np.full(1000, 7.0)
    tt = np.linspace(0, 10, 1000)
    u = cf.uniform_sphere(rr, tt, 2.0, 1.0, C)
    outside = (C * tt < 6.0) | (C * tt > 8.0)
    assert np.all(u[outside] == 0.0)
    inside = ~outside
    assert np.allclose(u[inside], 2.0 / 14.0 * (7.0 - C * tt[inside]), atol=1e-12, rtol=0)


# --------------------------------------------------------------------------- P5 adjoint identity
@pytest.mark.parametrize("kappa", [0.0, 5.0])
def test_P5_linearity_and_adjoint_identity(kappa):
    g = grid_of((6, 5, 7), 0.2)
    a = acq_of(160, 0.2, t0=1.0, kappa=kappa)
    rng = np.random.default_rng(0)
    tmpl = rng.normal(size=(3, 3))
    e = np.zeros((2, 6))
    e[:, :3] = rng.normal(scale=0.3, size=(2, 3))
    e[:, 3:] = rng.normal(scale=1.0, size=(2, 3)) + np.array([0, 0, -4.0])
    poses = gen.poses_from_euler(e)
    x1, x2 = gen.random_volume(g, 1), gen.random_volume(g, 2)
    yy = rng.normal(size=(2, 3, 160))
    A1 = oracle.forward(g, a, tmpl, poses, x1)
    A2 = oracle.forward(g, a, tmpl, poses, x2)
    A12 = oracle.forward(g, a, tmpl, poses, 2.0 * x1 - 3.0 * x2)
    assert rel(A12, 2.0 * A1 - 3.0 * A2) <= 1e-13
    lhs = np.sum(A1 * yy)
    rhs = np.sum(x1 * oracle.adjoint(g, a, tmpl, poses, yy))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    assert np.all(oracle.adjoint(g, a, tmpl, poses, np.zeros_like(yy)) == 0.0)
    assert np.all(oracle.forward(g, a, tmpl, poses, np.zeros_like(x1)) == 0.0)


# --------------------------------------------------------------------------- P6 finite differences
def _loss(g, a, tmpl, poses, p0, cot):
    return float(np.sum(cot * oracle.forward(g, a, tmpl, poses, p0)))


def test_P6_element_and_pose_gradients_vs_central_differences():
    """Dense mode (R11): central FD at 1e-4 mm for element positions, translations and
    rotation generators, against oracle_elem_grad / pose chain rule."""
    g = grid_of((8, 8, 8), 0.2)
    a = acq_of(384, 0.2, t0=0.5, kappa=0.0)
    rng = np.random.default_rng(5)
    p0 = gen.random_volume(g, 7)
    tmpl = np.array([[-0.6, 0.1, 0.0], [0.2, -0.3, 0.1], [0.9, 0.4, -0.2]])
    e = np.array([[0.2, -0.1, 0.15, 0.3, -0.4, -5.0]])
    poses = gen.poses_from_euler(e)
    cot = rng.normal(size=(1, 3, 384))
    gpose, gel = oracle.pose_grad(g, a, tmpl, poses, p0, cot)
    hh = 1e-4
    R = poses[0, :9].reshape(3, 3)
    # element positions: perturb template entry c of element k by hh along template axis;
    # x moves by R[:, c] hh, so dL/dtmpl[k,c] = G_k . R[:, c]
    for k in range(3):
        for c in range(3):
            tp, tm = tmpl.copy(), tmpl.copy()
            tp[k, c] += hh
            tm[k, c] -= hh
            fd = (_loss(g, a, tp, poses, p0, cot) - _loss(g, a, tm, poses, p0, cot)) / (2 * hh)
            an = gel[0, k] @ R[:, c]
            assert abs(fd - an) <= 1e-6 * max(np.abs(gel).max(), 1e-30)
    # translations
    for c in range(3):
        pp, pm = poses.copy(), poses.copy()
        pp[0, 9 + c] += hh
        pm[0, 9 + c] -= hh
        fd = (_loss(g, a, tmpl, pp, p0, cot) - _loss(g, a, tmpl, pm, p0, cot)) / (2 * hh)
        assert abs(fd - gpose[0, 9 + c]) <= 1e-6 * np.abs(gpose).max()
    # rotations: R(eps) = R expm(eps [w]_x); dL/deps = <dL/dR, R [w]_x>_F
    for w in np.eye(3):
        W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
        def posed(eps):
            Rp = R @ (np.eye(3) + eps * W + 0.5 * eps * eps * W @ W + eps ** 3 / 6 * W @ W @ W)
            p = poses.copy()
            p[0, :9] = Rp.reshape(-1)
            return p
        he = 1e-6
        fd = (_loss(g, a, tmpl, posed(he), p0, cot) - _loss(g, a, tmpl, posed(-he), p0, cot)) / (2 * he)
        an = np.sum(gpose[0, :9].reshape(3, 3) * (R @ W))
        assert abs(fd - an) <= 1e-5 * np.abs(gpose).max()


def test_P6b_step_euler_gradient_vs_fd():
    """oracle_step's dL/dEuler (ZYX chain, R8) and dL/dp0 against central FD of the MSE loss."""
    g = grid_of((6, 6, 6), 0.2)
    a = acq_of(256, 0.2, t0=0.5, kappa=0.0)
    tmpl = gen.linear_array(4, 0.3)
    e = np.array([[0.1, -0.2, 0.05, 0.2, 0.1, -4.0]])
    p0 = gen.random_volume(g, 11)
    meas = oracle.forward(g, a, tmpl, gen.poses_from_euler(e + 0.01), p0 * 0.9)
    nv = p0.size
    out = oracle.step(g, a, tmpl, meas, p0, e, np.zeros(2 * nv), np.zeros(12), lr_p0=0, lr_rot=0, lr_trans=0,
                      update_p0=False, update_pose=False)
    def L(ee, pp):
        return float(np.sum((oracle.forward(g, a, tmpl, gen.poses_from_euler(ee), pp) - meas) ** 2))
    assert abs(out["loss"] - L(e, p0)) <= 1e-12 * out["loss"]
    for q in range(6):
        h = 1e-6 if q < 3 else 1e-4
        ep, em = e.copy(), e.copy()
        ep[0, q] += h
        em[0, q] -= h
        fd = (L(ep, p0) - L(em, p0)) / (2 * h)
        assert abs(fd - out["grad_euler"][0, q]) <= 2e-5 * np.abs(out["grad_euler"]).max()
    for k in (0, 37, 100, 215):
        pp, pm = p0.copy().reshape(-1), p0.copy().reshape(-1)
        pp[k] += 1e-3
        pm[k] -= 1e-3
        fd = (L(e, pp) - L(e, pm)) / 2e-3
        assert abs(fd - out["grad_p0"][k]) <= 1e-7 * np.abs(out["grad_p0"]).max()


# --------------------------------------------------------------------------- P7 invariances
def test_P7_rigid_motion_invariance():
    g = grid_of((7, 6, 5), 0.2)
    a = acq_of(200, 0.2, t0=1.0)
    rng = np.random.default_rng(3)
    tmpl = rng.normal(size=(4, 3))
    e = np.array([[0.3, 0.1, -0.2, 0.5, 0.2, -4.5]])
    poses = gen.poses_from_euler(e)
    p0 = gen.random_volume(g, 4)
    y = oracle.forward(g, a, tmpl, poses, p0)
    # translation of the whole scene
    v = np.array([1.25, -0.5, 2.0])
    g2 = dict(g, origin=list(np.asarray(g["origin"]) + v))
    p2 = poses.copy()
    p2[0, 9:] += v
    assert rel(oracle.forward(g2, a, tmpl, p2, p0), y) <= 1e-12
    # 90 degree rotation about z: (x, y) -> (-y, x); volume axes permuted/flipped accordingly
    Q = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    o = np.asarray(g["origin"])
    nx, ny = g["nx"], g["ny"]
    # new grid: x' = -y, y' = x ; new voxel (i', j') = (ny-1-j, i) with origin' = Q @ (o + corner)
    corner = np.array([0.0, (ny - 1) * g["pitch"], 0.0])
    g3 = dict(nx=ny, ny=nx, nz=g["nz"], origin=list(Q @ (o + corner)), pitch=g["pitch"])
    p0r = np.transpose(p0, (0, 2, 1))[:, :, ::-1]   # [z][x][y] -> [z][j'=i][i'=ny-1-j]
    p3 = poses.copy()
    R = poses[0, :9].reshape(3, 3)
    p3[0, :9] = (Q @ R).reshape(-1)
    p3[0, 9:] = Q @ poses[0, 9:]
    assert rel(oracle.forward(g3, a, tmpl, p3, p0r), y) <= 1e-12


def test_P7b_ball_rotation_invariance_and_P10_structure():
    """Rotating the array about a Gaussian ball's centre leaves each element's trace unchanged
    (to lattice ripple), and each element gradient is parallel to x_e - c0 (P10)."""
    sigma, s = 0.2, 0.55
    g = grid_of((32, 32, 32), 0.2)
    a = acq_of(400, sigma, kappa=0.0)
    c0 = np.array([0.1, 0.0, -0.1])
    P = gaussian_ball_amplitudes(g, c0, s, sigma, 1.0)
    tmpl = np.array([[0.0, 0.0, -7.0], [1.5, 0.0, -6.5]])
    def posed(Rm):
        p = np.zeros((1, 12))
        p[0, :9] = Rm.reshape(-1)
        p[0, 9:] = c0 - Rm @ c0
        return p
    y0 = oracle.forward(g, a, tmpl, posed(np.eye(3)), P)
    y1 = oracle.forward(g, a, tmpl, posed(gen.rot_zyx(0.4, -0.3, 0.7)), P)
    assert rel(y1, y0) <= 1e-5
    cot = gen.random_cotangent((1, 2, 400), 9)
    G = oracle.elem_grad(g, a, tmpl, posed(np.eye(3)), P, cot)[0]
    pos = oracle.place(tmpl, posed(np.eye(3)))[0]
    for e in range(2):
        u = (pos[e] - c0) / np.linalg.norm(pos[e] - c0)
        perp = G[e] - (G[e] @ u) * u
        assert np.linalg.norm(perp) <= 1e-6 * np.linalg.norm(G[e])


def test_P11_linear_array_roll_is_unobservable():
    """Centred linear template x_e = s_e a: rolling about a leaves every element fixed, so
    <dL/dR, R [a]_x>_F = 0 exactly (R15)."""
    g = grid_of((8, 8, 8), 0.2)
    a = acq_of(300, 0.2, t0=1.0)
    tmpl = gen.linear_array(6, 0.3)
    e = np.array([[0.2, 0.1, -0.1, 0.1, 0.3, -4.0]])
    poses = gen.poses_from_euler(e)
    p0 = gen.random_volume(g, 1)
    cot = gen.random_cotangent((1, 6, 300), 2)
    gpose, _ = oracle.pose_grad(g, a, tmpl, poses, p0, cot)
    R = poses[0, :9].reshape(3, 3)
    ax = np.array([[0, 0, 0], [0, 0, -1.0], [0, 1.0, 0]])   # [x-axis]_x
    val = np.sum(gpose[0, :9].reshape(3, 3) * (R @ ax))
    assert abs(val) <= 1e-12 * np.abs(gpose).max()


# --------------------------------------------------------------------------- P8 brute force (third implementation)
def brute(grid, acq, tmpl, poses, p0, cot):
    """Independent numpy evaluation: dense enumeration of every (voxel, element, sample) term
    with the literal predicate; returns forward, adjoint, element gradient and count."""
    h = grid["pitch"]
    o = np.asarray(grid["origin"])
    kk, jj, ii = np.meshgrid(np.arange(grid["nz"]), np.arange(grid["ny"]), np.arange(grid["nx"]), indexing="ij")
    Y = np.stack([o[0] + h * ii, o[1] + h * jj, o[2] + h * kk], -1).reshape(-1, 3)
    P = np.asarray(p0).reshape(-1)
    F, E = poses.shape[0], tmpl.shape[0]
    t = acq["t0"] + acq["dt"] * np.arange(acq["nt"])
    s2 = acq["sigma"] ** 2
    fwd = np.zeros((F, E, acq["nt"]))
    adj = np.zeros(P.size)
    adj_abs = np.zeros(P.size)
    gel = np.zeros((F, E, 3))
    cnt = 0
    for f in range(F):
        R = poses[f, :9].reshape(3, 3)
        for e in range(E):
            x = R @ tmpl[e] + poses[f, 9:]
            d = x[None, :] - Y
            r = np.sqrt((d * d).sum(1))
            D = r[:, None] - acq["c"] * t[None, :]
            m = np.abs(D) <= acq["kappa"] * acq["sigma"] if acq["kappa"] > 0 else np.ones_like(D, bool)
            Ek = np.exp(-D * D / (2 * s2)) * m
            k = D / (2 * r[:, None]) * Ek
            fwd[f, e] = P @ k
            adj += k @ cot[f, e]
            adj_abs += np.abs(k) @ np.abs(cot[f, e])
            dk = Ek / (2 * r[:, None]) * ((1 - D * D / s2) - D / r[:, None])
            dLdr = P * (dk @ cot[f, e])
            gel[f, e] = (dLdr[:, None] * d / r[:, None]).sum(0)
            cnt += int(m.sum())
    brute.adj_abs = adj_abs.reshape(np.shape(p0))
    return fwd, adj.reshape(np.shape(p0)), gel, cnt


@pytest.mark.parametrize("kappa", [5.0, 4.0, 0.0])
def test_P8_brute_force_tiny(kappa):
    g = grid_of((4, 3, 4), 0.25, origin=[-0.3, 0.2, 0.1])
    a = acq_of(96, 0.25, t0=0.7, kappa=kappa)
    rng = np.random.default_rng(21)
    tmpl = rng.normal(size=(3, 3)) * 0.5
    e = np.array([[0.1, 0.2, -0.3, 0.0, 0.5, -2.0], [-0.2, 0.0, 0.4, 1.0, -0.5, -2.5]])
    poses = gen.poses_from_euler(e)
    p0 = gen.random_volume(g, 5)
    cot = rng.normal(size=(2, 3, 96))
    bf, ba, bg, bc = brute(g, a, tmpl, poses, p0, cot)
    assert rel(oracle.forward(g, a, tmpl, poses, p0), bf) <= 1e-12
    assert rel(oracle.adjoint(g, a, tmpl, poses, cot), ba) <= 1e-12
    assert rel(oracle.elem_grad(g, a, tmpl, poses, p0, cot), bg) <= 1e-12
    za = oracle.adjoint_abs(g, a, tmpl, poses, cot)  # the per-voxel error scale of the GPU parity tests
    assert rel(za, brute.adj_abs) <= 1e-12 and np.all(za >= np.abs(ba) - 1e-15)
    if kappa > 0:
        n, pf = oracle.count(g, a, tmpl, poses)
        assert n == bc and pf.sum() == n


def test_count_matches_brute_force_on_c1_geometry():
    """Exact unit-of-work count on the C1 geometry vs numpy brute force (clipping at both ends)."""
    w = gen.workload("c1")
    g = dict(w.grid, nx=8, ny=8, nz=8)
    a = dict(w.acq, nt=200, t0=2.0)
    poses = w.poses_true()
    _, _, _, bc = brute(g, a, w.tmpl[::8], poses, np.zeros((8, 8, 8)), np.zeros((1, 8, 200)))
    n, _ = oracle.count(g, a, w.tmpl[::8], poses)
    assert n == bc


# --------------------------------------------------------------------------- P9 bipolarity
def test_P9_single_source_bipolar():
    """The N-pulse integrates to ~0 over a window containing it."""
    g = grid_of((1, 1, 1), 0.2, origin=[0, 0, 0])
    a = acq_of(1024, 0.2, kappa=6.0)
    y = oracle.forward(g, a, np.zeros((1, 3)), ident_pose(t=(0, 0, -10.0)), np.ones(1))[0, 0]
    assert abs(y.sum()) <= 1e-4 * np.abs(y).max() * 1024


# --------------------------------------------------------------------------- losses / optimiser / Euler
def test_losses_closed_forms():
    y = np.arange(12.0).reshape(3, 4)
    L, g = oracle.mse(y + 1.0, y)
    assert L == 12.0 and np.all(g == 2.0)
    L, g = oracle.mse(y, y)
    assert L == 0.0 and np.all(g == 0.0)
    rng = np.random.default_rng(0)
    s = rng.normal(size=(2, 50))
    L, _ = oracle.nc(s, s)
    assert abs(L + 2.0) <= 1e-12
    L, _ = oracle.nc(-s, s)
    assert abs(L - 2.0) <= 1e-12
    L, g = oracle.nc(3.0 * s + 1.5, s)
    assert abs(L + 2.0) <= 1e-12 and np.abs(g).max() <= 1e-10
    L, _ = oracle.nc(s, s, mask=np.array([1, 0]))
    assert abs(L + 1.0) <= 1e-12
    # NC gradient vs central FD
    y = rng.normal(size=(1, 40))
    _, g = oracle.nc(y, s[:1, :40])
    for j in (0, 7, 39):
        yp, ym = y.copy(), y.copy()
        yp[0, j] += 1e-6
        ym[0, j] -= 1e-6
        fd = (oracle.nc(yp, s[:1, :40])[0] - oracle.nc(ym, s[:1, :40])[0]) / 2e-6
        assert abs(fd - g[0, j]) <= 1e-6


def test_adam_closed_forms():
    x = np.array([1.0, -2.0, 3.0, 0.5])
    z = np.zeros(4)
    xn, m, v = oracle.adam(x, z, z, z, lr=0.1)
    assert np.all(xn == x)
    g = np.array([0.5, -2.0, 1e-3, 4.0])
    xn, m, v = oracle.adam(x, z, z, g, lr=0.1, eps=1e-8, t=1)
    # first step from a zero state: mhat = g, vhat = g^2 => x - lr g/(|g| + eps)
    assert np.allclose(xn, x - 0.1 * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-15)
    xc, _, _ = oracle.adam(x, z, z, np.array([5.0, 5.0, 5.0, 5.0]), lr=1.0, t=1, clamp=0.0)
    assert np.allclose(xc, np.maximum(x - 5.0 / (5.0 + 1e-8), 0.0), rtol=0, atol=1e-15)
    assert xc[1] == 0.0 and xc[3] == 0.0
    # 10-step trajectory on f(x) = x^2 decreases monotonically towards 0
    xs, ms, vs = np.array([1.0]), np.zeros(1), np.zeros(1)
    prev = 1.0
    for t in range(1, 11):
        xs, ms, vs = oracle.adam(xs, ms, vs, 2 * xs, lr=0.05, t=t)
        assert 0.0 < xs[0] < prev
        prev = xs[0]


def test_euler_zyx():
    R, dR = oracle.euler_zyx([0.0, 0.0, 0.0])
    assert np.allclose(R, np.eye(3), atol=0)
    # derivatives at zero are the skew generators of z, y, x
    assert np.allclose(dR[0], [[0, -1, 0], [1, 0, 0], [0, 0, 0]])
    assert np.allclose(dR[1], [[0, 0, 1], [0, 0, 0], [-1, 0, 0]])
    assert np.allclose(dR[2], [[0, 0, 0], [0, 0, -1], [0, 1, 0]])
    R, _ = oracle.euler_zyx([math.pi / 2, 0, 0])
    assert np.allclose(R @ [1, 0, 0], [0, 1, 0], atol=1e-15)
    rng = np.random.default_rng(0)
    for _ in range(20):
        e = rng.uniform(-1.5, 1.5, size=3)
        R, dR = oracle.euler_zyx(e)
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-14) and abs(np.linalg.det(R) - 1) < 1e-14
        for q in range(3):
            ep, em = e.copy(), e.copy()
            ep[q] += 1e-6
            em[q] -= 1e-6
            fd = (oracle.euler_zyx(ep)[0] - oracle.euler_zyx(em)[0]) / 2e-6
            assert np.abs(fd - dR[q]).max() <= 1e-9


def test_step_composes_and_descends():
    """oracle_step == composition of the separate oracle functions; a small Adam step lowers the
    loss; p0 stays >= 0."""
    g = grid_of((6, 6, 6), 0.2)
    a = acq_of(256, 0.2, t0=0.5)
    tmpl = gen.linear_array(4, 0.3)
    e_true = np.array([[0.1, -0.2, 0.05, 0.2, 0.1, -4.0], [0.0, 0.1, 0.0, -0.2, 0.3, -4.2]])
    p_true = gen.random_volume(g, 11)
    meas = oracle.forward(g, a, tmpl, gen.poses_from_euler(e_true), p_true)
    e0 = e_true + 0.01
    p0 = np.full_like(p_true, 0.5)
    nv = p0.size
    out = oracle.step(g, a, tmpl, meas, p0, e0, np.zeros(2 * nv), np.zeros(24), lr_p0=1e-2, lr_rot=1e-3,
                      lr_trans=1e-3)
    poses0 = gen.poses_from_euler(e0)
    y = oracle.forward(g, a, tmpl, poses0, p0)
    L, cot = oracle.mse(y, meas)
    assert abs(out["loss"] - L) <= 1e-12 * L
    assert rel(out["grad_p0"], oracle.adjoint(g, a, tmpl, poses0, cot)) <= 1e-12
    gp, _ = oracle.pose_grad(g, a, tmpl, poses0, p0, cot)
    assert rel(out["grad_pose"], gp) <= 1e-12
    assert np.all(out["p0"] >= 0.0)
    L1 = float(np.sum((oracle.forward(g, a, tmpl, gen.poses_from_euler(out["euler_t"]), out["p0"]) - meas) ** 2))
    assert L1 < L


def _adam_golden():
    import os

    rows = []
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "adam_steps.txt")) as fh:
        for ln in fh:
            if ln.strip() and not ln.startswith("#"):
                p = ln.split()
                rows.append((float(p[0]), int(p[1]), int(p[2]), float(p[3]), float(p[4]), float(p[5])))
    return rows


def test_adam_three_steps_from_nonzero_state_golden():
    """oracle.adam against tests/golden/adam_steps.txt: three steps (t = 1..3) from m0 = 0.1, v0 = 3/999,
    b1 = 0.9, b2 = 0.999, worked by hand; with and without the p0 >= 0 clamp.
    A dropped b1 m_{t-1} term or bc2 = 1 - b2 (not 1 - b2^t) fails it."""
    rows = _adam_golden()
    grads = {1: 1.0, 2: -2.0, 3: 2.0}
    for x0 in sorted({r[0] for r in rows}):
        want = [r for r in rows if r[0] == x0]
        clamp = 0.0 if want[0][1] else None
        x, m, v = np.array([x0]), np.array([0.1]), np.array([3.0 / 999.0])
        for (_, _, t, xw, mw, vw) in sorted(want, key=lambda r: r[2]):
            x, m, v = oracle.adam(x, m, v, np.array([grads[t]]), lr=0.1, b1=0.9, b2=0.999, eps=1e-8, t=t, clamp=clamp)
            assert abs(x[0] - xw) <= 1e-12 and abs(m[0] - mw) <= 1e-15 and abs(v[0] - vw) <= 1e-15, (x0, t, x, m, v)
    # per-element learning rates (the pose Adam: angles and translations) scale the step only
    x, m, v = oracle.adam(np.array([1.0, 1.0]), np.array([0.1, 0.1]), np.array([3.0 / 999.0] * 2), np.array([1.0, 1.0]),
                          lr=np.array([0.1, 0.01]), t=1)
    assert abs(x[0] - 0.905000000475) <= 1e-12 and abs(x[1] - (1.0 - 0.0094999999525)) <= 1e-12


def test_step_adam_state_recurrence_t2_t3():
    """oracle.step carries the Adam state: from a nonzero state at t = 2 and 3 its p0 / Euler updates are
    oracle.adam (pinned above by the golden steps) applied to its own gradients (pinned by FD, P6), and the
    state it returns is that of oracle.adam."""
    g = grid_of((5, 5, 4), 0.2)
    a = acq_of(200, 0.2, t0=0.5)
    tmpl = gen.linear_array(3, 0.3)
    e_true = np.array([[0.1, -0.2, 0.05, 0.2, 0.1, -3.5]])
    p_true = gen.random_volume(g, 5)
    meas = oracle.forward(g, a, tmpl, gen.poses_from_euler(e_true), p_true)
    rng = np.random.default_rng(3)
    p0 = np.full_like(p_true, 0.4)
    e0 = e_true + 0.01
    nv = p0.size
    st_p = np.concatenate([rng.normal(size=nv) * 1e-3, rng.uniform(1e-7, 2e-6, size=nv)])
    st_q = np.concatenate([rng.normal(size=6) * 1e-2, rng.uniform(1e-5, 1e-4, size=6)])
    for t in (2, 3):
        out = oracle.step(g, a, tmpl, meas, p0, e0, st_p, st_q, lr_p0=1e-2, lr_rot=1e-3, lr_trans=2e-3, t=t)
        xp, mp, vp = oracle.adam(p0.ravel(), st_p[:nv], st_p[nv:], out["grad_p0"], lr=1e-2, t=t, clamp=0.0)
        lr_e = np.array([1e-3] * 3 + [2e-3] * 3)
        xe, me, ve = oracle.adam(e0.ravel(), st_q[:6], st_q[6:], out["grad_euler"].ravel(), lr=lr_e, t=t)
        assert np.allclose(out["p0"].ravel(), xp, rtol=0, atol=1e-15)
        assert np.allclose(out["adam_p0"], np.concatenate([mp, vp]), rtol=0, atol=1e-18)
        assert np.allclose(out["euler_t"].ravel(), xe, rtol=0, atol=1e-15)
        assert np.allclose(out["adam_pose"], np.concatenate([me, ve]), rtol=0, atol=1e-18)
        p0, e0, st_p, st_q = out["p0"], out["euler_t"], out["adam_p0"], out["adam_pose"]
