"""Seeded synthetic-input generators (shared by tests, bench and smoke).

This module holds NONE of the operator's arithmetic: it only builds inputs —
voxel grids, phantoms, array templates, freehand trajectories and cotangents —
whose shapes and statistics follow the paper's workloads (SURVEY.md §8 d).
Both the CUDA path and the fp64 oracle consume the arrays it returns.

Units: mm, µs, mm/µs.  Grids are [nz][ny][nx] (x fastest), poses are [F][12] =
R (row-major 3x3) then t; euler_t is [F][6] = ZYX Euler angles (a, b, c) then t.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

C_SOUND = 1.5          # mm/µs (1500 m/s, BASELINE configs)
FS_MHZ = 40.0          # sampling rate (BASELINE configs)
DT = 1.0 / FS_MHZ      # µs
KAPPA = 5.0            # window half-width in sigma (R4)


# ----------------------------------------------------------------------------------- geometry
def rot_zyx(a: float, b: float, c: float) -> np.ndarray:
    """Rz(a) @ Ry(b) @ Rx(c) — used only to *build* synthetic poses."""
    ca, sa, cb, sb, cc, sc = math.cos(a), math.sin(a), math.cos(b), math.sin(b), math.cos(c), math.sin(c)
    Rz = np.array([[ca, -sa, 0], [sa, ca, 0], [0, 0, 1.0]])
    Ry = np.array([[cb, 0, sb], [0, 1.0, 0], [-sb, 0, cb]])
    Rx = np.array([[1.0, 0, 0], [0, cc, -sc], [0, sc, cc]])
    return Rz @ Ry @ Rx


def poses_from_euler(euler_t: np.ndarray) -> np.ndarray:
    F = euler_t.shape[0]
    out = np.zeros((F, 12))
    for f in range(F):
        out[f, :9] = rot_zyx(*euler_t[f, :3]).reshape(-1)
        out[f, 9:] = euler_t[f, 3:]
    return out


def linear_array(E: int, pitch: float) -> np.ndarray:
    """Linear array of point elements along the template x axis, centred at 0."""
    x = (np.arange(E) - (E - 1) / 2.0) * pitch
    return np.stack([x, np.zeros(E), np.zeros(E)], axis=1)


def cap_array(n_total: int, radius: float, cap_deg: float, subset: int = 0, n_subsets: int = 1) -> np.ndarray:
    """Fibonacci lattice on a spherical cap (bowl opening toward +z, centre at the origin,
    elements at z <= 0), then an interleaved subset."""
    i = np.arange(n_total) + 0.5
    cos_max = math.cos(math.radians(cap_deg))
    z = 1.0 - (1.0 - cos_max) * i / n_total           # cos(polar) in [cos_max, 1]
    phi = i * math.pi * (3.0 - math.sqrt(5.0))
    s = np.sqrt(1.0 - z * z)
    pts = np.stack([s * np.cos(phi), s * np.sin(phi), -z], axis=1) * radius
    return pts[subset::n_subsets].copy()


# ----------------------------------------------------------------------------------- configs
@dataclass
class Workload:
    name: str
    grid: dict
    acq: dict
    tmpl: np.ndarray
    euler_true: np.ndarray            # [F][6]
    phantom: str = "vascular"
    seed: int = 42
    extra: dict = field(default_factory=dict)

    @property
    def F(self) -> int:
        return self.euler_true.shape[0]

    @property
    def E(self) -> int:
        return self.tmpl.shape[0]

    @property
    def nvox(self) -> int:
        g = self.grid
        return g["nx"] * g["ny"] * g["nz"]

    def poses_true(self) -> np.ndarray:
        return poses_from_euler(self.euler_true)


def make_grid(n, pitch):
    nx, ny, nz = n
    origin = [-(nx - 1) / 2.0 * pitch, -(ny - 1) / 2.0 * pitch, -(nz - 1) / 2.0 * pitch]
    return dict(nx=nx, ny=ny, nz=nz, origin=origin, pitch=pitch)


def make_acq(nt, sigma, t0=0.0, kappa=KAPPA, kernel="gauss", nu=0.0):
    """kernel: family of the designated kernel K (R23) — "gauss" | "exp" | "pow"."""
    return dict(c=C_SOUND, t0=t0, dt=DT, nt=nt, sigma=sigma, kappa=kappa, kernel=kernel, nu=nu)


def family_acq(acq: dict, kernel: str, nu: float = 1.5) -> dict:
    """The same acquisition with another kernel family (f3, R23), keeping the window kappa s at
    the Gaussian's 5 sigma: exponential s = sigma/2, kappa = 10 (tail e^-10); power law
    s = sigma/4, kappa = 20 (tail 20^-2nu)."""
    if kernel == "gauss":
        return dict(acq)
    if kernel == "exp":
        return dict(acq, kernel="exp", nu=0.0, sigma=acq["sigma"] / 2.0, kappa=10.0)
    if kernel == "pow":
        return dict(acq, kernel="pow", nu=float(nu), sigma=acq["sigma"] / 4.0, kappa=20.0)
    raise ValueError(f"unknown kernel family {kernel}")


def _smooth_angles(F, rng, amp_rad, n_terms=3):
    t = np.arange(F) / max(F - 1, 1)
    out = np.zeros(F)
    for _ in range(n_terms):
        freq = rng.uniform(0.3, 2.0)
        out += amp_rad / n_terms * np.sin(2 * math.pi * freq * t + rng.uniform(0, 2 * math.pi))
    return out


def sweep_trajectory(F, grid, standoff, step, jitter_mm, jitter_deg, seed):
    """Freehand linear sweep below the volume along y (elevation), array facing +z,
    with smooth low-frequency angle / translation jitter."""
    rng = np.random.default_rng(seed)
    zmin = grid["origin"][2]
    y0 = -(F - 1) / 2.0 * step
    e = np.zeros((F, 6))
    for q in range(3):
        e[:, q] = _smooth_angles(F, rng, math.radians(jitter_deg))
    e[:, 3] = _smooth_angles(F, rng, jitter_mm)
    e[:, 4] = y0 + step * np.arange(F) + _smooth_angles(F, rng, jitter_mm)
    e[:, 5] = zmin - standoff + _smooth_angles(F, rng, jitter_mm)
    return e


def azimuth_trajectory(F, seed, jitter_mm=0.5, jitter_deg=1.0):
    """C5: bowl array rotated about the vertical axis through 90 degrees + perturbation."""
    rng = np.random.default_rng(seed)
    e = np.zeros((F, 6))
    e[:, 0] = np.linspace(0.0, math.pi / 2, F) + _smooth_angles(F, rng, math.radians(jitter_deg))
    e[:, 1] = _smooth_angles(F, rng, math.radians(jitter_deg))
    e[:, 2] = _smooth_angles(F, rng, math.radians(jitter_deg))
    for q in range(3):
        e[:, 3 + q] = _smooth_angles(F, rng, jitter_mm)
    return e


def workload(name: str, frames: int | None = None) -> Workload:
    """Named BASELINE.json configs (c1..c5).  `frames` overrides the frame count (subsets)."""
    name = name.lower()
    if name == "c1":
        grid = make_grid((32, 32, 32), 0.2)
        acq = make_acq(512, 0.2, t0=0.0)
        tmpl = linear_array(64, 0.1)
        e = np.zeros((1, 6))
        e[0, 5] = grid["origin"][2] - 3.0
        return Workload("c1", grid, acq, tmpl, e, phantom="sphere", seed=42)
    if name == "c2":
        grid = make_grid((128, 128, 128), 0.2)
        acq = make_acq(1024, 0.2, t0=0.0)
        tmpl = linear_array(128, 0.2)
        F = frames or 100
        e = sweep_trajectory(F, grid, 3.0, 0.256 * 100 / F, 0.5, 2.0, seed=42 + 2)
        return Workload("c2", grid, acq, tmpl, e, seed=42 + 2)
    if name in ("c3", "c3_coarse"):
        grid = make_grid((128, 128, 128), 0.4)
        acq = make_acq(2048, 0.4, t0=2.0)
        tmpl = linear_array(128, 0.4)
        F = frames or 200
        e = sweep_trajectory(F, grid, 3.0, 0.256 * 200 / F, 0.5, 2.0, seed=42 + 3)
        return Workload("c3_coarse", grid, acq, tmpl, e, seed=42 + 3)
    if name == "c3_fine":
        grid = make_grid((256, 256, 256), 0.2)
        acq = make_acq(2048, 0.2, t0=2.0)
        tmpl = linear_array(128, 0.4)
        F = frames or 200
        e = sweep_trajectory(F, grid, 3.0, 0.256 * 200 / F, 0.5, 2.0, seed=42 + 3)
        return Workload("c3_fine", grid, acq, tmpl, e, seed=42 + 3)
    if name == "c4":
        grid = make_grid((256, 256, 256), 0.2)
        acq = make_acq(2048, 0.2, t0=2.0)
        tmpl = linear_array(128, 0.4)
        F = frames or 400
        e = sweep_trajectory(F, grid, 3.0, 0.128 * 400 / F, 0.5, 2.0, seed=42 + 4)
        return Workload("c4", grid, acq, tmpl, e, seed=42 + 4)
    if name == "c5":
        grid = make_grid((512, 512, 256), 0.1)
        acq = make_acq(2048, 0.1, t0=14.0)
        tmpl = cap_array(1024, 60.0, 60.0, subset=0, n_subsets=4)
        F = frames or 800
        e = azimuth_trajectory(F, seed=42 + 5)
        return Workload("c5", grid, acq, tmpl, e, seed=42 + 5)
    raise ValueError(f"unknown workload {name}")


def perturb_euler(euler: np.ndarray, deg: float, mm: float, seed: int) -> np.ndarray:
    """Initial pose guess: truth + N(0, deg) rotation / N(0, mm) translation."""
    rng = np.random.default_rng(seed)
    out = euler.copy()
    out[:, :3] += rng.normal(0.0, math.radians(deg), size=(euler.shape[0], 3))
    out[:, 3:] += rng.normal(0.0, mm, size=(euler.shape[0], 3))
    return out


# ----------------------------------------------------------------------------------- phantoms
def _centres(grid):
    g = grid
    xs = g["origin"][0] + g["pitch"] * np.arange(g["nx"])
    ys = g["origin"][1] + g["pitch"] * np.arange(g["ny"])
    zs = g["origin"][2] + g["pitch"] * np.arange(g["nz"])
    return xs, ys, zs


def sphere_fraction(grid, centre, radius, ss=4) -> np.ndarray:
    """Partial-volume fraction of a ball per voxel, ss^3 supersampling. [nz][ny][nx] float64."""
    xs, ys, zs = _centres(grid)
    h = grid["pitch"]
    off = (np.arange(ss) + 0.5) / ss - 0.5
    frac = np.zeros((grid["nz"], grid["ny"], grid["nx"]))
    for oz in off:
        dz2 = (zs[:, None, None] + oz * h - centre[2]) ** 2
        for oy in off:
            dy2 = (ys[None, :, None] + oy * h - centre[1]) ** 2
            for ox in off:
                dx2 = (xs[None, None, :] + ox * h - centre[0]) ** 2
                frac += (dx2 + dy2 + dz2 <= radius * radius)
    return frac / ss ** 3


def _capsule_raster(vol, grid, p, q, rad, amp, ss):
    """max-union of a capsule (segment p->q, radius rad) with partial volume."""
    h = grid["pitch"]
    o = np.asarray(grid["origin"])
    lo = np.floor((np.minimum(p, q) - rad - o) / h).astype(int) - 1
    hi = np.ceil((np.maximum(p, q) + rad - o) / h).astype(int) + 1
    n = np.array([grid["nx"], grid["ny"], grid["nz"]])
    lo = np.clip(lo, 0, n - 1)
    hi = np.clip(hi, 0, n - 1)
    if np.any(hi < lo):
        return
    ix = np.arange(lo[0], hi[0] + 1)
    iy = np.arange(lo[1], hi[1] + 1)
    iz = np.arange(lo[2], hi[2] + 1)
    off = (np.arange(ss) + 0.5) / ss - 0.5
    d = q - p
    L2 = max(float(d @ d), 1e-12)
    acc = np.zeros((iz.size, iy.size, ix.size))
    for oz in off:
        Z = o[2] + h * (iz[:, None, None] + oz)
        for oy in off:
            Y = o[1] + h * (iy[None, :, None] + oy)
            for ox in off:
                X = o[0] + h * (ix[None, None, :] + ox)
                u = np.clip(((X - p[0]) * d[0] + (Y - p[1]) * d[1] + (Z - p[2]) * d[2]) / L2, 0.0, 1.0)
                dist2 = (X - p[0] - u * d[0]) ** 2 + (Y - p[1] - u * d[1]) ** 2 + (Z - p[2] - u * d[2]) ** 2
                acc += dist2 <= rad * rad
    acc *= amp / ss ** 3
    sub = vol[iz[0]:iz[-1] + 1, iy[0]:iy[-1] + 1, ix[0]:ix[-1] + 1]
    np.maximum(sub, acc, out=sub)


def vascular_phantom(grid, seed=42, background=0.02) -> np.ndarray:
    """Seeded branching vessel tree (Murray's law radii, capsules with partial volume) plus a
    smooth positive background so that no voxel is zero; values in [0, 1]."""
    from scipy.ndimage import gaussian_filter, zoom

    rng = np.random.default_rng(seed)
    h = grid["pitch"]
    n = np.array([grid["nx"], grid["ny"], grid["nz"]])
    o = np.asarray(grid["origin"], dtype=np.float64)
    ext = (n - 1) * h
    vol = np.zeros((grid["nz"], grid["ny"], grid["nx"]))
    ss = 4 if grid["nx"] * grid["ny"] * grid["nz"] <= 128 ** 3 else 2
    scale = float(ext.max()) / 51.2
    segs = []

    def grow(p, direction, rad, depth, amp):
        if depth == 0 or rad < 0.05:
            return
        length = rng.uniform(8.0, 12.0) * max(rad, 0.08) * max(scale, 0.25) * 2.0
        q = p + direction * length
        segs.append((p, q, rad, amp))
        ratio = rng.uniform(0.6, 1.0)
        r1 = rad / (1.0 + ratio ** 3) ** (1.0 / 3.0)
        r2 = r1 * ratio
        for rc, sign in ((r1, 1.0), (r2, -1.0)):
            ang = math.radians(rng.uniform(20.0, 60.0)) * sign
            perp = np.cross(direction, rng.normal(size=3))
            perp /= np.linalg.norm(perp) + 1e-12
            nd = math.cos(ang) * direction + math.sin(ang) * perp
            nd /= np.linalg.norm(nd)
            grow(q, nd, max(min(rc, 0.5), 0.05), depth - 1, amp * rng.uniform(0.85, 1.0))

    n_roots = int(rng.integers(3, 7))
    for _ in range(n_roots):
        axis = int(rng.integers(0, 3))
        side = int(rng.integers(0, 2))
        p = o + rng.uniform(0.2, 0.8, size=3) * ext
        p[axis] = o[axis] + (ext[axis] if side else 0.0)
        d = np.zeros(3)
        d[axis] = -1.0 if side else 1.0
        d += rng.normal(scale=0.3, size=3)
        d /= np.linalg.norm(d)
        grow(p, d, rng.uniform(0.3, 0.5), int(rng.integers(6, 9)), rng.uniform(0.5, 1.0))
    for p, q, rad, amp in segs:
        _capsule_raster(vol, grid, p, q, rad, amp, ss)
    # smooth background: low-resolution noise, Gaussian filtered (2 mm), upsampled, normalised
    f = 8
    small = rng.random((max(grid["nz"] // f, 2), max(grid["ny"] // f, 2), max(grid["nx"] // f, 2)))
    small = gaussian_filter(small, sigma=2.0 / (h * f), mode="reflect")
    bg = zoom(small, (grid["nz"] / small.shape[0], grid["ny"] / small.shape[1], grid["nx"] / small.shape[2]), order=1)
    bg = bg[: grid["nz"], : grid["ny"], : grid["nx"]]
    bg = (bg - bg.min()) / max(bg.max() - bg.min(), 1e-12)
    vol = np.maximum(vol, background * (0.5 + 0.5 * bg))
    return np.clip(vol, 0.0, 1.0)


def phantom(w: Workload) -> np.ndarray:
    if w.phantom == "sphere":
        # single uniform sphere R = 2 mm, partial volume, centred (C1)
        return sphere_fraction(w.grid, (0.0, 0.0, 0.0), 2.0, ss=4)
    return vascular_phantom(w.grid, seed=w.seed)


def random_cotangent(shape, seed) -> np.ndarray:
    return np.random.default_rng(seed).normal(size=shape)


def random_volume(grid, seed) -> np.ndarray:
    return np.random.default_rng(seed).random((grid["nz"], grid["ny"], grid["nx"]))
