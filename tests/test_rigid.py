"""Host rigid-body code (Stage 3 analogues) on CPU (-m "not gpu")."""
import math

import numpy as np

from paper_2604_09643_b200 import gen, rigid


def random_R(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def test_kabsch_exact_and_proper():
    """Random rigid transforms recovered to 1e-10; reflected inputs never give det R = -1 (S:665 crit. 4)."""
    rng = np.random.default_rng(0)
    for _ in range(1000):
        A = rng.normal(size=(6, 3))
        R = random_R(rng)
        t = rng.normal(size=3) * 10
        R2, t2 = rigid.kabsch(A, A @ R.T + t)
        assert np.linalg.norm(R2 - R) < 1e-10 and np.linalg.norm(t2 - t) < 1e-10
        Rr, _ = rigid.kabsch(A, (A * np.array([1, 1, -1])) @ R.T)
        assert abs(np.linalg.det(Rr) - 1.0) < 1e-12


def test_ransac_rigid_with_outliers():
    """33-element spherical-cap template (P:180 geometry), 40% grossly wrong sensor estimates:
    pose recovered within 0.1 deg / 0.05 mm and no corrupted index kept as inlier."""
    tmpl = gen.cap_array(33, 30.0, 60.0)
    ok = 0
    for seed in range(40):
        rng = np.random.default_rng(seed)
        R = random_R(rng)
        t = rng.normal(size=3) * 5
        X = tmpl @ R.T + t + rng.normal(scale=0.005, size=tmpl.shape)
        bad = rng.choice(33, 13, replace=False)
        X[bad] += rng.normal(scale=3.0, size=(13, 3))
        R2, t2, inl = rigid.ransac_rigid(X, tmpl, thr=0.05, edge_tol=0.05, iters=300, seed=seed)
        if R2 is None:
            continue
        ang = math.degrees(rigid.rot_angle(R, R2))
        if ang < 0.1 and np.linalg.norm(t2 - t) < 0.05 and not inl[bad].any():
            ok += 1
    assert ok >= 38


def test_euler_roundtrip():
    rng = np.random.default_rng(1)
    for _ in range(200):
        e = rng.uniform([-3, -1.4, -3], [3, 1.4, 3])
        R = rigid.euler_to_R(e)
        assert np.allclose(rigid.euler_to_R(rigid.R_to_euler(R)), R, atol=1e-12)
        assert np.allclose(R, gen.rot_zyx(*e), atol=1e-14)


def test_trajectory_outliers_and_reinit():
    """Freehand sweep (C4 recipe) with 10% glitch frames (5 deg / 3 mm): the consistency
    check finds every glitch and the rigid re-initialisation brings them back within 0.2 mm."""
    w = gen.workload("c4", frames=60)
    rng = np.random.default_rng(3)
    e = w.euler_true.copy()
    e_noisy = e.copy()
    e_noisy[:, :3] += rng.normal(scale=math.radians(0.05), size=(60, 3))
    e_noisy[:, 3:] += rng.normal(scale=0.02, size=(60, 3))
    glitch = rng.choice(np.arange(2, 58), 6, replace=False)
    e_noisy[glitch, :3] += rng.choice([-1, 1], size=(6, 3)) * math.radians(5)
    e_noisy[glitch, 3:] += rng.choice([-1, 1], size=(6, 3)) * 3.0
    bad = rigid.trajectory_outliers(e_noisy, w.tmpl)
    assert set(glitch.tolist()) <= set(np.nonzero(bad)[0].tolist())
    assert bad.sum() <= 8
    e_fix = rigid.reinit_from_neighbours(e_noisy, bad)
    X = rigid.element_positions(e_fix, w.tmpl)
    Xt = rigid.element_positions(e, w.tmpl)
    err = np.linalg.norm(X - Xt, axis=2).mean(1)
    assert err[glitch].max() < 0.2
