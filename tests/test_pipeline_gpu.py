"""The PA-SFM chain Stage 2 -> 3 -> 4 on the GPU (-m gpu; Alg. 1).

A frame of a rigid 2-D array (5 x 5 elements, so the rotation is fully observable; a linear array's roll
is not, R15) over a vascular reference map.  40% of its elements carry corrupted measurements (traces of
the same map seen from displaced positions: Stage 2 localises them confidently but wrongly).  Stage 3's
modified RANSAC must reject them, and Stage 4's inlier-masked NC fine-tuning must bring every element of
the rigid array — the corrupted ones included — back to its true position.  Qualitative thresholds: the
paper prints no localisation accuracy usable as a pin (its numbers need its phantom)."""
import math

import numpy as np
import pytest
import torch

from paper_2604_09643_b200 import gen

pytestmark = pytest.mark.gpu


def grid_array(n, pitch):
    g = (np.arange(n) - (n - 1) / 2) * pitch
    xx, yy = np.meshgrid(g, g, indexing="ij")
    return np.stack([xx.ravel(), yy.ravel(), np.zeros(n * n)], 1)


def test_stage2_3_4_recovers_frame_with_40pct_corrupted_sensors():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    from paper_2604_09643_b200 import Context, rigid
    from paper_2604_09643_b200.pipeline import calibrate_frames, candidate_offsets

    __graft_entry__.build()
    ctx = Context(0)
    grid = gen.make_grid((40, 40, 40), 0.2)
    acq_lo = gen.make_acq(640, 0.2, t0=1.0)
    acq_hi = gen.make_acq(640, 0.4, t0=1.0)
    p_true = gen.vascular_phantom(grid, seed=11)
    T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")  # noqa: E731
    p_ref = T(p_true)  # Stage 1's reference map
    tmpl = grid_array(5, 0.6)
    E = tmpl.shape[0]
    e_true = np.array([[0.10, -0.08, 0.12, 0.3, -0.2, grid["origin"][2] - 3.0]])
    X_true = rigid.element_positions(e_true, tmpl)[0]
    # measured traces: the good elements at their true positions, 40% corrupted (seen from 0.5-0.8 mm away)
    rng = np.random.default_rng(4)
    bad = np.zeros(E, bool)
    bad[rng.choice(E, int(round(0.4 * E)), replace=False)] = True
    X_meas = X_true.copy()
    d = rng.normal(size=(E, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    X_meas[bad] += d[bad] * rng.uniform(0.5, 0.8, size=(bad.sum(), 1))
    P = np.zeros((E, 12))
    P[:, [0, 4, 8]] = 1.0
    P[:, 9:] = X_meas
    S = ctx.forward(grid, acq_lo, T(np.zeros((1, 3))), T(P), p_ref)[:, 0, :]
    meas = S.reshape(1, E, -1).contiguous()
    # initial guess: 1 degree / 0.5 mm off
    e0 = e_true.copy()
    e0[0, :3] += np.radians([1.0, -1.0, 0.7])
    e0[0, 3:] += [0.3, -0.3, 0.25]
    res = calibrate_frames(ctx, grid, [acq_hi, acq_lo], p_ref, meas, tmpl, e0,
                           offsets=candidate_offsets(1.5, 0.3), topk=2, loc_iters=30, loc_lr=0.02,
                           ransac_thr=0.15, edge_tol=0.2, ransac_iters=500, ft_iters=40, ft_lr=3e-3)
    # Stage 2: the good elements are localised, the corrupted ones land where their traces were recorded
    err2 = np.linalg.norm(res.sensors[0] - X_true, axis=1)
    assert np.median(err2[~bad]) < 0.1, err2
    assert np.median(err2[bad]) > 0.4, err2
    # Stage 3: RANSAC rejects the corrupted elements and keeps (nearly) all good ones
    inl = res.inliers[0]
    assert not (inl & bad).any(), (inl, bad)
    assert (inl & ~bad).sum() >= 0.8 * (~bad).sum()
    # a plain Kabsch on all localised elements is pulled away by the corrupted ones
    Rk, tk = rigid.kabsch(tmpl, res.sensors[0])
    err_plain = np.linalg.norm(tmpl @ Rk.T + tk - X_true, axis=1).max()
    err3 = np.linalg.norm(rigid.element_positions(res.euler_ransac, tmpl)[0] - X_true, axis=1).max()
    assert err3 < 0.1 < err_plain, (err3, err_plain)
    # Stage 4: inlier-masked NC fine-tuning; every element of the rigid array (corrupted ones included)
    err4 = np.linalg.norm(rigid.element_positions(res.euler_t, tmpl)[0] - X_true, axis=1)
    assert err4.max() < 0.05, err4
    assert math.degrees(rigid.rot_angle(rigid.euler_to_R(res.euler_t[0, :3]), rigid.euler_to_R(e_true[0, :3]))) < 0.5
    assert set(res.stage_s) == {"stage2", "stage3", "stage4"} and res.stage4_ms_per_iter > 0
