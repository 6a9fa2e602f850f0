"""Edge cases of the deposit-form forward K1d (reading R24) against the fp64 oracle (-m gpu):
near-field elements (the r_lo floor of the fixed-point scale), elements inside the volume, mixed-sign and
tiny/huge amplitudes (the 1/Pmax normalisation), long traces (16-warp CTAs) and traces too long for the
row accumulators (fallback to the direct kernel K1), and the exact power-of-two scale invariance of the
fixed-point deposits."""
import numpy as np
import pytest
import torch

import oracle
from paper_2604_09643_b200 import gen, plan_info

from test_gpu_parity import TOL_FA, T, acq32, ctx, f64, grid32, random_scene, rel  # noqa: F401

pytestmark = pytest.mark.gpu


def fwd_pair(ctx, grid, acq, tmpl, poses, p0):
    g, a = grid32(grid), acq32(acq)
    y = ctx.forward(g, a, T(tmpl), T(poses), T(p0)).cpu().numpy()
    yo = oracle.forward(g, a, f64(tmpl), f64(poses), f64(p0))
    return y, yo


def test_near_field_and_inside_elements(ctx, record_parity):
    grid = gen.make_grid((20, 18, 12), 0.2)
    acq = gen.make_acq(320, 0.2, t0=0.0)
    p0 = gen.random_volume(grid, 3)
    o = np.asarray(grid["origin"])
    # element 1: 0.05 mm below the first voxel layer; element 2: between voxel centres inside the volume
    tmpl = np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 0.0]])
    e = np.zeros((2, 6))
    e[0, 3:] = o + np.array([1.0 * 0.2 + 0.03, 2.0 * 0.2 + 0.07, -0.05])
    e[1, 3:] = o + np.array([7.5 * 0.2, 9.5 * 0.2, 5.5 * 0.2])
    poses = gen.poses_from_euler(e)
    assert plan_info(grid32(grid), acq32(acq), 2)["fwd_deposit"] == 1
    y, yo = fwd_pair(ctx, grid, acq, tmpl, poses, p0)
    r = rel(y, yo)
    record_parity("near_inside_forward", r, TOL_FA)
    assert r <= TOL_FA, r


@pytest.mark.parametrize("kind", ["mixed_sign", "tiny", "huge", "range1e3"])
def test_amplitude_scales(ctx, kind, record_parity):
    grid = gen.make_grid((17, 15, 11), 0.2)
    acq = gen.make_acq(300, 0.2, t0=1.0)
    tmpl, poses = random_scene(11, grid, E=4, F=2)
    p0 = gen.random_volume(grid, 5)
    if kind == "mixed_sign":
        p0 = p0 - 0.5
    elif kind == "tiny":
        p0 = p0 * 1e-30
    elif kind == "huge":
        p0 = p0 * 1e30
    else:  # a few bright voxels 1e3 above a dim background
        rng = np.random.default_rng(7)
        p0 = p0 * 1e-3
        p0.reshape(-1)[rng.choice(p0.size, 20, replace=False)] = 1.0
    y, yo = fwd_pair(ctx, grid, acq, tmpl, poses, p0)
    r = rel(y, yo)
    record_parity(f"amplitude_{kind}", r, TOL_FA)
    assert r <= TOL_FA, r


def test_power_of_two_scale_is_exact(ctx):
    grid = gen.make_grid((16, 16, 8), 0.2)
    acq = gen.make_acq(256, 0.2, t0=1.0)
    tmpl, poses = random_scene(12, grid, E=3, F=2)
    p = T(gen.random_volume(grid, 6))
    y1 = ctx.forward(grid32(grid), acq32(acq), T(tmpl), T(poses), p)
    y4 = ctx.forward(grid32(grid), acq32(acq), T(tmpl), T(poses), 4.0 * p)
    # 1/Pmax normalisation: the integer deposits are identical, only the decode scale changes
    assert torch.equal(4.0 * y1, y4)


# the fp32 row accumulators (NJ x (R + 1) floats) bound the deposit form: at rank 4, 4096 samples fit two 8-warp
# CTAs per SM, 6000 one 16-warp CTA next to the round-accumulator ring, 10000 do not (direct K1)
@pytest.mark.parametrize("nt,want_dep,want_warps", [(4096, 1, 8), (6000, 1, 16), (10000, 0, 0)])
def test_long_traces(ctx, nt, want_dep, want_warps, record_parity):
    grid = gen.make_grid((12, 10, 8), 0.2)
    acq = gen.make_acq(nt, 0.2, t0=0.0)
    tmpl, poses = random_scene(13, grid, E=3, F=2)
    # push the elements out so that the windows land late in the long trace
    poses[:, 11] -= 0.0375 * (nt - 400)
    info = plan_info(grid32(grid), acq32(acq), 3)
    assert info["fwd_deposit"] == want_dep and (want_warps == 0 or info["dep_warps"] == want_warps), info
    p0 = gen.random_volume(grid, 7)
    y, yo = fwd_pair(ctx, grid, acq, tmpl, poses, p0)
    assert np.abs(yo).max() > 0  # the windows are inside the trace
    r = rel(y, yo)
    record_parity(f"long_trace_{nt}", r, TOL_FA)
    assert r <= TOL_FA, r


@pytest.mark.parametrize("variant", ["adj_svd", "fwd_direct", "adj_direct", "adj_taylor"])
def test_alternative_kernels_parity(ctx, variant, record_parity):
    """The alternative kernels a context's policy selects (pa_set_policy: K2s, direct K1, direct K2, K2c) keep
    parity with the oracle on a ragged multi-tile case."""
    ctx.set_policy(variant)
    try:
        _alternative(ctx, variant, record_parity)
    finally:
        ctx.set_policy("default")


def _alternative(ctx, variant, record_parity):
    grid = gen.make_grid((21, 19, 13), 0.2)
    acq = gen.make_acq(301, 0.2, t0=1.3)
    tmpl, poses = random_scene(14, grid, E=5, F=3)
    p0 = gen.random_volume(grid, 8)
    cot = gen.random_cotangent((3, 5, 301), 9)
    g, a = grid32(grid), acq32(acq)
    info = ctx.plan_info(g, a, 5)
    want = {"adj_svd": ("adj_kernel", 2), "fwd_direct": ("fwd_deposit", 0), "adj_direct": ("adj_kernel", 0),
            "adj_taylor": ("adj_kernel", 1)}[variant]
    assert info[want[0]] == want[1], info
    y = ctx.forward(g, a, T(tmpl), T(poses), T(p0)).cpu().numpy()
    gz, gp, _ = ctx.adjoint_pose(g, a, T(tmpl), T(poses), T(p0), T(cot))
    yo = oracle.forward(g, a, f64(tmpl), f64(poses), f64(p0))
    zo = oracle.adjoint(g, a, f64(tmpl), f64(poses), f64(cot))
    po, _ = oracle.pose_grad(g, a, f64(tmpl), f64(poses), f64(p0), f64(cot))
    ef, ez, ep = rel(y, yo), rel(gz.cpu().numpy(), zo), rel(gp.cpu().numpy(), po)
    record_parity(f"{variant}:forward", ef, TOL_FA)
    record_parity(f"{variant}:adjoint", ez, TOL_FA)
    record_parity(f"{variant}:pose", ep, 1e-3)
    assert ef <= TOL_FA and ez <= TOL_FA and ep <= 1e-3, (ef, ez, ep)
