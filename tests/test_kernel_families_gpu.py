"""GPU vs oracle parity for the kernel families (f3: exponential and power-law K, P:313-323,
P:345; reading R23) — through the C ABI, -m gpu.

Same bars as the Gaussian path: forward / adjoint <= 1e-4 relative L2, pose and
element gradients <= 1e-3.  Every compiled window class is exercised (the class depends only
on the window length 2 kappa s / (c dt) and the pitch, not on the family).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2604_09643_b200 import gen
from paper_2604_09643_b200._pa import PAError, PA_EINVAL

from test_gpu_parity import T, f64, rel, grid32, acq32, run_all, random_scene, TOL_FA, TOL_POSE

pytestmark = pytest.mark.gpu

# (kernel, nu, s, kappa) with kappa s = 1.0 mm: the L_min = 53 class at c dt = 0.0375 mm
FAMS53 = [("exp", 0.0, 0.1, 10.0), ("pow", 1.5, 0.05, 20.0), ("pow", 0.8, 0.1, 10.0), ("pow", 3.0, 0.2, 5.0)]


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_09643_b200 import Context
    import __graft_entry__

    __graft_entry__.build()
    return Context(0)


def check(record_parity, tag, res):
    (y, yo), (z, zo), (gp, po), (ge, geo) = res
    out = {}
    for m, a, b, t in (("forward", y, yo, TOL_FA), ("adjoint", z, zo, TOL_FA), ("pose", gp, po, TOL_POSE),
                       ("elem", ge, geo, TOL_POSE)):
        record_parity(f"{tag}:{m}", rel(a, b), t)
        out[m] = rel(a, b)
        assert np.all(np.isfinite(a)), m
    assert out["forward"] <= TOL_FA and out["adjoint"] <= TOL_FA, out
    assert out["pose"] <= TOL_POSE and out["elem"] <= TOL_POSE, out


@pytest.mark.parametrize("kernel,nu,s,kappa", FAMS53)
def test_c1_geometry_families(ctx, record_parity, kernel, nu, s, kappa):
    """C1 geometry (32^3 @ 0.2 mm sphere, 64-element linear array, 512 samples), tilted pose."""
    w = gen.workload("c1")
    acq = dict(w.acq, sigma=s, kappa=kappa, kernel=kernel, nu=nu)
    p0 = gen.phantom(w)
    e = w.euler_true.copy()
    e[0, :3] = [0.3, -0.2, 0.15]
    poses = gen.poses_from_euler(e)
    cot = gen.random_cotangent((1, 64, 512), seed=7)
    check(record_parity, f"c1-{kernel}{nu}", run_all(ctx, w.grid, acq, w.tmpl, poses, p0, cot))


@pytest.mark.parametrize("kernel,nu,s,kappa", FAMS53[:2])
@pytest.mark.parametrize("shape", [(21, 19, 13), (1, 1, 1), (33, 9, 5)])
def test_ragged_multi_tile_families(ctx, record_parity, kernel, nu, s, kappa, shape):
    grid = gen.make_grid(shape, 0.2)
    acq = gen.make_acq(301, s, t0=1.3, kappa=kappa, kernel=kernel, nu=nu)
    tmpl, poses = random_scene(3, grid, E=5, F=3)
    p0 = gen.random_volume(grid, 4)
    cot = gen.random_cotangent((3, 5, 301), seed=5)
    check(record_parity, f"ragged-{kernel}", run_all(ctx, grid, acq, tmpl, poses, p0, cot))


@pytest.mark.parametrize("kernel,nu", [("exp", 0.0), ("pow", 1.5)])
@pytest.mark.parametrize("pitch,ks", [(0.1, 0.5), (0.4, 2.0)])
def test_other_window_classes_families(ctx, record_parity, kernel, nu, pitch, ks):
    """L_min = 26 (pitch 0.1, kappa s = 0.5 mm) and L_min = 106 (pitch 0.4, kappa s = 2 mm)."""
    kappa = 10.0 if kernel == "exp" else 20.0
    grid = gen.make_grid((24, 20, 16), pitch)
    acq = gen.make_acq(700, ks / kappa, t0=0.4, kappa=kappa, kernel=kernel, nu=nu)
    tmpl, poses = random_scene(11, grid, E=6, F=2, standoff=2.0)
    p0 = gen.random_volume(grid, 12)
    cot = gen.random_cotangent((2, 6, 700), seed=13)
    check(record_parity, f"class-{kernel}-{pitch}", run_all(ctx, grid, acq, tmpl, poses, p0, cot))


@pytest.mark.parametrize("kernel,nu,s,kappa", FAMS53[:2])
def test_c2_geometry_element_subset_families(ctx, record_parity, kernel, nu, s, kappa):
    """C2 geometry at full size (128^3 vascular phantom, 1024 samples, frame 0): the GPU runs
    all 128 elements; the oracle checks 6 of them (forward rows; adjoint and pose with the
    cotangent nonzero on those rows only, so both sides see the same operator)."""
    w = gen.workload("c2", frames=1)
    acq = acq32(dict(w.acq, sigma=s, kappa=kappa, kernel=kernel, nu=nu))
    grid = grid32(w.grid)
    p0 = gen.phantom(w)
    poses = w.poses_true()
    sub = np.array([0, 17, 50, 64, 101, 127])
    cot = np.zeros((1, w.E, acq["nt"]))
    cot[:, sub] = gen.random_cotangent((1, len(sub), acq["nt"]), seed=3)
    y = ctx.forward(grid, acq, T(w.tmpl), T(poses), T(p0)).cpu().numpy()
    z = ctx.adjoint(grid, acq, T(w.tmpl), T(poses), T(cot)).cpu().numpy()
    gp, ge = ctx.pose_grad(grid, acq, T(w.tmpl), T(poses), T(p0), T(cot))
    ts = f64(w.tmpl)[sub]
    yo = oracle.forward(grid, acq, ts, f64(poses), f64(p0))
    zo = oracle.adjoint(grid, acq, ts, f64(poses), f64(cot[:, sub]))
    _, geo = oracle.pose_grad(grid, acq, ts, f64(poses), f64(p0), f64(cot[:, sub]))
    r = {"forward": rel(y[:, sub], yo), "adjoint": rel(z, zo), "elem": rel(ge.cpu().numpy()[:, sub], geo)}
    for m, t in (("forward", TOL_FA), ("adjoint", TOL_FA), ("elem", TOL_POSE)):
        record_parity(f"c2sub-{kernel}:{m}", r[m], t)
    assert r["forward"] <= TOL_FA and r["adjoint"] <= TOL_FA and r["elem"] <= TOL_POSE, r


@pytest.mark.parametrize("kernel,nu,s,kappa", FAMS53[:2])
def test_family_step_parity(ctx, record_parity, kernel, nu, s, kappa):
    """pa_step vs oracle_step (MSE) with a non-Gaussian kernel: loss, dL/dp0 (1e-4), dL/dEuler (1e-3)."""
    grid = gen.make_grid((16, 14, 12), 0.2)
    acq = gen.make_acq(320, s, t0=1.0, kappa=kappa, kernel=kernel, nu=nu)
    tmpl = gen.linear_array(8, 0.3)
    e_true = np.array([[0.05, -0.1, 0.02, 0.1, 0.2, -4.5], [-0.05, 0.08, 0.0, -0.3, 0.1, -4.8]])
    p_true = gen.random_volume(grid, 3)
    meas = oracle.forward(grid32(grid), acq32(acq), f64(tmpl), f64(gen.poses_from_euler(e_true)), f64(p_true))
    e0 = e_true + np.array([0.01, -0.01, 0.005, 0.05, -0.05, 0.02])
    p0 = np.full(p_true.shape, 0.4)
    nv = p0.size
    cfg = dict(lr_p0=1e-2, lr_rot=1e-3, lr_trans=1e-2, beta1=0.9, beta2=0.999, eps=1e-8, step=1, loss_kind=0)
    out = oracle.step(grid32(grid), acq32(acq), f64(tmpl), f64(meas), f64(p0), f64(e0), np.zeros(2 * nv),
                      np.zeros(24), lr_p0=cfg["lr_p0"], lr_rot=cfg["lr_rot"], lr_trans=cfg["lr_trans"], loss_kind=0)
    p_d, e_d = T(p0), T(e0)
    am, ap = torch.zeros(2 * nv, device="cuda"), torch.zeros(24, device="cuda")
    gbuf, loss, geul = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda"), torch.empty((2, 6), device="cuda")
    ctx.step(grid32(grid), acq32(acq), T(tmpl), T(meas), p_d, e_d, am, ap, gbuf, loss, cfg, grad_euler=geul)
    torch.cuda.synchronize()
    assert abs(float(loss[0]) - out["loss"]) <= 1e-4 * abs(out["loss"])
    rg, re = rel(gbuf.cpu().numpy().ravel(), out["grad_p0"]), rel(geul.cpu().numpy(), out["grad_euler"])
    record_parity(f"step-{kernel}:grad_p0", rg, TOL_FA)
    record_parity(f"step-{kernel}:grad_euler", re, TOL_POSE)
    assert rg <= TOL_FA and re <= TOL_POSE, (rg, re)


def test_family_argument_errors(ctx):
    grid = gen.make_grid((8, 8, 4), 0.2)
    tmpl, poses = random_scene(1, grid, E=2, F=1)
    p0 = T(gen.random_volume(grid, 1))
    for bad in (dict(kernel=3), dict(kernel="pow", nu=0.5), dict(kernel="pow", nu=17.0),
                dict(kernel="exp", kappa=31.0, sigma=0.03)):
        acq = dict(gen.make_acq(128, 0.2), **bad)
        with pytest.raises(PAError) as ei:
            ctx.forward(grid, acq, T(tmpl), T(poses), p0)
        assert ei.value.status == PA_EINVAL, bad


# runtime classes of the direct kernels (r2, R26): window lengths outside {26, 53, 106}, and the Gaussian
# forced onto the direct kernels at a general acquisition
RT_CASES = [("exp", 0.0, 0.075, 10.0, 0.2, 40), ("pow", 1.5, 0.0375, 20.0, 0.2, 40), ("exp", 0.0, 0.125, 10.0, 0.2, 66),
            ("pow", 0.8, 0.15, 10.0, 0.2, 80), ("exp", 0.0, 0.07, 10.0, 0.1, 37), ("gauss", 0.0, 0.25, 5.0, 0.2, 66),
            ("gauss", 0.0, 0.061, 5.0, 0.1, 16), ("gauss", 0.0, 0.05, 5.0, 0.2, 13)]


@pytest.mark.parametrize("kernel,nu,s,kappa,pitch,lmin", RT_CASES)
def test_runtime_direct_classes(ctx, record_parity, kernel, nu, s, kappa, pitch, lmin):
    """Ragged multi-tile grid, several frames, windows clipped at both ends, on a runtime class of K1/K2."""
    from paper_2604_09643_b200 import plan_info

    grid = gen.make_grid((21, 17, 13), pitch)
    acq = dict(gen.make_acq(700, 0.2, t0=1.0), sigma=s, kappa=kappa, kernel=kernel, nu=nu)
    tmpl, poses = random_scene(41, grid, E=4, F=2, standoff=2.0)
    p0 = gen.random_volume(grid, 42)
    cot = gen.random_cotangent((2, 4, 700), seed=43)
    if kernel == "gauss":
        ctx.set_policy(["fwd_direct", "adj_direct"])
    try:
        info = ctx.plan_info(grid32(grid), acq32(acq), 4)
        assert info["lmin"] == lmin and info["direct_class"] < 0 and info["fwd_deposit"] == 0 and info["adj_kernel"] == 0, info
        check(record_parity, f"rt-{kernel}{nu}-L{lmin}", run_all(ctx, grid, acq, tmpl, poses, p0, cot))
    finally:
        ctx.set_policy("default")
