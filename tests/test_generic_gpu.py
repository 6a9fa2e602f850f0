"""The generic kernels K1g / K2g / K3g on the GPU (-m gpu): windows no other kernel holds — exponential and
power-law windows longer than the direct kernels' register windows, a Gaussian window beyond the fast path's
PA_LMAX, a Gaussian window shorter than its cluster spread — run through the same C ABI and match the fp64
oracle (Eq. gpu_forward_model P:341-345 with the family kernels of R23; tolerances of DESIGN.md §5)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2604_09643_b200 import gen, plan_info

from test_gpu_parity import TOL_FA, TOL_POSE, T, acq32, ctx, f64, grid32, random_scene, rel, run_all  # noqa: F401

pytestmark = pytest.mark.gpu

CASES = {
    # name: (pitch, sigma (scale s), kappa, family, nu, expected L_min)
    "exp_kappa30": (0.2, 0.3, 30.0, "exp", 0.0, 480),
    "pow1.5_kappa10": (0.2, 0.5, 10.0, "pow", 1.5, 266),
    "pow0.8_kappa20": (0.2, 0.2, 20.0, "pow", 0.8, 213),
    "gauss_sigma2.0": (0.2, 2.0, 5.0, "gauss", 0.0, 533),
    "gauss_sigma0.02": (0.2, 0.02, 5.0, "gauss", 0.0, 5),
}


def case(name, nt=1400):
    pitch, s, kappa, kern, nu, lmin = CASES[name]
    grid = grid32(gen.make_grid((11, 9, 7), pitch))
    acq = acq32(gen.make_acq(nt, s, t0=0.5, kappa=kappa, kernel=kern, nu=nu))
    return grid, acq, lmin


@pytest.mark.parametrize("name", sorted(CASES))
def test_generic_parity(ctx, name, record_parity):
    grid, acq, lmin = case(name)
    info = plan_info(grid, acq, 3)
    assert info["lmin"] == lmin and info["generic"] == 1, info
    tmpl, poses = random_scene(41, grid, E=3, F=2, standoff=1.5)
    p0 = gen.random_volume(grid, 42)
    cot = gen.random_cotangent((2, 3, acq["nt"]), seed=43)
    (y, yo), (z, zo), (gp, po), (ge, geo) = run_all(ctx, grid, acq, tmpl, poses, p0, cot)
    assert np.abs(yo).max() > 0 and np.abs(zo).max() > 0
    errs = dict(forward=rel(y, yo), adjoint=rel(z, zo), pose=rel(gp, po), elem=rel(ge, geo))
    tol = dict(forward=TOL_FA, adjoint=TOL_FA, pose=TOL_POSE, elem=TOL_POSE)
    for k, v in errs.items():
        record_parity(f"generic_{name}:{k}", v, tol[k])
    assert all(errs[k] <= tol[k] for k in errs), errs
    # deterministic: bitwise run to run
    y2 = ctx.forward(grid, acq, T(tmpl), T(poses), T(p0)).cpu().numpy()
    z2 = ctx.adjoint(grid, acq, T(tmpl), T(poses), T(cot)).cpu().numpy()
    assert np.array_equal(y, y2) and np.array_equal(z, z2)
    # the unit of work is the same window count as the oracle's
    n, _ = ctx.count(grid, acq, T(tmpl), T(poses))
    no, _ = oracle.count(grid, acq, f64(tmpl), f64(poses))
    assert n == no


def test_generic_adjoint_identity(ctx):
    """<A x, y> = <x, A^T y> through K1g / K2g (fp32): the forward and adjoint use one window predicate."""
    grid, acq, _ = case("exp_kappa30", nt=900)
    tmpl, poses = random_scene(44, grid, E=3, F=2, standoff=1.5)
    x = gen.random_volume(grid, 45)
    yv = gen.random_cotangent((2, 3, acq["nt"]), seed=46)
    Ax = ctx.forward(grid, acq, T(tmpl), T(poses), T(x)).double().cpu().numpy()
    ATy = ctx.adjoint(grid, acq, T(tmpl), T(poses), T(yv)).double().cpu().numpy()
    lhs, rhs = float(np.sum(Ax * f64(yv))), float(np.sum(f64(x) * ATy))
    assert abs(lhs - rhs) <= 1e-5 * max(abs(lhs), abs(rhs)), (lhs, rhs)


@pytest.mark.parametrize("name", ["pow1.5_kappa10", "gauss_sigma2.0"])
def test_generic_step(ctx, name):
    """pa_step (forward + NC loss + adjoint + pose gradient + Adam) on the generic kernels vs oracle.step."""
    grid, acq, _ = case(name, nt=1000)
    tmpl = gen.linear_array(6, 0.3)
    e_true = np.array([[0.05, -0.1, 0.02, 0.1, 0.2, grid["origin"][2] - 1.5],
                       [-0.05, 0.08, 0.0, -0.3, 0.1, grid["origin"][2] - 1.8]])
    p_true = gen.random_volume(grid, 3)
    meas = oracle.forward(grid, acq, f64(tmpl), f64(gen.poses_from_euler(e_true)), f64(p_true))
    e0 = e_true + np.array([0.01, -0.01, 0.005, 0.05, -0.05, 0.02])
    p0 = np.full(p_true.shape, 0.4)
    nv = p0.size
    out = oracle.step(grid, acq, f64(tmpl), f64(meas), f64(p0), f64(e0), np.zeros(2 * nv), np.zeros(24), lr_p0=1e-2,
                      lr_rot=1e-3, lr_trans=1e-2, loss_kind=1)
    g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    geul = torch.empty((2, 6), device="cuda")
    p_d, e_d = T(p0), T(e0)
    ctx.step(grid, acq, T(tmpl), T(meas), p_d, e_d, torch.zeros(2 * nv, device="cuda"), torch.zeros(24, device="cuda"),
             g, L, dict(lr_p0=1e-2, lr_rot=1e-3, lr_trans=1e-2, step=1, loss_kind=1), grad_euler=geul, check=True)
    torch.cuda.synchronize()
    assert rel(g.cpu().numpy(), out["grad_p0"]) <= TOL_FA
    assert rel(geul.cpu().numpy(), out["grad_euler"]) <= TOL_POSE
    assert abs(float(L[0]) - out["loss"]) <= 1e-4 * abs(out["loss"])
