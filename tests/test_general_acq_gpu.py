"""General acquisition parameters on the GPU (-m gpu): the speed of sound c, the sampling interval dt, the
Gaussian width sigma and the cut-off kappa are free parameters of Eq. gpu_forward_model; the
paper's dynamic smoothing decays sigma continuously (Alg. 1).  The Gaussian fast path (K1d,
K2a/K2c, K2s) takes the window length L_min = floor(2 kappa sigma / (c dt)) at run time, so any such
acquisition with 21 <= L_min <= 512 runs.  Each case: forward, adjoint and pose gradient vs
the fp64 oracle on a ragged multi-tile grid, several frames, windows clipped at both ends."""
import numpy as np
import pytest

import oracle
from paper_2604_09643_b200 import gen, plan_info

from test_gpu_parity import TOL_FA, TOL_POSE, T, acq32, ctx, f64, grid32, random_scene, rel  # noqa: F401

pytestmark = pytest.mark.gpu

CASES = {
    # name: (pitch, acquisition overrides, expected L_min)
    "tissue_c1.54": (0.2, dict(c=1.54), 51),
    "fs50MHz": (0.2, dict(dt=0.02), 66),
    "kappa6": (0.2, dict(kappa=6.0), 64),
    "sigma0.15": (0.2, dict(sigma=0.15), 40),
    "sigma0.25": (0.2, dict(sigma=0.25), 66),
    "sigma0.3": (0.2, dict(sigma=0.3), 80),
    "sigma0.5": (0.2, dict(sigma=0.5), 133),
    "sigma0.6": (0.2, dict(sigma=0.6), 160),
    "sigma0.9": (0.2, dict(sigma=0.9), 239),
    "sigma1.0": (0.2, dict(sigma=1.0), 266),
    "sigma1.6_h0.8": (0.8, dict(sigma=1.6), 426),
    "sigma1.9": (0.2, dict(sigma=1.9), 506),
    "sigma0.08_h0.1": (0.1, dict(sigma=0.08), 21),
    "c1.54_fs50_kappa6_s0.22": (0.2, dict(c=1.54, dt=0.02, kappa=6.0, sigma=0.22), 85),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_general_acquisition_parity(ctx, name, record_parity):
    pitch, over, lmin = CASES[name]
    grid = gen.make_grid((21, 17, 13), pitch)
    acq = dict(gen.make_acq(700, 0.2, t0=1.0), **over)
    tmpl, poses = random_scene(31, grid, E=4, F=2, standoff=2.0)
    g, a = grid32(grid), acq32(acq)
    info = plan_info(g, a, 4)
    assert info["lmin"] == lmin and info["fwd_deposit"] == 1 and info["adj_kernel"] in (1, 2), info
    p0 = gen.random_volume(grid, 32)
    cot = gen.random_cotangent((2, 4, 700), seed=33)
    y = ctx.forward(g, a, T(tmpl), T(poses), T(p0)).cpu().numpy()
    gz, gp, ge = ctx.adjoint_pose(g, a, T(tmpl), T(poses), T(p0), T(cot))
    yo = oracle.forward(g, a, f64(tmpl), f64(poses), f64(p0))
    zo = oracle.adjoint(g, a, f64(tmpl), f64(poses), f64(cot))
    po, geo = oracle.pose_grad(g, a, f64(tmpl), f64(poses), f64(p0), f64(cot))
    assert np.abs(yo).max() > 0
    errs = dict(forward=rel(y, yo), adjoint=rel(gz.cpu().numpy(), zo), pose=rel(gp.cpu().numpy(), po),
                elem=rel(ge.cpu().numpy(), geo))
    tol = dict(forward=TOL_FA, adjoint=TOL_FA, pose=TOL_POSE, elem=TOL_POSE)
    for k, v in errs.items():
        record_parity(f"{name}:{k}", v, tol[k])
    assert all(errs[k] <= tol[k] for k in errs), errs
    # the unit of work: exact count, bit-exact vs the oracle
    n, pf = ctx.count(g, a, T(tmpl), T(poses))
    no, pfo = oracle.count(g, a, f64(tmpl), f64(poses))
    assert n == no and np.array_equal(pf, pfo)


@pytest.mark.parametrize("name", ["tissue_c1.54", "sigma0.3"])
def test_general_acquisition_step(ctx, name):
    """pa_step (forward + NC loss + adjoint + pose gradient + Adam) at a general acquisition vs oracle.step."""
    pitch, over, _ = CASES[name]
    grid = grid32(gen.make_grid((16, 14, 12), pitch))
    acq = acq32(dict(gen.make_acq(400, 0.2, t0=1.0), **over))
    tmpl = gen.linear_array(8, 0.3)
    e_true = np.array([[0.05, -0.1, 0.02, 0.1, 0.2, -4.5], [-0.05, 0.08, 0.0, -0.3, 0.1, -4.8]])
    p_true = gen.random_volume(grid, 3)
    meas = oracle.forward(grid, acq, f64(tmpl), f64(gen.poses_from_euler(e_true)), f64(p_true))
    e0 = e_true + np.array([0.01, -0.01, 0.005, 0.05, -0.05, 0.02])
    p0 = np.full(p_true.shape, 0.4)
    nv = p0.size
    out = oracle.step(grid, acq, f64(tmpl), f64(meas), f64(p0), f64(e0), np.zeros(2 * nv), np.zeros(24), lr_p0=1e-2,
                      lr_rot=1e-3, lr_trans=1e-2, loss_kind=1)
    import torch

    g, L, geul = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda"), torch.empty((2, 6), device="cuda")
    ctx.step(grid, acq, T(tmpl), T(meas), T(p0), T(e0), torch.zeros(2 * nv, device="cuda"),
             torch.zeros(24, device="cuda"), g, L, dict(lr_p0=1e-2, lr_rot=1e-3, lr_trans=1e-2, step=1, loss_kind=1),
             grad_euler=geul, check=True)
    torch.cuda.synchronize()
    assert abs(float(L[0]) - out["loss"]) <= 1e-4 * abs(out["loss"])
    assert rel(g.cpu().numpy(), out["grad_p0"]) <= TOL_FA
    assert rel(geul.cpu().numpy(), out["grad_euler"]) <= TOL_POSE
