"""GPU (libpa, sm_100a) vs fp64 oracle parity — the parity tests proper (-m gpu).

Tolerances (north_star): forward and adjoint <= 1e-4 relative L2, pose gradients
<= 1e-3 relative L2 (over the stacked tensor, R15); the unit-of-work count is bit-exact.
All inputs are seeded synthetic data from paper_2604_09643_b200.gen.  Everything is
computed through the C ABI (ctypes binding).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2604_09643_b200 import gen
from paper_2604_09643_b200._pa import PAError, PA_EINVAL, PA_EDEGENERATE, PA_EUNSUPPORTED, PA_ESHAPE

pytestmark = pytest.mark.gpu

TOL_FA = 1e-4
TOL_POSE = 1e-3


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_09643_b200 import Context
    import __graft_entry__

    __graft_entry__.build()
    return Context(0)


def T(a):
    return torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")


def f64(a):
    """The exact fp32 values the GPU sees, widened for the oracle."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rel(a, b):
    a, b = np.ravel(np.asarray(a, dtype=np.float64)), np.ravel(np.asarray(b, dtype=np.float64))
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def grid32(g):
    """grid dict with the fp32-rounded origin/pitch the ABI receives (so the oracle sees them too)."""
    return dict(g, origin=[float(np.float32(o)) for o in g["origin"]], pitch=float(np.float32(g["pitch"])))


def acq32(a):
    return {k: (float(np.float32(v)) if isinstance(v, float) else v) for k, v in a.items()}


def run_all(ctx, grid, acq, tmpl, poses, p0, cot):
    grid, acq = grid32(grid), acq32(acq)
    y = ctx.forward(grid, acq, T(tmpl), T(poses), T(p0)).cpu().numpy()
    z = ctx.adjoint(grid, acq, T(tmpl), T(poses), T(cot)).cpu().numpy()
    gp, ge = ctx.pose_grad(grid, acq, T(tmpl), T(poses), T(p0), T(cot))
    yo = oracle.forward(grid, acq, f64(tmpl), f64(poses), f64(p0))
    zo = oracle.adjoint(grid, acq, f64(tmpl), f64(poses), f64(cot))
    po, geo = oracle.pose_grad(grid, acq, f64(tmpl), f64(poses), f64(p0), f64(cot))
    return (y, yo), (z, zo), (gp.cpu().numpy(), po), (ge.cpu().numpy(), geo)


def random_scene(seed, grid, E, F, standoff=3.0):
    rng = np.random.default_rng(seed)
    tmpl = rng.normal(size=(E, 3)) * 1.5
    e = np.zeros((F, 6))
    e[:, :3] = rng.normal(scale=0.3, size=(F, 3))
    e[:, 3:5] = rng.normal(scale=1.0, size=(F, 2))
    e[:, 5] = grid["origin"][2] - standoff - rng.uniform(0, 2, size=F)
    return tmpl, gen.poses_from_euler(e)


# ------------------------------------------------------------------------------------ C1 parity
def test_c1_forward_adjoint_pose_parity(ctx, record_parity):
    """BASELINE config 1 in full: 32^3 @ 0.2 mm sphere phantom, 64-element linear array, 512 samples."""
    w = gen.workload("c1")
    p0 = gen.phantom(w)
    cot = gen.random_cotangent((1, 64, 512), seed=7)
    (y, yo), (z, zo), (gp, po), (ge, geo) = run_all(ctx, w.grid, w.acq, w.tmpl, w.poses_true(), p0, cot)
    for m, a, b, t in (("forward", y, yo, TOL_FA), ("adjoint", z, zo, TOL_FA), ("pose", gp, po, TOL_POSE),
                       ("elem", ge, geo, TOL_POSE)):
        record_parity(m, rel(a, b), t)
    assert rel(y, yo) <= TOL_FA, rel(y, yo)
    assert rel(z, zo) <= TOL_FA, rel(z, zo)
    assert rel(gp, po) <= TOL_POSE, rel(gp, po)
    assert rel(ge, geo) <= TOL_POSE, rel(ge, geo)


def test_c1_tilted_pose_and_residual_cotangent(ctx, record_parity):
    w = gen.workload("c1")
    p0 = gen.phantom(w)
    e = w.euler_true.copy()
    e[0, :3] = [0.3, -0.2, 0.15]
    e[0, 3:5] = [0.7, -0.4]
    poses = gen.poses_from_euler(e)
    y_true = oracle.forward(grid32(w.grid), acq32(w.acq), f64(w.tmpl), f64(w.poses_true()), f64(p0))
    cot = 2.0 * (oracle.forward(grid32(w.grid), acq32(w.acq), f64(w.tmpl), f64(poses), f64(p0)) - y_true)
    (y, yo), (z, zo), (gp, po), _ = run_all(ctx, w.grid, w.acq, w.tmpl, poses, p0, cot)
    for m, a, b, t in (("forward", y, yo, TOL_FA), ("adjoint", z, zo, TOL_FA), ("pose", gp, po, TOL_POSE)):
        record_parity(m, rel(a, b), t)
    assert rel(y, yo) <= TOL_FA and rel(z, zo) <= TOL_FA and rel(gp, po) <= TOL_POSE, (rel(y, yo), rel(z, zo), rel(gp, po))


# ------------------------------------------------------------------------------------ ragged multi-tile
@pytest.mark.parametrize("shape", [(21, 19, 13), (8, 8, 4), (1, 1, 1), (33, 9, 5)])
def test_ragged_multi_tile_multi_frame(ctx, shape, record_parity):
    """Grids that span several 8x8x4 tiles with ragged edges, several frames with random poses,
    nt not a multiple of anything, windows clipped at t0 and at nt."""
    grid = gen.make_grid(shape, 0.2)
    acq = gen.make_acq(301, 0.2, t0=1.3)
    tmpl, poses = random_scene(3, grid, E=5, F=3)
    p0 = gen.random_volume(grid, 4)
    cot = gen.random_cotangent((3, 5, 301), seed=5)
    (y, yo), (z, zo), (gp, po), (ge, geo) = run_all(ctx, grid, acq, tmpl, poses, p0, cot)
    for m, a, b, t in (("forward", y, yo, TOL_FA), ("adjoint", z, zo, TOL_FA), ("pose", gp, po, TOL_POSE)):
        record_parity(m, rel(a, b), t)
    assert rel(y, yo) <= TOL_FA, rel(y, yo)
    assert rel(z, zo) <= TOL_FA, rel(z, zo)
    assert rel(gp, po) <= TOL_POSE, rel(gp, po)


@pytest.mark.parametrize("sigma,pitch,t0", [(0.1, 0.1, 3.0), (0.4, 0.4, 1.0), (0.2, 0.1, 2.0)])
def test_other_window_classes(ctx, record_parity, sigma, pitch, t0):
    """The C5 class (sigma = h = 0.1), the C3-coarse class (sigma = h = 0.4), and a finer grid."""
    grid = gen.make_grid((20, 18, 12), pitch)
    acq = gen.make_acq(700, sigma, t0=t0)
    tmpl, poses = random_scene(11, grid, E=4, F=2, standoff=2.0)
    p0 = gen.random_volume(grid, 12)
    cot = gen.random_cotangent((2, 4, 700), seed=13)
    (y, yo), (z, zo), (gp, po), _ = run_all(ctx, grid, acq, tmpl, poses, p0, cot)
    for m, a, b, t in (("forward", y, yo, TOL_FA), ("adjoint", z, zo, TOL_FA), ("pose", gp, po, TOL_POSE)):
        record_parity(m, rel(a, b), t)
    assert rel(y, yo) <= TOL_FA and rel(z, zo) <= TOL_FA and rel(gp, po) <= TOL_POSE, (rel(y, yo), rel(z, zo), rel(gp, po))


# ------------------------------------------------------------------------------------ C2 geometry
def test_c2_geometry_frame_element_subset(ctx, record_parity):
    """BASELINE config 2 geometry (128^3 vascular phantom, 128-element array, 1024 samples) on a
    deterministic frame/element subset small enough for the oracle."""
    w = gen.workload("c2")
    p0 = gen.phantom(w)
    frames = [0, 50]
    tmpl = w.tmpl[::16]
    poses = w.poses_true()[frames]
    cot = gen.random_cotangent((2, tmpl.shape[0], 1024), seed=21)
    (y, yo), (z, zo), (gp, po), _ = run_all(ctx, w.grid, w.acq, tmpl, poses, p0, cot)
    for m, a, b, t in (("forward", y, yo, TOL_FA), ("adjoint", z, zo, TOL_FA), ("pose", gp, po, TOL_POSE)):
        record_parity(m, rel(a, b), t)
    assert rel(y, yo) <= TOL_FA and rel(z, zo) <= TOL_FA and rel(gp, po) <= TOL_POSE, (rel(y, yo), rel(z, zo), rel(gp, po))


# ------------------------------------------------------------------------------------ GPU properties
def test_adjoint_identity_fp32_and_determinism(ctx):
    grid = gen.make_grid((24, 20, 16), 0.2)
    acq = gen.make_acq(400, 0.2, t0=1.0)
    tmpl, poses = random_scene(8, grid, E=6, F=3)
    x = T(gen.random_volume(grid, 1))
    yv = T(gen.random_cotangent((3, 6, 400), 2))
    Ax = ctx.forward(grid32(grid), acq32(acq), T(tmpl), T(poses), x)
    ATy = ctx.adjoint(grid32(grid), acq32(acq), T(tmpl), T(poses), yv)
    lhs = float((Ax.double() * yv.double()).sum())
    rhs = float((x.double() * ATy.double()).sum())
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)
    Ax2 = ctx.forward(grid32(grid), acq32(acq), T(tmpl), T(poses), x)
    ATy2 = ctx.adjoint(grid32(grid), acq32(acq), T(tmpl), T(poses), yv)
    gz, gp, ge = ctx.adjoint_pose(grid32(grid), acq32(acq), T(tmpl), T(poses), x, yv)
    gz2, gp2, ge2 = ctx.adjoint_pose(grid32(grid), acq32(acq), T(tmpl), T(poses), x, yv)
    assert torch.equal(Ax, Ax2) and torch.equal(ATy, ATy2)
    assert torch.equal(gz, gz2) and torch.equal(gp, gp2) and torch.equal(ge, ge2)
    # fused pass == separate passes
    gp_s, ge_s = ctx.pose_grad(grid32(grid), acq32(acq), T(tmpl), T(poses), x, yv)
    assert torch.equal(gz, ATy) and torch.equal(gp, gp_s) and torch.equal(ge, ge_s)
    # pose = chain rule of element gradients (a6)
    G = ge.double().cpu().numpy()
    tm = np.asarray(tmpl, dtype=np.float32).astype(np.float64)
    want = np.concatenate([np.einsum("fea,eb->fab", G, tm).reshape(3, 9), G.sum(1)], axis=1)
    assert rel(gp.double().cpu().numpy(), want) <= 1e-5


def test_linearity_and_zero(ctx):
    grid = gen.make_grid((16, 16, 8), 0.2)
    acq = gen.make_acq(256, 0.2, t0=1.0)
    tmpl, poses = random_scene(9, grid, E=3, F=2)
    a, b = T(gen.random_volume(grid, 1)), T(gen.random_volume(grid, 2))
    fa = ctx.forward(grid32(grid), acq32(acq), T(tmpl), T(poses), a)
    fb = ctx.forward(grid32(grid), acq32(acq), T(tmpl), T(poses), b)
    fab = ctx.forward(grid32(grid), acq32(acq), T(tmpl), T(poses), 2 * a - b)
    assert rel((2 * fa - fb).cpu().numpy(), fab.cpu().numpy()) <= 1e-6
    z = ctx.forward(grid32(grid), acq32(acq), T(tmpl), T(poses), torch.zeros_like(a))
    assert torch.count_nonzero(z) == 0


# ------------------------------------------------------------------------------------ count (bit-exact)
@pytest.mark.parametrize("name", ["c1", "ragged"])
def test_count_bit_exact(ctx, name):
    if name == "c1":
        w = gen.workload("c1")
        grid, acq, tmpl, poses = w.grid, w.acq, w.tmpl, w.poses_true()
    else:
        grid = gen.make_grid((21, 19, 13), 0.2)
        acq = gen.make_acq(301, 0.2, t0=1.3)
        tmpl, poses = random_scene(3, grid, E=5, F=3)
    n, pf = ctx.count(grid32(grid), acq32(acq), T(tmpl), T(poses))
    no, pfo = oracle.count(grid32(grid), acq32(acq), f64(tmpl), f64(poses))
    assert n == no and np.array_equal(pf, pfo)


# ------------------------------------------------------------------------------------ losses and the step
@pytest.mark.parametrize("kind", [0, 1])
def test_loss_parity(ctx, kind):
    rng = np.random.default_rng(3)
    y = rng.normal(size=(3, 4, 200))
    S = y * 0.7 + rng.normal(size=y.shape) * 0.3
    mask = np.array([[1, 1, 0, 1], [1, 0, 1, 1], [1, 1, 1, 1]], dtype=np.uint8)
    L, cot = ctx.loss(kind, T(y), T(S), row_mask=torch.tensor(mask, device="cuda"))
    if kind == 0:
        Lo, co = oracle.mse(f64(y), f64(S))
        co = co * mask[..., None]
        Lo = float(np.sum(((f64(y) - f64(S)) ** 2) * mask[..., None]))
    else:
        Lo, co = oracle.nc(f64(y), f64(S), mask=mask)
    assert abs(float(L) - Lo) <= 1e-5 * abs(Lo)
    assert rel(cot.cpu().numpy(), co) <= 1e-5


@pytest.mark.parametrize("loss_kind", [0, 1])
def test_step_parity(ctx, loss_kind, record_parity):
    """pa_step vs oracle_step: loss, dL/dp0 (1e-4), dL/dEuler (1e-3); Adam updates compared where
    |g| > 1e-3 max|g| (R13: the first Adam step is sign-like)."""
    grid = gen.make_grid((16, 14, 12), 0.2)
    acq = gen.make_acq(320, 0.2, t0=1.0)
    tmpl = gen.linear_array(8, 0.3)
    e_true = np.array([[0.05, -0.1, 0.02, 0.1, 0.2, -4.5], [-0.05, 0.08, 0.0, -0.3, 0.1, -4.8]])
    p_true = gen.random_volume(grid, 3)
    meas = oracle.forward(grid32(grid), acq32(acq), f64(tmpl), f64(gen.poses_from_euler(e_true)), f64(p_true))
    e0 = e_true + np.array([0.01, -0.01, 0.005, 0.05, -0.05, 0.02])
    p0 = np.full(p_true.shape, 0.4)
    nv = p0.size
    cfg = dict(lr_p0=1e-2, lr_rot=1e-3, lr_trans=1e-2, beta1=0.9, beta2=0.999, eps=1e-8, step=1, loss_kind=loss_kind)
    out = oracle.step(grid32(grid), acq32(acq), f64(tmpl), f64(meas), f64(p0), f64(e0), np.zeros(2 * nv),
                      np.zeros(24), lr_p0=cfg["lr_p0"], lr_rot=cfg["lr_rot"], lr_trans=cfg["lr_trans"],
                      loss_kind=loss_kind)
    p_d, e_d = T(p0), T(e0)
    am, ap = torch.zeros(2 * nv, device="cuda"), torch.zeros(24, device="cuda")
    gbuf, loss, geul = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda"), torch.empty((2, 6), device="cuda")
    ctx.step(grid32(grid), acq32(acq), T(tmpl), T(meas), p_d, e_d, am, ap, gbuf, loss, cfg, grad_euler=geul)
    torch.cuda.synchronize()
    assert abs(float(loss[0]) - out["loss"]) <= 1e-4 * abs(out["loss"])
    g = gbuf.cpu().numpy().ravel()
    record_parity("step_grad_p0", rel(g, out["grad_p0"]), TOL_FA)
    record_parity("step_grad_euler", rel(geul.cpu().numpy(), out["grad_euler"]), TOL_POSE)
    assert rel(g, out["grad_p0"]) <= TOL_FA
    assert rel(geul.cpu().numpy(), out["grad_euler"]) <= TOL_POSE
    big = np.abs(out["grad_p0"]) > 1e-3 * np.abs(out["grad_p0"]).max()
    dp = p_d.cpu().numpy().ravel() - p0.ravel()
    dpo = out["p0"].ravel() - p0.ravel()
    assert rel(dp[big], dpo[big]) <= 1e-3
    de = e_d.cpu().numpy() - e0
    deo = out["euler_t"] - e0
    bige = np.abs(out["grad_euler"]) > 1e-3 * np.abs(out["grad_euler"]).max()
    assert rel(de[bige], deo[bige]) <= 1e-3


# ------------------------------------------------------------------------------------ errors / degenerate cases
def test_errors(ctx):
    w = gen.workload("c1")
    p0 = T(gen.phantom(w))
    bad = dict(w.acq, kappa=3.0)
    with pytest.raises(PAError) as ei:
        ctx.forward(w.grid, bad, T(w.tmpl), T(w.poses_true()), p0)
    assert ei.value.status == PA_EINVAL
    with pytest.raises(PAError) as ei:
        ctx.forward(dict(w.grid, pitch=0.0), w.acq, T(w.tmpl), T(w.poses_true()), p0)
    assert ei.value.status == PA_EINVAL
    # an element exactly on a voxel centre
    poses = w.poses_true()
    poses[0, 9:] = [w.grid["origin"][0] + 0.2 * 3, w.grid["origin"][1] + 0.2 * 4, w.grid["origin"][2] + 0.2 * 5]
    tm = np.zeros((1, 3))
    with pytest.raises(PAError) as ei:
        ctx.forward(grid32(w.grid), w.acq, T(tm), T(poses), p0)
    assert ei.value.status == PA_EDEGENERATE
    assert "frame 0 element 0" in str(ei.value)
    # exponential family, L_min = 480: beyond every direct-kernel class -> the generic kernels (parity in
    # test_generic_gpu.py); PA_EUNSUPPORTED only where no kernel at all holds the geometry (nt > 51200 there)
    y = ctx.forward(w.grid, dict(w.acq, sigma=0.3, kappa=30.0, kernel="exp"), T(w.tmpl), T(w.poses_true()), p0)
    assert torch.isfinite(y).all() and float(y.abs().max()) > 0
    with pytest.raises(PAError) as ei:
        ctx.forward(w.grid, dict(w.acq, sigma=0.3, kappa=30.0, kernel="exp", nt=60000), T(w.tmpl), T(w.poses_true()), p0)
    assert ei.value.status == PA_EUNSUPPORTED
    # a Gaussian window below the fast path (L_min = 13) runs on a runtime class of the direct kernels
    y = ctx.forward(grid32(w.grid), dict(w.acq, sigma=0.05), T(w.tmpl), T(w.poses_true()), p0)
    assert torch.isfinite(y).all()


def test_empty_and_far(ctx):
    w = gen.workload("c1")
    p0 = T(gen.phantom(w))
    y = ctx.forward(w.grid, w.acq, T(w.tmpl), T(np.zeros((0, 12))), p0)
    assert y.shape == (0, 64, 512)
    z = ctx.adjoint(w.grid, w.acq, T(w.tmpl), T(np.zeros((0, 12))), T(np.zeros((0, 64, 512))))
    assert torch.count_nonzero(z) == 0
    far = w.poses_true()
    far[0, 11] = -500.0  # all windows beyond nt: everything culled
    y = ctx.forward(w.grid, w.acq, T(w.tmpl), T(far), p0)
    assert torch.count_nonzero(y) == 0


# ------------------------------------------------------------------------------------ full-size sampled parity
TOL_VOX = 1e-4  # per voxel, relative to the voxel's own sum of |terms| (oracle.adjoint_abs)


@pytest.mark.parametrize("name,frames", [("c2", None), ("c4", None), ("c5", (0, 100)), ("c5", (700, 800))])
def test_full_size_sampled_parity(ctx, name, frames, record_parity):
    """At the full BASELINE size and in the launch configuration bench.py times (all frames, all
    elements, full grid), compare sampled outputs the oracle can compute one by one: trace rows (f, e),
    adjoint voxels (1-voxel oracle grids at the exact fp64 centre), each voxel judged against its OWN sum
    of |terms| (a wrong small voxel cannot hide behind a large one), and element-gradient rows.  C5
    (512x512x256 @ 0.1 mm, 256-element bowl, sigma = 0.1) runs its full grid, array and record length on
    100-frame shards of its 800-frame sweep (one GPU's shard at 8 GPUs): frames 0-99 and 700-799, the far
    end of the 90 degree sweep."""
    w = gen.workload(name)
    grid, acq = grid32(w.grid), acq32(w.acq)
    p0 = gen.phantom(w).astype(np.float32)
    poses = w.poses_true()
    if frames is not None:
        poses = poses[frames[0]:frames[1]]
    F = poses.shape[0]
    rng = np.random.default_rng(99)
    cot = rng.normal(size=(F, w.E, acq["nt"])).astype(np.float32)
    y = ctx.forward(grid, acq, T(w.tmpl), T(poses), T(p0))
    gz, gp, ge = ctx.adjoint_pose(grid, acq, T(w.tmpl), T(poses), T(p0), T(cot))
    y, gz, ge = y.cpu().numpy(), gz.cpu().numpy(), ge.cpu().numpy()
    tag = name if frames is None else f"{name}_f{frames[0]}"
    # sampled trace rows
    for f, e in [(0, 0), (F // 2, w.E // 2), (F - 1, w.E - 1)]:
        yo = oracle.forward(grid, acq, f64(w.tmpl[e:e + 1]), f64(poses[f:f + 1]), f64(p0))[0, 0]
        record_parity(f"{tag}_forward_row_{f}_{e}", rel(y[f, e], yo), TOL_FA)
        assert rel(y[f, e], yo) <= TOL_FA, (f, e, rel(y[f, e], yo))
    # sampled adjoint voxels, each against its own sum of |terms|
    worst = 0.0
    nz_checked = 0
    for _ in range(24):
        i, j, k = rng.integers(0, grid["nx"]), rng.integers(0, grid["ny"]), rng.integers(0, grid["nz"])
        o = [float(np.float32(grid["origin"][0])) + float(np.float32(grid["pitch"])) * i,
             float(np.float32(grid["origin"][1])) + float(np.float32(grid["pitch"])) * j,
             float(np.float32(grid["origin"][2])) + float(np.float32(grid["pitch"])) * k]
        g1 = dict(nx=1, ny=1, nz=1, origin=o, pitch=grid["pitch"])
        zo = oracle.adjoint(g1, acq, f64(w.tmpl), f64(poses), f64(cot))[0, 0, 0]
        za = oracle.adjoint_abs(g1, acq, f64(w.tmpl), f64(poses), f64(cot))[0, 0, 0]
        if za == 0.0:
            assert gz[k, j, i] == 0.0
            continue
        nz_checked += 1
        err = abs(float(gz[k, j, i]) - zo) / za
        worst = max(worst, err)
        assert err <= TOL_VOX, ((i, j, k), float(gz[k, j, i]), zo, za)
    record_parity(f"{tag}_adjoint_voxel_vs_sum_abs_terms", worst, TOL_VOX)
    assert nz_checked >= 12
    # sampled element-gradient rows
    for f, e in [(0, w.E // 3), (F - 1, 2 * w.E // 3)]:
        go = oracle.elem_grad(grid, acq, f64(w.tmpl[e:e + 1]), f64(poses[f:f + 1]), f64(p0), f64(cot[f:f + 1, e:e + 1]))
        record_parity(f"{tag}_elem_row_{f}_{e}", rel(ge[f, e], go[0, 0]), TOL_POSE)
        assert rel(ge[f, e], go[0, 0]) <= TOL_POSE, (f, e, rel(ge[f, e], go[0, 0]))
    # sampled frames of the pose gradient [F][12] (every element of the frame) where the oracle affords it
    if name == "c2":
        for f in (0, F - 1):
            po, _ = oracle.pose_grad(grid, acq, f64(w.tmpl), f64(poses[f:f + 1]), f64(p0), f64(cot[f:f + 1]))
            record_parity(f"{tag}_pose_frame_{f}", rel(gp[f].cpu().numpy(), po[0]), TOL_POSE)
            assert rel(gp[f].cpu().numpy(), po[0]) <= TOL_POSE, (f, rel(gp[f].cpu().numpy(), po[0]))
