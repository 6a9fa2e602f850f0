"""pa_step on the GPU beyond the first iteration (-m gpu), through the C ABI:

* several consecutive steps with a NONZERO Adam state, both loss kinds, pose updates on, against the same
  oracle.step sequence (Adam: P:87; the oracle's Adam is pinned by tests/golden/adam_steps.txt);
* the cross-rank all-reduce callback (a7, Stage 5 "coherently combining") as libpa calls it from
  inside pa_step: a world-1 callback that doubles the buffer, a failing callback (PA_ECUDA);
* the asynchronous degenerate-geometry check of pa_step (R10): no host synchronisation, the step's Adam
  updates skipped on the device, the verdict from pa_step_status;
* the TGV weight lambda applied inside the kernel (no fp32 rounding of lambda - 1, R20).
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from oracle.tgv import tgv as tgv_oracle
from paper_2604_09643_b200 import gen
from paper_2604_09643_b200._pa import ALLREDUCE_FN, PA_ECUDA, PA_EDEGENERATE, PAError

from test_gpu_parity import TOL_FA, TOL_POSE, T, acq32, ctx, f64, grid32, rel  # noqa: F401

pytestmark = pytest.mark.gpu


def small_problem(seed=3, F=3):
    grid = gen.make_grid((16, 14, 12), 0.2)
    acq = gen.make_acq(320, 0.2, t0=1.0)
    tmpl = gen.linear_array(8, 0.3)
    rng = np.random.default_rng(seed)
    e_true = np.zeros((F, 6))
    e_true[:, :3] = rng.normal(scale=0.05, size=(F, 3))
    e_true[:, 3:5] = rng.normal(scale=0.3, size=(F, 2))
    e_true[:, 5] = -4.5 - rng.uniform(0, 0.4, size=F)
    p_true = gen.random_volume(grid, seed)
    meas = oracle.forward(grid32(grid), acq32(acq), f64(tmpl), f64(gen.poses_from_euler(e_true)), f64(p_true))
    e0 = e_true + rng.normal(scale=[0.01, 0.01, 0.01, 0.05, 0.05, 0.05], size=(F, 6))
    p0 = np.full(p_true.shape, 0.4) + 0.05 * rng.random(p_true.shape)
    return grid32(grid), acq32(acq), tmpl, meas, p0, e0


@pytest.mark.parametrize("loss_kind", [0, 1])
def test_multistep_adam_parity(ctx, loss_kind, record_parity):
    """5 consecutive pa_step calls (t = 2..6) from a nonzero Adam state vs oracle.step.  State-synced: before
    every step the oracle receives the GPU's state (p0, Euler+t, both Adam states), so each step's map is
    compared on identical inputs: loss, dL/dp0 (1e-4), dL/dEuler (1e-3), the p0 / pose updates and the new
    Adam moments (1e-3; the state is nonzero everywhere, so no sign-like first step, R13).  Then the
    free-running 5-step trajectories of both sides are compared (1e-3)."""
    grid, acq, tmpl, meas, p0, e0 = small_problem(seed=4 + loss_kind)
    F, nv = e0.shape[0], p0.size
    lr = dict(lr_p0=5e-3, lr_rot=2e-3, lr_trans=1e-2)
    # gradient scale for a meaningful nonzero initial state
    g0 = oracle.step(grid, acq, f64(tmpl), f64(meas), f64(p0), f64(e0), np.zeros(2 * nv), np.zeros(12 * F),
                     loss_kind=loss_kind, update_p0=False, update_pose=False, **lr)
    rng = np.random.default_rng(11)
    gs, qs = np.sqrt(np.mean(g0["grad_p0"] ** 2)), np.sqrt(np.mean(g0["grad_euler"] ** 2, axis=0))
    st_p = np.concatenate([0.5 * gs * rng.normal(size=nv), gs * gs * rng.uniform(0.5, 1.5, size=nv)])
    qrep = np.tile(qs, F)
    st_q = np.concatenate([0.5 * qrep * rng.normal(size=6 * F), qrep * qrep * rng.uniform(0.5, 1.5, size=6 * F)])
    p_d, e_d = T(p0), T(e0)
    ap_d, aq_d = T(st_p), T(st_q)
    gbuf, loss = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    geul = torch.empty((F, 6), device="cuda")
    free = dict(p0=f64(p0), euler_t=f64(e0), adam_p0=f64(st_p), adam_pose=f64(st_q))
    worst = {}
    for t in range(2, 7):
        before = dict(p0=p_d.double().cpu().numpy(), euler_t=e_d.double().cpu().numpy(),
                      adam_p0=ap_d.double().cpu().numpy(), adam_pose=aq_d.double().cpu().numpy())
        out = oracle.step(grid, acq, f64(tmpl), f64(meas), before["p0"], before["euler_t"], before["adam_p0"],
                          before["adam_pose"], t=t, loss_kind=loss_kind, **lr)
        cfg = dict(beta1=0.9, beta2=0.999, eps=1e-8, step=t, loss_kind=loss_kind, **lr)
        ctx.step(grid, acq, T(tmpl), T(meas), p_d, e_d, ap_d, aq_d, gbuf, loss, cfg, grad_euler=geul, check=True)
        torch.cuda.synchronize()
        errs = {
            "loss": abs(float(loss[0]) - out["loss"]) / abs(out["loss"]),
            "grad_p0": rel(gbuf.cpu().numpy(), out["grad_p0"]),
            "grad_euler": rel(geul.cpu().numpy(), out["grad_euler"]),
            "dp0": rel(p_d.double().cpu().numpy().ravel() - before["p0"].ravel(), out["p0"].ravel() - before["p0"].ravel()),
            "deuler": rel(e_d.double().cpu().numpy() - before["euler_t"], out["euler_t"] - before["euler_t"]),
            "adam_m_p0": rel(ap_d.cpu().numpy()[:nv], out["adam_p0"][:nv]),
            "adam_v_p0": rel(ap_d.cpu().numpy()[nv:], out["adam_p0"][nv:]),
            "adam_pose": rel(aq_d.cpu().numpy(), out["adam_pose"]),
        }
        tol = {"loss": 1e-4, "grad_p0": TOL_FA, "grad_euler": TOL_POSE}
        for k, v in errs.items():
            worst[k] = max(worst.get(k, 0.0), v)
            assert v <= tol.get(k, 1e-3), (t, k, v)
        free_out = oracle.step(grid, acq, f64(tmpl), f64(meas), free["p0"], free["euler_t"], free["adam_p0"],
                               free["adam_pose"], t=t, loss_kind=loss_kind, **lr)
        free = {k: free_out[k] for k in free}
    for k, v in worst.items():
        record_parity(f"multistep_{k}", v, {"loss": 1e-4, "grad_p0": TOL_FA, "grad_euler": TOL_POSE}.get(k, 1e-3))
    # free-running: 5 GPU steps vs 5 oracle steps from the same start
    d0 = p_d.double().cpu().numpy().ravel() - f64(p0).ravel()
    record_parity("multistep_free_p0", rel(d0, free["p0"].ravel() - f64(p0).ravel()), 1e-3)
    assert rel(d0, free["p0"].ravel() - f64(p0).ravel()) <= 1e-3
    de = e_d.double().cpu().numpy() - f64(e0)
    assert rel(de, free["euler_t"] - f64(e0)) <= 1e-3


def test_allreduce_callback_inside_pa_step(ctx):
    """a7 as libpa runs it: pa_step calls the callback for grad_p0 (nvox floats) and for loss + 1 (1 float)
    on its stream.  A world-1 callback that doubles the buffer -> grad_p0 exactly 2x, loss[1] = 2 loss[0], and
    Adam (run after the callback) sees the doubled gradient; a callback returning non-zero -> PA_ECUDA."""
    grid, acq, tmpl, meas, p0, e0 = small_problem(seed=7, F=2)
    nv, F = p0.size, e0.shape[0]
    cfg = dict(lr_p0=1e-2, lr_rot=1e-3, lr_trans=1e-3, step=1, update_p0=0, update_pose=0)

    def run(allreduce, c=cfg):
        g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
        p = T(p0)
        ctx.step(grid, acq, T(tmpl), T(meas), p, T(e0), torch.zeros(2 * nv, device="cuda"),
                 torch.zeros(12 * F, device="cuda"), g, L, c, allreduce=allreduce)
        torch.cuda.synchronize()
        return g, L, p

    calls = []

    def double(t):
        calls.append(t.numel())
        t.mul_(2.0)

    g1, L1, _ = run(None)
    g2, L2, _ = run(double)
    assert calls == [nv, 1]
    assert torch.equal(g2, 2.0 * g1)
    assert float(L2[1]) == 2.0 * float(L2[0]) and float(L2[0]) == float(L1[0])
    # Adam runs after the callback, on the reduced gradient: from a nonzero second moment the update depends on
    # the gradient's scale, and matches oracle.adam (pinned by tests/golden/adam_steps.txt) applied to 2 g
    g_np = g1.double().cpu().numpy()
    v0 = np.full(nv, float(np.mean(g_np ** 2)))
    am = torch.cat([torch.zeros(nv, device="cuda"), T(v0)])
    g3, L3 = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    p3 = T(p0)
    ctx.step(grid, acq, T(tmpl), T(meas), p3, T(e0), am, torch.zeros(12 * F, device="cuda"), g3, L3,
             dict(cfg, update_p0=1, step=2), allreduce=double)
    torch.cuda.synchronize()
    want, _, _ = oracle.adam(f64(p0).ravel(), np.zeros(nv), f64(v0), 2.0 * g_np, lr=1e-2, t=2, clamp=0.0)
    assert rel(p3.double().cpu().numpy().ravel() - f64(p0).ravel(), want - f64(p0).ravel()) <= 1e-4  # fp32 ulp(p0) / update
    not_doubled, _, _ = oracle.adam(f64(p0).ravel(), np.zeros(nv), f64(v0), g_np, lr=1e-2, t=2, clamp=0.0)
    assert rel(want - f64(p0).ravel(), not_doubled - f64(p0).ravel()) > 0.1  # the check can tell them apart

    def broken(t):
        raise RuntimeError("collective failed")

    with pytest.raises(PAError) as ei:
        run(broken)
    assert ei.value.status == PA_ECUDA and "all-reduce callback failed" in str(ei.value)
    # a raw C callback returning non-zero (no Python exception path)
    rc = ALLREDUCE_FN(lambda buf, n, s, u: 3)
    from paper_2604_09643_b200._pa import StepCfg, make_acq, make_grid
    c = StepCfg()
    c.lr_p0, c.lr_rot, c.lr_trans, c.beta1, c.beta2, c.eps, c.step = 1e-2, 1e-3, 1e-3, 0.9, 0.999, 1e-8, 1
    g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    p, e = T(p0), T(e0)
    am, aq = torch.zeros(2 * nv, device="cuda"), torch.zeros(12 * F, device="cuda")
    m, tm = T(meas), T(tmpl)
    st = ctx.lib.pa_step(ctx.h, ctypes.byref(make_grid(grid)), ctypes.byref(make_acq(acq)),
                         ctypes.c_void_p(tm.data_ptr()), 8, F, ctypes.c_void_p(m.data_ptr()), None,
                         ctypes.c_void_p(p.data_ptr()), ctypes.c_void_p(e.data_ptr()), ctypes.c_void_p(am.data_ptr()),
                         ctypes.c_void_p(aq.data_ptr()), ctypes.byref(c), rc, None, ctypes.c_void_p(g.data_ptr()),
                         ctypes.c_void_p(L.data_ptr()), None, None, None, None,
                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == PA_ECUDA


def test_allreduce_on_a_side_stream(ctx):
    """pa_step on a non-current stream: the callback runs the collective on libpa's stream (the binding makes
    it current), so the reduced gradient is what Adam consumes (stream ordering)."""
    grid, acq, tmpl, meas, p0, e0 = small_problem(seed=8, F=2)
    nv, F = p0.size, e0.shape[0]
    s = torch.cuda.Stream()
    seen = []

    def on_stream(t):
        seen.append(torch.cuda.current_stream().cuda_stream)
        t.mul_(3.0)

    g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    g_ref, L_ref = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    cfg = dict(lr_p0=1e-2, lr_rot=1e-3, lr_trans=1e-3, step=1, update_p0=0, update_pose=0)
    args = (grid, acq, T(tmpl), T(meas), T(p0), T(e0))
    torch.cuda.synchronize()
    ctx.step(*args, torch.zeros(2 * nv, device="cuda"), torch.zeros(12 * F, device="cuda"), g, L, cfg,
             allreduce=on_stream, stream=s)
    s.synchronize()
    ctx.step(*args, torch.zeros(2 * nv, device="cuda"), torch.zeros(12 * F, device="cuda"), g_ref, L_ref, cfg)
    torch.cuda.synchronize()
    assert seen and all(x == s.cuda_stream for x in seen)
    assert torch.equal(g, 3.0 * g_ref)


def test_degenerate_step_is_async_and_skips_adam(ctx):
    """An element exactly on a voxel centre (R10): pa_step returns without synchronising, leaves p0, the
    poses and both Adam states untouched, and pa_step_status reports PA_EDEGENERATE naming the pair; the
    next good step clears the verdict."""
    grid, acq, tmpl, meas, p0, e0 = small_problem(seed=9, F=2)
    nv, F = p0.size, e0.shape[0]
    bad = e0.copy()
    bad[1, :3] = 0.0
    o = np.asarray(grid["origin"])
    bad[1, 3:] = o + 0.2 * np.array([3, 4, 5]) - np.asarray(tmpl[0])  # element 0 of frame 1 on voxel (3,4,5)
    p, e = T(p0), T(bad)
    am, aq = T(np.full(2 * nv, 1e-3)), T(np.full(12 * F, 1e-3))
    snap = [x.clone() for x in (p, e, am, aq)]
    g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    cfg = dict(lr_p0=1e-2, lr_rot=1e-3, lr_trans=1e-3, step=2)
    ctx.step(grid, acq, T(tmpl), T(meas), p, e, am, aq, g, L, cfg)
    with pytest.raises(PAError) as ei:
        ctx.step_status()
    assert ei.value.status == PA_EDEGENERATE and "frame 1 element 0" in str(ei.value)
    for a, b in zip((p, e, am, aq), snap):
        assert torch.equal(a, b)
    ctx.step(grid, acq, T(tmpl), T(meas), p, T(e0), am, aq, g, L, cfg, check=True)  # good geometry: no error
    assert not torch.equal(p, snap[0])


def test_tgv_lambda_applied_in_kernel(ctx):
    """The w update uses lambda dTGV/dw for a lambda so small that the r1 form (scaling by lambda - 1 in fp32)
    lost it (1e-8): the first Adam moment of w equals (1 - b1) lambda dTGV/dw of pa_tgv and of the oracle."""
    grid, acq, tmpl, meas, p0, e0 = small_problem(seed=10, F=2)
    nv, F = p0.size, e0.shape[0]
    rng = np.random.default_rng(2)
    w = rng.normal(size=(3,) + p0.shape) * 0.1
    lam = 1e-8
    g_data = torch.empty(nv, device="cuda")
    L = torch.empty(2, device="cuda")
    base = dict(lr_p0=1e-3, lr_rot=0.0, lr_trans=0.0, step=1, update_p0=0, update_pose=0)
    ctx.step(grid, acq, T(tmpl), T(meas), T(p0), T(e0), torch.zeros(2 * nv, device="cuda"),
             torch.zeros(12 * F, device="cuda"), g_data, L, base)
    g = torch.empty(nv, device="cuda")
    wt = T(w)
    aw = torch.zeros(6 * nv, device="cuda")
    cfg = dict(base, update_p0=1, tgv_lambda=lam, tgv_alpha1=1.0, tgv_alpha0=2.0, tgv_eps=1e-3)
    ctx.step(grid, acq, T(tmpl), T(meas), T(p0), T(e0), torch.zeros(2 * nv, device="cuda"),
             torch.zeros(12 * F, device="cuda"), g, L, cfg, tgv_w=wt, adam_w=aw)
    _, gP, gw = ctx.tgv(grid, T(p0), T(w), 1.0, 2.0, 1e-3)
    torch.cuda.synchronize()
    # grad_p0 += lambda dTGV/dP is below fp32 resolution of the data gradient here (checked at lambda = 0.3 in
    # test_tgv_gpu.test_step_with_tgv); the w gradient is lambda dTGV/dw alone:
    # Adam moment of w after one step from zero: m = (1 - b1) lambda dTGV/dw, exactly representable scale
    m_w = aw[: 3 * nv].double()
    assert rel(m_w.cpu().numpy(), (0.1 * lam * gw.double().ravel()).cpu().numpy()) <= 1e-6
    vo, _, gwo = tgv_oracle(f64(p0), f64(w), float(np.float32(0.2)), 1.0, 2.0, 1e-3)
    assert rel(m_w.cpu().numpy(), 0.1 * lam * gwo.ravel()) <= 1e-5


def test_pa_step_does_not_synchronise_the_host(ctx):
    """pa_step enqueues its whole SfM iteration and returns (R25): on the C2 workload (~0.2 s of
    device work per step) the host call returns in a small fraction of the device time, and a second step can be
    enqueued behind the first without waiting."""
    import time

    w = gen.workload("c2", frames=60)
    grid, acq = grid32(w.grid), acq32(w.acq)
    tm = T(w.tmpl)
    meas = ctx.forward(grid, acq, tm, T(w.poses_true()), T(gen.phantom(w)))
    nv = w.grid["nx"] * w.grid["ny"] * w.grid["nz"]
    p = torch.full((nv,), 0.05, device="cuda")
    eu = T(w.euler_true)
    am, aq = torch.zeros(2 * nv, device="cuda"), torch.zeros(12 * w.F, device="cuda")
    g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    cfg = dict(lr_p0=1e-3, lr_rot=1e-3, lr_trans=1e-2, step=1)
    ctx.step(grid, acq, tm, meas, p, eu, am, aq, g, L, cfg)  # warm-up (workspace allocation)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    ctx.step(grid, acq, tm, meas, p, eu, am, aq, g, L, dict(cfg, step=2))
    ctx.step(grid, acq, tm, meas, p, eu, am, aq, g, L, dict(cfg, step=3))
    host_s = time.perf_counter() - t0
    b.record()
    torch.cuda.synchronize()
    dev_s = a.elapsed_time(b) / 1e3
    assert dev_s > 0.05 and host_s < 0.25 * dev_s, (host_s, dev_s)
    ctx.step_status()


@pytest.mark.parametrize("loss_kind", [0, 1])
def test_p0_only_step_skips_pose_gradient(ctx, loss_kind):
    """update_pose = 0 with no grad_euler requested runs the adjoint without the pose moment (pa.h): grad_p0,
    the loss and the p0 update are bitwise those of the same step with the pose gradient computed, the poses
    are untouched, and fewer libpa kernels run (no pose reduction / Euler chain)."""
    grid, acq, tmpl, meas, p0, e0 = small_problem(seed=11, F=3)
    nv, F = p0.size, e0.shape[0]
    cfg = dict(lr_p0=1e-2, lr_rot=1e-3, lr_trans=1e-3, step=1, update_p0=1, update_pose=0, loss_kind=loss_kind)

    def run(want_euler):
        g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
        p, e = T(p0), T(e0)
        geul = torch.empty((F, 6), device="cuda") if want_euler else None
        n0 = ctx.launch_count()
        ctx.step(grid, acq, T(tmpl), T(meas), p, e, torch.zeros(2 * nv, device="cuda"),
                 torch.zeros(12 * F, device="cuda"), g, L, cfg, grad_euler=geul)
        torch.cuda.synchronize()
        return g, L, p, e, ctx.launch_count() - n0

    g1, L1, p1, e1, n1 = run(True)
    g2, L2, p2, e2, n2 = run(False)
    assert torch.equal(g1, g2) and torch.equal(L1, L2) and torch.equal(p1, p2)
    assert torch.equal(e2, T(e0)) and torch.equal(e1, T(e0))
    assert n2 < n1
