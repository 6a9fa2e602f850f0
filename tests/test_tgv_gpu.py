"""TGV^2 regulariser on the GPU (f4; reading R20 of Eq. 2) vs the fp64 oracle, through the ABI."""
import numpy as np
import pytest
import torch

import oracle
from oracle.tgv import tgv as tgv_oracle
from paper_2604_09643_b200 import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    from paper_2604_09643_b200 import Context

    __graft_entry__.build()
    return Context(0)


def T(a):
    return torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")


def f64(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rel(a, b):
    a, b = np.ravel(a), np.ravel(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# nz > 32: several z slabs; nx % 4 == 0 runs the TMA-staged kernel (k_tgv_tma), other widths the
# register-streamed k_tgv
@pytest.mark.parametrize("shape", [(13, 19, 21), (2, 2, 2), (32, 32, 32), (1, 5, 7), (70, 9, 11), (33, 12, 40),
                                   (70, 9, 12), (5, 3, 4), (40, 17, 68)])
def test_tgv_parity(ctx, shape, record_parity):
    rng = np.random.default_rng(sum(shape))
    grid = gen.make_grid(shape[::-1], 0.2)
    P = rng.random(shape) if shape != (32, 32, 32) else gen.vascular_phantom(grid, seed=2)
    w = rng.normal(size=(3,) + shape) * 0.5
    a1, a0, eps = 1.0, 2.0, 1e-3
    v, gP, gw = ctx.tgv(grid, T(P), T(w), a1, a0, eps)
    vo, gPo, gwo = tgv_oracle(f64(P), f64(w), float(np.float32(0.2)), a1, a0, eps)
    if vo == 0.0:
        assert float(v[0]) == 0.0 and torch.count_nonzero(gP) == 0
        return
    record_parity("tgv_value", abs(float(v[0]) - vo) / abs(vo), 1e-5)
    record_parity("tgv_grad_P", rel(gP.cpu().numpy(), gPo), 1e-5)
    record_parity("tgv_grad_w", rel(gw.cpu().numpy(), gwo), 1e-5)
    assert abs(float(v[0]) - vo) <= 1e-5 * abs(vo)
    assert rel(gP.cpu().numpy(), gPo) <= 1e-5 and rel(gw.cpu().numpy(), gwo) <= 1e-5


def test_step_with_tgv(ctx):
    """pa_step with lambda > 0: grad_p0 = data gradient + lambda dTGV/dP, loss[1] = data + lambda TGV."""
    grid = gen.make_grid((16, 14, 12), 0.2)
    acq = gen.make_acq(320, 0.2, t0=1.0)
    tmpl = gen.linear_array(8, 0.3)
    e = np.array([[0.05, -0.1, 0.02, 0.1, 0.2, -4.5], [-0.05, 0.08, 0.0, -0.3, 0.1, -4.8]])
    p_true = gen.random_volume(grid, 3)
    meas = oracle.forward(grid, acq, f64(tmpl), f64(gen.poses_from_euler(e)), f64(p_true))
    p0 = np.full(p_true.shape, 0.4)
    rng = np.random.default_rng(5)
    w = rng.normal(size=(3,) + p0.shape) * 0.1
    lam, a1, a0, eps = 0.3, 1.0, 2.0, 1e-3
    out = oracle.step(grid, acq, f64(tmpl), meas, p0, e, np.zeros(2 * p0.size), np.zeros(24), lr_p0=0.0,
                      lr_rot=0.0, lr_trans=0.0, update_p0=False, update_pose=False)
    vo, gPo, _ = tgv_oracle(p0, w, float(np.float32(0.2)), a1, a0, eps)
    nv = p0.size
    gbuf, loss = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    cfg = dict(lr_p0=1e-3, lr_rot=0.0, lr_trans=0.0, step=1, tgv_lambda=lam, tgv_alpha1=a1, tgv_alpha0=a0, tgv_eps=eps)
    wt = T(w)
    ctx.step(grid, acq, T(tmpl), T(meas), T(p0), T(e), torch.zeros(2 * nv, device="cuda"),
             torch.zeros(24, device="cuda"), gbuf, loss, cfg, tgv_w=wt, adam_w=torch.zeros(6 * nv, device="cuda"))
    torch.cuda.synchronize()
    want = out["grad_p0"] + lam * gPo.ravel()
    assert rel(gbuf.cpu().numpy(), want) <= 1e-4
    assert abs(float(loss[1]) - (out["loss"] + lam * vo)) <= 1e-4 * (out["loss"] + lam * vo)
    assert not torch.equal(wt, T(w))  # the auxiliary field was updated
