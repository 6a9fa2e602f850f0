"""Stage 2 single-sensor localisation end to end on the GPU: coarse NC grid search
+ Top-K + Adam refinement through decreasing sigma recovers sensor positions.  Qualitative (the
paper prints no localisation number usable as a pin, P:180 needs its phantom)."""
import numpy as np
import pytest
import torch

from paper_2604_09643_b200 import gen

pytestmark = pytest.mark.gpu


def test_localize_sensors():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    from paper_2604_09643_b200 import Context
    from paper_2604_09643_b200.localize import localize

    __graft_entry__.build()
    ctx = Context(0)
    grid = gen.make_grid((48, 48, 48), 0.2)
    acq_hi = gen.make_acq(600, 0.4, t0=1.0)
    acq_lo = gen.make_acq(600, 0.2, t0=1.0)
    p_ref = torch.tensor(gen.vascular_phantom(grid, seed=3).astype(np.float32), device="cuda")
    rng = np.random.default_rng(0)
    n = 6
    true = np.stack([rng.uniform(-3, 3, n), rng.uniform(-3, 3, n), np.full(n, grid["origin"][2] - 3.0)
                     + rng.uniform(-0.5, 0.5, n)], 1)
    P = np.zeros((n, 12))
    P[:, [0, 4, 8]] = 1.0
    P[:, 9:] = true
    T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")  # noqa: E731
    S = ctx.forward(grid, acq_lo, T(np.zeros((1, 3))), T(P), p_ref)[:, 0, :].contiguous()
    g1 = np.arange(-4.0, 4.01, 0.5)
    gz = grid["origin"][2] - 3.0 + np.arange(-1.0, 1.01, 0.5)
    cand = np.stack(np.meshgrid(g1, g1, gz, indexing="ij"), -1).reshape(-1, 3)
    est, nc = localize(ctx, grid, [acq_hi, acq_lo], p_ref, S, cand, topk=4, iters=40, lr=0.02)
    err = np.linalg.norm(est - true, axis=1)
    assert np.median(err) < 0.1, err
    assert (nc < -0.95).mean() >= 0.8, nc
