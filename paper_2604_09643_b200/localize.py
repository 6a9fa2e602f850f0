"""Stage 2 — differentiable single-sensor localisation (Alg. 1).

Thin host scheduling over libpa; the compute is the same operator in a new batch shape:
  * every (sensor, candidate position) pair is one "frame" with a single element at the template
    origin and pose t = candidate, so one `pa_forward` evaluates all candidate traces at once;
  * global coarse search: NC loss (Eq. 3) of each candidate trace against the sensor's
    measured trace (`pa_loss`, per-row losses), Top-K per sensor;
  * gradient refinement of (x, y, z): `pa_step` with update_p0 = 0 on the Top-K
    candidates, NC loss, Adam on the translation only (the rotation of a point element is void);
  * dynamic smoothing (Alg. 1): the refinement runs through decreasing sigma.
Returns the refined position (best NC) per sensor.
"""
from __future__ import annotations

import numpy as np
import torch


def _poses_for(points: np.ndarray) -> np.ndarray:
    P = np.zeros((points.shape[0], 12))
    P[:, [0, 4, 8]] = 1.0
    P[:, 9:] = points
    return P


def coarse_search(ctx, grid, acq, p_ref: torch.Tensor, S: torch.Tensor, cand: np.ndarray, topk: int):
    """S [n][nt] measured traces, cand [C][3] candidate positions (shared by all sensors).
    Returns (best [n][topk][3] positions, nc [n][topk])."""
    dev = p_ref.device
    n, nt = S.shape
    C = cand.shape[0]
    T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device=dev)  # noqa: E731
    tmpl = T(np.zeros((1, 3)))
    poses = T(_poses_for(cand))
    y = ctx.forward(grid, acq, tmpl, poses, p_ref)                      # [C][1][nt]
    out_p = np.zeros((n, topk, 3))
    out_l = np.zeros((n, topk))
    for i in range(n):
        Srep = S[i].reshape(1, 1, nt).expand(C, 1, nt).contiguous()
        _, _, rl = ctx.loss(1, y, Srep, row_loss=True)
        r = rl.view(-1).cpu().numpy()
        r = np.where(np.isfinite(r), r, np.inf)
        idx = np.argpartition(r, topk - 1)[:topk]
        idx = idx[np.argsort(r[idx])]
        out_p[i] = cand[idx]
        out_l[i] = r[idx]
    return out_p, out_l


def refine(ctx, grid, acqs, p_ref: torch.Tensor, S: torch.Tensor, start: np.ndarray, iters: int, lr: float):
    """Adam on positions through decreasing-sigma `acqs`.  start [n][k][3].  Returns the refined
    positions [n][k][3] and their final NC losses [n][k]."""
    dev = p_ref.device
    n, k, _ = start.shape
    nt = S.shape[1]
    F = n * k
    T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device=dev)  # noqa: E731
    tmpl = T(np.zeros((1, 3)))
    e = np.zeros((F, 6))
    e[:, 3:] = start.reshape(F, 3)
    eu = T(e)
    meas = S.repeat_interleave(k, dim=0).reshape(F, 1, nt).contiguous()
    nv = p_ref.numel()
    dummy_adam = torch.zeros(2 * nv, device=dev)
    gbuf = torch.empty(nv, device=dev)
    loss = torch.empty(2, device=dev)
    rl = torch.empty((F, 1), device=dev)
    p = p_ref.clone()
    for acq in acqs:
        adam_q = torch.zeros(12 * F, device=dev)
        for it in range(iters):
            cfg = dict(lr_p0=0.0, lr_rot=0.0, lr_trans=lr, step=it + 1, loss_kind=1, update_p0=0, update_pose=1)
            ctx.step(grid, acq, tmpl, meas, p, eu, dummy_adam, adam_q, gbuf, loss, cfg, row_loss=rl)
    # final losses at the last sigma
    y = ctx.forward(grid, acqs[-1], tmpl, T(_poses_for(eu.cpu().numpy()[:, 3:].astype(np.float64))), p)
    _, _, rl = ctx.loss(1, y, meas, row_loss=True)
    return eu.cpu().numpy()[:, 3:].reshape(n, k, 3).astype(np.float64), rl.view(n, k).cpu().numpy()


def localize(ctx, grid, acqs, p_ref, S, cand, topk=4, iters=30, lr=0.02):
    """Coarse search at the largest sigma, then refinement through `acqs` (decreasing sigma).
    Returns best position [n][3] per sensor and its NC loss."""
    tops, _ = coarse_search(ctx, grid, acqs[0], p_ref, S, cand, topk)
    ref, nc = refine(ctx, grid, acqs, p_ref, S, tops, iters, lr)
    best = np.argmin(nc, axis=1)
    return ref[np.arange(len(best)), best], nc[np.arange(len(best)), best]
