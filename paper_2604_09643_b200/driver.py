"""Thin coarse-to-fine SfM driver (Alg. 1 Stages 1/4/5) — host code.

Every iteration is one `pa_step` (forward + loss + adjoint + pose gradient + all-reduce + Adam,
all in libpa).  The driver only schedules:
  * the pyramid: levels of (grid, sigma) — coarse 128^3 @ 0.4 mm with sigma = 0.4 mm, then the
    full 256^3 @ 0.2 mm with sigma = 0.2 mm; with sigma = pitch the pyramid IS the paper's
    dynamic smoothing / sigma annealing (Alg. 1; R3);
    p0 is carried to the finer grid by trilinear interpolation (cell-centred grids);
  * a p0 warm-up with frozen poses (the reference-map stage) before joint updates;
  * every `check_every` iterations, the geometric-consistency / rigid-body outlier step on the
    host: frames whose pose leaves the smooth freehand trajectory, or whose loss is
    an outlier, are rigidly re-initialised from their neighbours (`rigid.py`), and their rows are
    masked (Eq. 4 inlier mask) for one check period.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as Fnn

from . import rigid


@dataclass
class Level:
    grid: dict
    acq: dict
    iters: int
    lr_p0: float = 1e-2
    pose_warmup: int = 5


@dataclass
class DriverResult:
    p0: torch.Tensor
    euler_t: np.ndarray
    history: list = field(default_factory=list)
    ms_per_iter: list = field(default_factory=list)
    reinit_events: list = field(default_factory=list)


def upsample(p: torch.Tensor, grid_to: dict) -> torch.Tensor:
    """Trilinear resampling of a cell-centred volume onto a finer cell-centred grid of the same
    extent (align_corners=False)."""
    out = Fnn.interpolate(p[None, None], size=(grid_to["nz"], grid_to["ny"], grid_to["nx"]), mode="trilinear",
                          align_corners=False)
    return out[0, 0].contiguous()


def run_pyramid(ctx, levels, tmpl: np.ndarray, meas: torch.Tensor, euler_init: np.ndarray, *, lr_trans=2e-2,
                check_every=10, p_init=0.05, allreduce=None, outlier_k=6.0, log=None, pose_loss="mse",
                p_start: torch.Tensor | None = None, pose_frames: np.ndarray | None = None) -> DriverResult:
    """pose_loss "mse": one pa_step per iteration updates p0 and the poses from the MSE cotangent (R12);
    "nc": the paper's split (P:85 MSE for P_c, P:92 / P:113 NC for the poses) — after the warm-up,
    iterations alternate a p0 step (MSE, poses frozen) and a pose step (NC, masked rows out of the loss,
    p0 frozen).  p_start: initial volume (e.g. Stage 1's reference map); pose_frames: bool [F], frames whose
    pose is optimised (the others, e.g. tracked "Pose A" frames, stay fixed)."""
    dev = meas.device
    T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device=dev)  # noqa: E731
    F, E = euler_init.shape[0], tmpl.shape[0]
    radius = float(np.max(np.linalg.norm(tmpl, axis=1))) or 1.0
    tm = T(tmpl)
    eu = T(euler_init)
    p = None
    res = DriverResult(p0=None, euler_t=None)
    loss = torch.empty(2, device=dev)
    rl = torch.empty((F, E), device=dev)
    mask = torch.ones((F, E), device=dev, dtype=torch.uint8)
    masked_until = np.full(F, -1)
    flagged_prev = np.zeros(F, bool)
    for li, L in enumerate(levels):
        g = L.grid
        if p is None:
            p = p_start.clone() if p_start is not None else torch.full((g["nz"], g["ny"], g["nx"]), p_init, device=dev)
            if p.shape != (g["nz"], g["ny"], g["nx"]):
                p = upsample(p, g)
        else:
            p = upsample(p, g)
        nv = p.numel()
        adam_p = torch.zeros(2 * nv, device=dev)
        adam_q = torch.zeros(12 * F, device=dev)
        gbuf = torch.empty(nv, device=dev)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot_ms = 0.0
        n_p = n_q = 0  # Adam step counters of p0 and of the poses
        frozen = None if pose_frames is None else torch.as_tensor(~np.asarray(pose_frames, bool), device=dev)
        for it in range(L.iters):
            pose_on = it >= L.pose_warmup
            if pose_loss == "nc" and pose_on and (it - L.pose_warmup) % 2 == 1:
                n_q += 1  # pose step: NC (Eq. 3/4), p0 frozen
                cfg = dict(lr_p0=0.0, lr_trans=lr_trans, lr_rot=lr_trans / radius, step=n_q, loss_kind=1,
                           update_p0=0, update_pose=1)
            elif pose_loss == "nc":
                n_p += 1  # p0 step: MSE (Eq. 2), poses frozen
                cfg = dict(lr_p0=L.lr_p0, lr_trans=0.0, lr_rot=0.0, step=n_p, loss_kind=0, update_p0=1, update_pose=0)
            else:
                n_p += 1
                cfg = dict(lr_p0=L.lr_p0, lr_trans=lr_trans, lr_rot=lr_trans / radius, step=n_p, loss_kind=0,
                           update_p0=1, update_pose=int(pose_on))
            e_keep = eu.clone() if (frozen is not None and cfg["update_pose"]) else None
            ev0.record()
            ctx.step(g, L.acq, tm, meas, p, eu, adam_p, adam_q, gbuf, loss, cfg, row_mask=mask, allreduce=allreduce,
                     row_loss=rl)
            if e_keep is not None:  # tracked frames keep their poses
                eu[frozen] = e_keep[frozen]
            ev1.record()
            torch.cuda.synchronize()
            tot_ms += ev0.elapsed_time(ev1)
            res.history.append((li, it, float(loss[1]), int(cfg["loss_kind"])))
            if log:
                log(li, it, float(loss[1]))
            if (it + 1) % check_every == 0 and it >= L.pose_warmup and cfg["loss_kind"] == 0:
                e = eu.cpu().numpy().astype(np.float64)
                bad = rigid.trajectory_outliers(e, tmpl, k=outlier_k)
                fl = rl.sum(1).cpu().numpy().astype(np.float64)
                med = np.median(fl)
                mad = np.median(np.abs(fl - med)) + 1e-30
                bad |= fl > med + outlier_k * 1.4826 * mad
                repeat = bad & flagged_prev
                flagged_prev = bad.copy()
                masked_until[repeat] = it + check_every  # inconsistent twice: out of the loss for a period
                bad &= ~repeat
                if frozen is not None:
                    bad &= np.asarray(pose_frames, bool)
                if bad.any():
                    e2 = rigid.reinit_from_neighbours(e, bad)
                    eu.copy_(T(e2))
                    aq = adam_q.view(2, F, 6)
                    aq[:, torch.as_tensor(np.nonzero(bad)[0], device=dev)] = 0.0
                    res.reinit_events.append((li, it, np.nonzero(bad)[0].tolist()))
            m = torch.as_tensor(masked_until < it + 1, device=dev)
            mask.copy_(m[:, None].to(torch.uint8).expand(F, E).contiguous())
        res.ms_per_iter.append(tot_ms / max(L.iters, 1))
    res.p0 = p
    res.euler_t = eu.cpu().numpy().astype(np.float64)
    return res


def element_errors(euler_est: np.ndarray, euler_true: np.ndarray, tmpl: np.ndarray) -> np.ndarray:
    """Per-frame mean element-position error (mm) — the observable part of the pose (a linear
    array's roll about its own axis is not observable, R15)."""
    a = rigid.element_positions(euler_est, tmpl)
    b = rigid.element_positions(euler_true, tmpl)
    return np.linalg.norm(a - b, axis=2).mean(1)


def pose_errors(euler_est: np.ndarray, euler_true: np.ndarray):
    """Per-frame rotation error (deg) and translation error (mm)."""
    rot = np.array([np.degrees(rigid.rot_angle(rigid.euler_to_R(a[:3]), rigid.euler_to_R(b[:3])))
                    for a, b in zip(euler_est, euler_true)])
    tr = np.linalg.norm(euler_est[:, 3:] - euler_true[:, 3:], axis=1)
    return rot, tr
