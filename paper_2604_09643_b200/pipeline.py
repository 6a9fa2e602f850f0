"""The PA-SFM stages after the reference map, chained (PAPER Alg. 1) — host code.

For frames with unknown poses (the paper's "Pose B"), given a reference map P_ref (Stage 1):

* Stage 2 — every element of every frame is localised independently: a coarse grid of
  candidate positions around the element's guessed position, ranked by the NC loss (Eq. 3) of the
  simulated single-element trace against the element's measured trace (one batched pa_forward + pa_loss),
  Top-K priors, then Adam on (x, y, z) through decreasing sigma (dynamic smoothing) — `localize`.
* Stage 3 — per frame, the modified RANSAC (pairwise-edge pre-check, then Kabsch) fits the
  rigid template to the localised elements: R_f, t_f and the inlier set I_f (`rigid.ransac_rigid`).
* Stage 4 — per frame, (theta, t) fine-tuned by pa_step with the NC loss masked to the
  inliers (Eq. 4: masked loss, gradients still move the whole rigid array), update_p0 = 0.
* Stage 5 — the joint reconstruction over known and calibrated frames (`driver.run_pyramid`).

Every operator evaluation runs in libpa (pa_forward / pa_loss / pa_step); this module only schedules.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import localize as loc
from . import rigid


@dataclass
class CalibResult:
    euler_t: np.ndarray                 # [F][6] calibrated poses (Stage 4)
    euler_ransac: np.ndarray            # [F][6] Stage 3 poses
    sensors: np.ndarray                 # [F][Es][3] Stage 2 localised elements (the selected ones)
    inliers: np.ndarray                 # [F][E] bool, Stage 3 inlier sets
    stage_s: dict = field(default_factory=dict)  # wall seconds per stage
    stage4_ms_per_iter: float = 0.0


def candidate_offsets(half: float, step: float) -> np.ndarray:
    g = np.arange(-half, half + 1e-9, step)
    return np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)


def localize_elements(ctx, grid, acqs, p_ref: torch.Tensor, S: torch.Tensor, guess: np.ndarray, offsets: np.ndarray,
                      topk=2, iters=30, lr=0.02, chunk=512):
    """Stage 2 for n sensors with individual search regions: S [n][nt] measured traces, guess [n][3].
    Candidates = guess + offsets; NC Top-K per sensor, then the batched Adam refinement through `acqs`
    (decreasing sigma).  Returns positions [n][3] and their final NC losses [n]."""
    dev = p_ref.device
    n, nt = S.shape
    C = offsets.shape[0]
    T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device=dev)  # noqa: E731
    tmpl0 = T(np.zeros((1, 3)))
    tops = np.zeros((n, topk, 3))
    for s0 in range(0, n, chunk):
        s1 = min(n, s0 + chunk)
        cand = (guess[s0:s1, None, :] + offsets[None, :, :]).reshape(-1, 3)           # [(s1-s0) C][3]
        y = ctx.forward(grid, acqs[0], tmpl0, T(loc._poses_for(cand)), p_ref)          # [(s1-s0) C][1][nt]
        Srep = S[s0:s1, None, None, :].expand(s1 - s0, C, 1, nt).reshape(-1, 1, nt).contiguous()
        _, _, rl = ctx.loss(1, y, Srep, row_loss=True)
        r = rl.view(s1 - s0, C).cpu().numpy().astype(np.float64)
        r = np.where(np.isfinite(r), r, np.inf)
        idx = np.argsort(r, axis=1)[:, :topk]
        tops[s0:s1] = cand.reshape(s1 - s0, C, 3)[np.arange(s1 - s0)[:, None], idx]
    ref, nc = loc.refine(ctx, grid, acqs, p_ref, S, tops, iters, lr)
    best = np.argmin(nc, axis=1)
    return ref[np.arange(n), best], nc[np.arange(n), best]


def calibrate_frames(ctx, grid, acqs, p_ref: torch.Tensor, meas: torch.Tensor, tmpl: np.ndarray,
                     euler_guess: np.ndarray, *, offsets=None, topk=2, loc_iters=30, loc_lr=0.02,
                     ransac_thr=0.15, edge_tol=0.2, ransac_iters=400, ft_iters=40, ft_lr=5e-3, seed=0, elems=None):
    """Stages 2-4 for F frames of E elements: meas [F][E][nt], initial guesses euler_guess [F][6].  `elems`
    (optional index array): the elements localised in Stage 2 (RANSAC needs only a few; the inlier set I of
    Stage 4 is then a subset of them), default all."""
    dev = p_ref.device
    F, E = euler_guess.shape[0], tmpl.shape[0]
    nt = meas.shape[2]
    T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device=dev)  # noqa: E731
    if offsets is None:
        offsets = candidate_offsets(1.0, 0.25)
    el = np.arange(E) if elems is None else np.asarray(elems)
    Es = len(el)
    st = {}
    # ---- Stage 2: every (selected) element localised independently
    t0 = time.perf_counter()
    guess = rigid.element_positions(euler_guess, tmpl[el]).reshape(F * Es, 3)
    S = meas[:, torch.as_tensor(el, device=dev)].reshape(F * Es, nt).contiguous()
    X, _ = localize_elements(ctx, grid, acqs, p_ref, S, guess, offsets, topk, loc_iters, loc_lr)
    X = X.reshape(F, Es, 3)
    torch.cuda.synchronize()
    st["stage2"] = time.perf_counter() - t0
    # ---- Stage 3: modified RANSAC (edge pre-check) + Kabsch per frame
    t0 = time.perf_counter()
    e3 = euler_guess.copy()
    inl = np.zeros((F, E), bool)
    for f in range(F):
        R, t, m = rigid.ransac_rigid(X[f], tmpl[el], ransac_thr, edge_tol, iters=ransac_iters, seed=seed + f)
        if R is not None:
            e3[f, :3] = rigid.R_to_euler(R)
            e3[f, 3:] = t
            inl[f, el] = m
        else:  # no consensus: keep the guess, the selected rows in the loss
            inl[f, el] = True
    st["stage3"] = time.perf_counter() - t0
    # ---- Stage 4: inlier-masked NC fine-tuning of (theta, t), rigid kinematics
    t0 = time.perf_counter()
    eu = T(e3)
    mask = torch.as_tensor(inl, device=dev).to(torch.uint8).contiguous()
    nv = p_ref.numel()
    p = p_ref.clone()
    dummy = torch.zeros(2 * nv, device=dev)
    g = torch.empty(nv, device=dev)
    loss = torch.empty(2, device=dev)
    radius = float(np.max(np.linalg.norm(tmpl, axis=1))) or 1.0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    n_it = 0
    for acq in acqs:
        adam_q = torch.zeros(12 * F, device=dev)
        for it in range(ft_iters):
            cfg = dict(lr_p0=0.0, lr_rot=ft_lr / radius, lr_trans=ft_lr, step=it + 1, loss_kind=1, update_p0=0,
                       update_pose=1)
            ctx.step(grid, acq, T(tmpl), meas, p, eu, dummy, adam_q, g, loss, cfg, row_mask=mask)
            n_it += 1
    ev1.record()
    torch.cuda.synchronize()
    ctx.step_status()
    st["stage4"] = time.perf_counter() - t0
    return CalibResult(euler_t=eu.cpu().numpy().astype(np.float64), euler_ransac=e3, sensors=X, inliers=inl,
                       stage_s=st, stage4_ms_per_iter=ev0.elapsed_time(ev1) / max(n_it, 1))
