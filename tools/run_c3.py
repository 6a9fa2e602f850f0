"""BASELINE config 3 end to end: coarse-to-fine joint p0 + 6-DoF pose optimisation, 200 frames,
128^3 (sigma 0.4) -> 256^3 (sigma 0.2) pyramid, rigid-body outlier rejection.  Prints one JSON line.
  python tools/run_c3.py [--frames 200] [--iters 20 20]"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09643_b200 import Context, gen  # noqa: E402
from paper_2604_09643_b200.driver import Level, element_errors, run_pyramid  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=200)
ap.add_argument("--iters", type=int, nargs=2, default=[20, 20])
ap.add_argument("--glitch", type=float, default=0.1)
args = ap.parse_args()
import __graft_entry__  # noqa: E402

__graft_entry__.build()
ctx = Context(0)
wf = gen.workload("c3_fine", frames=args.frames)
wc = gen.workload("c3_coarse", frames=args.frames)
T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")  # noqa: E731
t0 = time.time()
p_true = gen.phantom(wf)
meas = ctx.forward(wf.grid, wf.acq, T(wf.tmpl), T(wf.poses_true()), T(p_true))
rng = np.random.default_rng(wf.seed + 7)
F = wf.F
e0 = gen.perturb_euler(wf.euler_true, 1.0, 0.5, seed=wf.seed + 9)
ng = int(round(args.glitch * F))
glitch = rng.choice(np.arange(2, F - 2), ng, replace=False)
e0[glitch, :3] += rng.choice([-1, 1], size=(ng, 3)) * math.radians(5.0)
e0[glitch, 3:] += rng.choice([-1, 1], size=(ng, 3)) * 3.0
err0 = element_errors(e0, wf.euler_true, wf.tmpl)
setup_s = time.time() - t0
res = run_pyramid(ctx, [Level(wc.grid, wc.acq, args.iters[0], lr_p0=2e-2, pose_warmup=5),
                        Level(wf.grid, wf.acq, args.iters[1], lr_p0=1e-2, pose_warmup=2)],
                  wf.tmpl, meas, e0, lr_trans=2e-2, check_every=5)
err1 = element_errors(res.euler_t, wf.euler_true, wf.tmpl)
flagged = sorted(set(i for ev in res.reinit_events for i in ev[2]))
print(json.dumps({
    "config": "c3: 128^3@0.4 (sigma 0.4) -> 256^3@0.2 (sigma 0.2), %d frames, 128-el linear, 2048 samples" % F,
    "s_per_iteration": {"coarse": res.ms_per_iter[0] / 1e3, "fine": res.ms_per_iter[1] / 1e3},
    "iters": args.iters, "setup_s": setup_s,
    "loss_first_last": {"coarse": [res.history[0][2], [h for h in res.history if h[0] == 0][-1][2]],
                        "fine": [[h for h in res.history if h[0] == 1][0][2], res.history[-1][2]]},
    "elem_err_mm": {"init_mean": float(err0.mean()), "init_glitch_mean": float(err0[glitch].mean()),
                    "final_mean": float(err1.mean()), "final_max": float(err1.max()),
                    "final_glitch_max": float(err1[glitch].max())},
    "glitch_frames": int(ng), "glitch_found": int(len(set(glitch.tolist()) & set(flagged))),
    "flagged": len(flagged)}))
