"""Timing of a p0-only pa_step (update_pose = 0, no dL/dEuler: the adjoint without the pose moment) vs the joint
step on the C4 geometry: python tools/p0only_time.py [frames]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09643_b200 import Context, gen  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 16
w = gen.workload("c4", frames=frames)
ctx = Context(0)
T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")  # noqa: E731
tmpl = T(w.tmpl)
meas = ctx.forward(w.grid, w.acq, tmpl, T(w.poses_true()), T(gen.phantom(w)))
nv = w.grid["nx"] * w.grid["ny"] * w.grid["nz"]
out = {}
for name, up in (("joint", 1), ("p0_only", 0)):
    p = T(np.full((w.grid["nz"], w.grid["ny"], w.grid["nx"]), 0.05))
    eu = T(gen.perturb_euler(w.euler_true, 1.0, 0.5, 7))
    am, aq = torch.zeros(2 * nv, device="cuda"), torch.zeros(12 * w.F, device="cuda")
    g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
    ad = []
    for s in range(1, 5):
        ctx.step(w.grid, w.acq, tmpl, meas, p, eu, am, aq, g, L,
                 dict(lr_p0=1e-3, lr_rot=1e-3, lr_trans=1e-2, step=s, update_pose=up))
        torch.cuda.synchronize()
        if s > 1:
            ad.append(ctx.last_kernel_ms()[1])
    out[name] = float(np.median(ad))
print(json.dumps({"frames": frames, "adjoint_ms": out}))
