"""One pa_step on a workload (for ncu / compute-sanitizer captures): python tools/profile_step.py [config] [frames]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09643_b200 import Context, gen  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = gen.workload(cfgname, frames=frames)
ctx = Context(0)
T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")  # noqa: E731
p_true = gen.phantom(w)
tmpl = T(w.tmpl)
meas = ctx.forward(w.grid, w.acq, tmpl, T(w.poses_true()), T(p_true))
p = T(np.full(p_true.shape, 0.05))
eu = T(gen.perturb_euler(w.euler_true, 1.0, 0.5, 7))
nv = p.numel()
am, aq = torch.zeros(2 * nv, device="cuda"), torch.zeros(12 * w.F, device="cuda")
g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
for s in range(1, steps + 1):
    ctx.step(w.grid, w.acq, tmpl, meas, p, eu, am, aq, g, L, dict(lr_p0=1e-3, lr_rot=1e-3, lr_trans=1e-2, step=s))
    torch.cuda.synchronize()
    print("step", s, "loss", float(L[0]), "fwd/adj ms", ctx.last_kernel_ms())
