"""A/B timing of the operator passes on the C4 geometry: python tools/ab_time.py [frames] [steps]
(run once per library variant: PA_LIB_PATH=variants/<name>/libpa.so).  Prints fwd / adj ms per step."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09643_b200 import Context, gen  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfgname = sys.argv[3] if len(sys.argv) > 3 else "c4"
w = gen.workload(cfgname, frames=frames)
ctx = Context(0)
if os.environ.get("AB_POLICY"):  # e.g. adj_taylor: the kernel-selection policy of the timed context
    ctx.set_policy(os.environ["AB_POLICY"].split(","))
T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")  # noqa: E731
tmpl = T(w.tmpl)
meas = ctx.forward(w.grid, w.acq, tmpl, T(w.poses_true()), T(gen.phantom(w)))
p = T(np.full((w.grid["nz"], w.grid["ny"], w.grid["nx"]), 0.05))
eu = T(gen.perturb_euler(w.euler_true, 1.0, 0.5, 7))
nv = p.numel()
am, aq = torch.zeros(2 * nv, device="cuda"), torch.zeros(12 * w.F, device="cuda")
g, L = torch.empty(nv, device="cuda"), torch.empty(2, device="cuda")
fw, ad = [], []
for s in range(1, steps + 2):
    ctx.step(w.grid, w.acq, tmpl, meas, p, eu, am, aq, g, L, dict(lr_p0=1e-3, lr_rot=1e-3, lr_trans=1e-2, step=s))
    torch.cuda.synchronize()
    if s > 1:
        a, b = ctx.last_kernel_ms()
        fw.append(a)
        ad.append(b)
print(json.dumps({"lib": os.environ.get("PA_LIB_PATH", "default"), "policy": os.environ.get("AB_POLICY", "default"),
                  "config": cfgname, "frames": frames,
                  "fwd_ms": float(np.median(fw)), "adj_ms": float(np.median(ad)), "loss": float(L[0])}))
