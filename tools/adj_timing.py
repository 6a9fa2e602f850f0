"""Diagnostic: adjoint(+pose) time inside pa_step vs. alone, vs. after a forward (C4 by default).
usage: python tools/adj_timing.py [config] [frames]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09643_b200 import Context, gen  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = gen.workload(cfgname, frames=frames)
ctx = Context(0)
T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")  # noqa: E731
p_true = T(gen.phantom(w))
tmpl = T(w.tmpl)
poses = T(w.poses_true())
meas = ctx.forward(w.grid, w.acq, tmpl, poses, p_true)
p = torch.full_like(p_true, 0.05)
cot = (ctx.forward(w.grid, w.acq, tmpl, poses, p) - meas) * 2.0
torch.cuda.synchronize()


def timed(fn, n=2):
    out = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return out


print("adjoint_pose alone ms:", timed(lambda: ctx.adjoint_pose(w.grid, w.acq, tmpl, poses, p, cot, want_elem=False)))
print("forward alone ms:", timed(lambda: ctx.forward(w.grid, w.acq, tmpl, poses, p)))
print("forward+adjoint_pose ms:", timed(lambda: (ctx.forward(w.grid, w.acq, tmpl, poses, p),
                                                 ctx.adjoint_pose(w.grid, w.acq, tmpl, poses, p, cot, want_elem=False))))
print("  last kernel ms (fwd, adj):", ctx.last_kernel_ms())
time.sleep(2.0)
print("adjoint_pose after 2 s idle ms:", timed(lambda: ctx.adjoint_pose(w.grid, w.acq, tmpl, poses, p, cot, want_elem=False), 1))
