"""Probe: do the forward (K1d) and the adjoint (K2a/K2c) gain from running concurrently on two streams?
usage: python tools/overlap_probe.py [config] [frames]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09643_b200 import Context, gen  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 16
w = gen.workload(cfgname, frames=frames)
c1, c2 = Context(0), Context(0)
T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")  # noqa: E731
p = T(gen.phantom(w))
tmpl, poses = T(w.tmpl), T(w.poses_true())
cot = c1.forward(w.grid, w.acq, tmpl, poses, p) * 1e-3
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()


def fwd(stream):
    c1.forward(w.grid, w.acq, tmpl, poses, p, stream=stream)


def adj(stream):
    c2.adjoint_pose(w.grid, w.acq, tmpl, poses, p, cot, want_elem=False, stream=stream)


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    fn()
    torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for rep in range(2):
    tf = timed(lambda: fwd(s1))
    ta = timed(lambda: adj(s2))
    tb = timed(lambda: (fwd(s1), adj(s2)))
    print(f"forward {tf:.1f} ms, adjoint {ta:.1f} ms, sum {tf + ta:.1f}, concurrent {tb:.1f} ms")
