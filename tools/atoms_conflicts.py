"""Offline model of K1d's shared-memory deposit conflicts: for sampled (frame, element, tile
pair) of a workload, the 32 lanes of each deposit instruction -> window positions -> accumulator words -> banks.
Wavefronts per instruction: ADD (distinct values) = max lanes on one bank (same-address adds serialise);
INC (the count word, same-address lanes merged) = max distinct words on one bank.  Reproduces the ncu
numbers of the r2 build (ADD 2.71, POPC.INC 1.69 wavefronts per instruction at C4).
usage: python tools/atoms_conflicts.py [config] [samples] [map] [layout]
  map: pair (r2: 4 x-lanes x 4 z planes x 2 stacked tiles), ypair (4 y-lanes instead of x), best (the better
       of the two per (element, tile)), zcol (2 x-lanes x 16 z planes)
  layout: lin<k> (word = position x k, r2: k = 9), blk<pad> ([32-position block][channel][32 + pad])"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09643_b200 import gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 400
mp = sys.argv[3] if len(sys.argv) > 3 else "pair"
lay = sys.argv[4] if len(sys.argv) > 4 else "lin9"
w = gen.workload(cfg, frames=4)
g, a = w.grid, w.acq
h, c, ks = g["pitch"], a["c"], a["kappa"] * a["sigma"]
A = c * a["dt"]
poses = w.poses_true()
rng = np.random.default_rng(0)
NR = 512
lane = np.arange(32)
bx, bz, dzt, bl = 2 * (lane & 3), (lane >> 2) & 3, lane >> 4, lane & 3
MAPS = {
    "pair": [(bx + vx, 0 * lane + vy, bz + 4 * dzt) for vy in range(4) for vx in range(2)],
    "ypair": [(0 * lane + 2 * vy + vx, bl, bz + 4 * dzt) for vy in range(4) for vx in range(2)],
    "zcol": [(2 * (lane & 1) + vx, 0 * lane + vy, lane >> 1) for vy in range(4) for vx in range(2)],
}
cands = {"best": ["pair", "ypair"], "dir": ["dir"]}.get(mp, [mp])


def bank_of(pos):
    ring = pos & (NR - 1)
    if lay.startswith("blk"):
        pad = int(lay[3:])
        word = (ring >> 5) * (32 * 8 + pad) + (ring & 31)
    else:
        word = ring * int(lay[3:])
    return word, word % 32


add, inc, pick = [], [], {}
for _ in range(ns):
    f, e = rng.integers(w.F), rng.integers(w.E)
    R = poses[f, :9].reshape(3, 3)
    x = R @ w.tmpl[e] + poses[f, 9:]
    t = [rng.integers(0, g["nx"] // 8), rng.integers(0, g["ny"] // 8), rng.integers(0, g["nz"] // 8)]
    best = None
    for name in cands:
        aa, ii = [], []
        if name == "dir":  # the rule: lanes across x when the tile-centre direction leans more along x than y
            cx = g["origin"][0] + h * (8 * t[0] + 3.5) - x[0]
            cy = g["origin"][1] + h * (8 * t[1] + 3.5) - x[1]
            name = "pair" if 2.0 * abs(cx) >= abs(cy) else "ypair"
        for vx_, vy_, vz_ in MAPS[name]:
            X = g["origin"][0] + h * (8 * t[0] + vx_)
            Y = g["origin"][1] + h * (8 * t[1] + vy_)
            Z = g["origin"][2] + h * (8 * t[2] + vz_)
            r = np.sqrt((X - x[0]) ** 2 + (Y - x[1]) ** 2 + (Z - x[2]) ** 2)
            pos = np.ceil((r - c * a["t0"] - ks) / A).astype(np.int64)
            word, bank = bank_of(pos)
            aa.append(max(np.bincount(bank, minlength=32)))
            ii.append(max(len(set(word[bank == b])) for b in set(bank)))
        if best is None or sum(aa) < sum(best[0]):
            best = (aa, ii, name)
    add += best[0]
    inc += best[1]
    pick[best[2]] = pick.get(best[2], 0) + 1
print(f"{cfg} map={mp} layout={lay}: ADD {np.mean(add):.2f} wavefronts/instr, INC {np.mean(inc):.2f}  picks {pick}")
