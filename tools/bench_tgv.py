"""HBM roofline of the TGV^2 kernel (f4): 256^3 volume (C4 grid), value + gradients per launch.
Algorithmic bytes per voxel: read P (4) + w (12), write dP (4) + dw (12) = 32 B.  One JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09643_b200 import Context, gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = Context(0)
grid = gen.make_grid((n, n, n), 0.2)
P = torch.rand((n, n, n), device="cuda")
w = torch.randn((3, n, n, n), device="cuda") * 0.1
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(3):
    ctx.tgv(grid, P, w)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.tgv(grid, P, w)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
gbs = 32.0 * n ** 3 / (ms / 1e3) / 1e9
print(json.dumps({"kernel": "k_tgv (+k_sum_parts)", "grid": f"{n}^3", "ms": ms, "bound": "hbm", "achieved": gbs,
                  "peak": peak, "unit": "GB/s", "frac": gbs / peak, "bytes_per_voxel": 32,
                  "note": "L2 flushed (256 MiB write) before every launch; median of %d" % reps}))
