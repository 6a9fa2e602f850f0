"""Hardware-side counters of the two operator passes, stamped with libpa's source hash.

On the GPU box:  python tools/issue_capture.py run  [tag]
  runs `ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum` over
  tools/profile_step.py (C4 geometry, 16 frames, one pa_step) and writes gpurun_out/<tag>_issue_c4.csv;
then (here or there):  python tools/issue_capture.py parse gpurun_out/<tag>_issue_c4.csv <tag>
  writes profiles/<tag>_issue_c4.json: warp instructions each pass issues per in-window update (exact count of
  the captured step), with the libpa source hash; bench.py uses it only when the hash matches its own build.
"""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FRAMES = 16
METRICS = "smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum"


def run(tag):
    out = os.path.join(ROOT, "gpurun_out", f"{tag}_issue_c4.csv")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--csv", "--log-file", out, sys.executable,
           os.path.join(ROOT, "tools", "profile_step.py"), "c4", str(FRAMES), "1"]
    subprocess.check_call(cmd)
    print(out)


def parse(src, tag):
    import numpy as np
    import torch

    from paper_2604_09643_b200 import Context, build, gen, plan_info

    rows = list(csv.reader(open(src)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    iN, iV, iM = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    per = {}
    for r in rows[i + 1:]:
        name = re.sub(r"\(.*$", "", re.sub(r"^void\s+", "", r[iN]))
        per.setdefault((r[0], name), {})[r[iM]] = float(r[iV].replace(",", ""))
    # the step's launches: the forward (second k_fwd_dep: the first one makes the synthetic measurements)
    fwd = [v for (k, n), v in sorted(per.items(), key=lambda kv: int(kv[0][0])) if "k_fwd_dep" in n]
    adj = [v for (k, n), v in per.items() if "k_adjoint_tay2" in n or "k_adj_filter" in n or "k_adjoint_svd" in n
           or "k_adj_svd_filter" in n]
    w = gen.workload("c4", frames=FRAMES)
    # exact in-window updates of the step (same count on both passes)
    if torch.cuda.is_available():
        ctx = Context(0)
        T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda")  # noqa: E731
        eu = gen.perturb_euler(w.euler_true, 1.0, 0.5, 7)
        U, _ = ctx.count(w.grid, w.acq, T(w.tmpl), T(gen.poses_from_euler(eu)))
    else:
        import oracle

        U, _ = oracle.count(w.grid, w.acq, w.tmpl, gen.poses_from_euler(gen.perturb_euler(w.euler_true, 1.0, 0.5, 7)))
    fi = fwd[-1]["smsp__inst_executed.sum"]
    ai = sum(v["smsp__inst_executed.sum"] for v in adj)
    info = plan_info(w.grid, w.acq, w.E)
    out = {
        "note": "warp instructions each pass issues per in-window update (ncu smsp__inst_executed.sum over the pass's "
                "launches of one C4-geometry pa_step, 16 frames, / the step's exact update count); bench.py multiplies "
                "by its own updates and divides by the live pass time for roofline.issue (peak 148 SM x 4 warp-instr/clk "
                "x sm_max), and uses it only when libpa_hash matches its build",
        "libpa_hash": build.source_hash(),
        "updates": float(U),
        "plan": info,
        "forward": {"kernel": "k_fwd_dep (K1d)", "warp_inst": fi, "warp_inst_per_update": fi / U},
        "adjoint": {"kernel": "K2a + K2c (or K2s) over the step's frame chunks", "warp_inst": ai, "warp_inst_per_update": ai / U},
        "source": os.path.basename(src),
    }
    path = os.path.join(ROOT, "profiles", f"{tag}_issue_c4.json")
    json.dump(out, open(path, "w"), indent=1)
    print(path, json.dumps({k: out[k]["warp_inst_per_update"] for k in ("forward", "adjoint")}))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2] if len(sys.argv) > 2 else "r2")
    else:
        parse(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "r2")
