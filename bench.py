#!/usr/bin/env python
"""Benchmark: one SfM iteration (pa_step = every §8(a) row) per step, frame-sharded over N GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c2|c1|c3_fine|c5] [--impl ours|reference]

Metric (BASELINE.json): forward+adjoint voxel·element·sample updates/s — the exact in-window
count of the operator for the forward pass plus the same count for the fused
adjoint+pose pass, per step, over all ranks, divided by the max-over-ranks device time.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "forward+adjoint voxel·element·sample updates/s; s per SfM iteration @1/2/4/8"
UNIT = "updates/s"
N_SM = 148
LANES = 128
# Roofline basis: ALGORITHMIC lane-ops per (voxel, element) pair of the kernel that runs, counted
# from its arithmetic (FP32 ops, packed ops as 2, MUFU, integer ops of the algorithm, loads / shared-memory
# atomics as 1; loop control, addressing and spills not counted), against 148 SM x 128 lanes x clock (the
# FP32-pipe peak = the issue peak of 4 warp-instr/clk/SM x 32 lanes).  Pairs = updates / W, W = 2 kappa sigma /
# (c dt) (in-window samples per pair).  The direct kernels (exp / power-law families, Gaussian fallback) walk the
# window: the survey's per-update basis x W.
OPS_PAIR = {
    "k_fwd_dep": 72.5,            # K1d at rank R = 5 (47.5 + 5 R in general, dep_ops below): geometry + window 31.5,
                                  # Horner channels 4 R + 10, R + 3 ATOMS (R + 2 words + count) + 3 address
    "k_adjoint_tay2_8": 76.25,    # K2c, 32-B records: geometry 25 + series & moments 36 + gradient 8.5 + reduction 6.75
    "k_adjoint_tay2_12": 88.25,   # K2c, 48-B records (short windows): synthetic division 27 instead of 15
    "k_adjoint_svd": 84.0,        # K2s: geometry 25 + rank-R basis evaluation 44 + gradient 8.5 + reduction 6.75
}
OPS_UPDATE_DIRECT = {"fwd": 4.5, "adj": 8.5}  # recurrence walk, FP32 lane-ops per in-window update
# kernel families (f3): the direct kernels and the pipe that bounds them
#   exp: E = min(A K_i, B/K_i) -> 2 FMUL + 1 MIN + D + FFMA (+0.5 setup) forward; adjoint + pose adds
#        g E, |D| and three sums (SE, SD, SX)
#   pow: MUFU-bound: lg2 + ex2 per update forward, + ex2(-lg2 x) for the pose sum; 16 XU lanes/SM
FAMILIES = {
    "gauss": dict(fwd=4.5, adj=8.5, lanes=LANES, unit="T lane-op/s", pipe="128 lanes (FP32 pipe = issue peak)"),
    "exp": dict(fwd=5.5, adj=9.5, lanes=LANES, unit="T lane-op/s", pipe="128 lanes (FP32 pipe = issue peak)"),
    "pow": dict(fwd=2.0, adj=3.0, lanes=16, unit="T MUFU-op/s", pipe="16 MUFU (XU) lanes"),
}


def describe(w):
    g, a = w.grid, w.acq
    k = a.get("kernel", "gauss")
    kern = {"gauss": "Gaussian kernel, sigma", "exp": "exponential kernel, s", "pow": f"power-law kernel nu={a.get('nu')}, s"}[k]
    return (f"{w.name}: {g['nx']}x{g['ny']}x{g['nz']} voxels @{g['pitch']} mm, {w.F} frames, {w.E}-element array, "
            f"{a['nt']} samples @40 MHz, {kern}={a['sigma']} mm, kappa={a['kappa']}, c=1.5 mm/us")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(w, p0, poses, rows=None, sub=128, frame=0):
    """The bounded oracle sample of a workload: frame `frame`, the first `rows` elements (default 4 x the host's
    cores, so the oracle's (frame, element)-parallel loops use every core), on the central sub^3 voxel
    sub-volume; forward + adjoint + element gradient (the GPU's two passes), exact in-window count n.
    Returns (run, n, description); run() executes the sample once."""
    import oracle

    oracle.build()
    cores = os.cpu_count() or 1
    rows = min(w.E, rows or 4 * cores)
    g = dict(w.grid)
    lo = [max(0, (g[k] - sub) // 2) for k in ("nx", "ny", "nz")]
    n3 = [min(sub, g[k]) for k in ("nx", "ny", "nz")]
    sg = dict(nx=n3[0], ny=n3[1], nz=n3[2], pitch=g["pitch"],
              origin=[g["origin"][i] + g["pitch"] * lo[i] for i in range(3)])
    sp = np.ascontiguousarray(p0[lo[2]:lo[2] + n3[2], lo[1]:lo[1] + n3[1], lo[0]:lo[0] + n3[0]])
    tm, pz = w.tmpl[:rows], poses[frame:frame + 1]
    n, _ = oracle.count(sg, w.acq, tm, pz)
    cot = np.random.default_rng(0).normal(size=(1, rows, w.acq["nt"]))

    def run():
        oracle.forward(sg, w.acq, tm, pz, sp)
        oracle.adjoint(sg, w.acq, tm, pz, cot)
        oracle.elem_grad(sg, w.acq, tm, pz, sp, cot)

    desc = (f"frame {frame}, elements 0..{rows - 1} of {w.E} ({rows} (frame, element) rows), central "
            f"{n3[0]}x{n3[1]}x{n3[2]} sub-volume: forward + adjoint + element gradient, {2 * n:.3e} counted updates")
    return run, n, desc


def cpu_oracle_sample(w, p0, poses):
    """cpu_baseline: the fp64 oracle (as it stands) on all host cores and on 1 thread, on a bounded sample of
    the workload (~10-20 s).  Returns the cpu_baseline dict."""
    import oracle

    cores = os.cpu_count() or 1
    run, n, desc = oracle_sample(w, p0, poses)
    oracle.set_threads(cores)
    t0 = time.perf_counter()
    run()
    dt = time.perf_counter() - t0
    # 1-thread rate on 1/cores of the rows (same per-row work)
    run1, n1, desc1 = oracle_sample(w, p0, poses, rows=max(1, 4))
    oracle.set_threads(1)
    t1 = time.perf_counter()
    run1()
    dt1 = time.perf_counter() - t1
    oracle.set_threads(cores)
    return {"value": 2.0 * n / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc + f" ({dt:.1f} s)",
            "single_thread": {"value": 2.0 * n1 / dt1, "unit": UNIT, "sample": desc1 + f" ({dt1:.1f} s)"},
            "cpu": cpu_model()}


def run_reference(args):
    """--impl reference: the fp64 oracle on all host cores, each step a bounded sample of the same workload
    (rank 0 only; the sample is sized to ~8 s so that --steps 20 --warmup 5 ends within a few minutes)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2604_09643_b200 import gen
    import oracle

    w = gen.workload(args.config)
    w.acq = gen.family_acq(w.acq, args.kernel, args.nu)
    p0 = gen.phantom(w)
    poses = w.poses_true()
    cores = os.cpu_count() or 1
    oracle.set_threads(cores)
    sub = 128
    run, n, desc = oracle_sample(w, p0, poses, sub=sub)
    t0 = time.perf_counter()
    run()
    if time.perf_counter() - t0 > 12.0:  # keep the whole run within minutes
        sub = 96
        run, n, desc = oracle_sample(w, p0, poses, sub=sub)
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    value = 2.0 * n / dt
    sample = desc + " per step"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": describe(w), "kernel": args.kernel, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--frames", type=int, default=None, help="override the frame count (debug)")
    ap.add_argument("--kernel", default="gauss", choices=sorted(FAMILIES),
                    help="kernel family of K (f3): gauss (the paper's, default), exp, pow")
    ap.add_argument("--nu", type=float, default=1.5, help="power-law exponent for --kernel pow")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2604_09643_b200 import Context, gen
    from paper_2604_09643_b200.dist import make_allreduce, shard_frames
    import __graft_entry__

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PA_BENCH_BACKEND=gloo: a functional check of the multi-rank path on a box with fewer GPUs than ranks (ranks
    # share devices, gloo carries the all-reduce; the timing of such a run is not a measurement)
    backend = os.environ.get("PA_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            torch.cuda.set_device(local % torch.cuda.device_count())
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    ctx = Context(dev.index)
    stream = torch.cuda.current_stream()

    # ---------------------------------------------------------------- workload (setup, untimed)
    w = gen.workload(args.config, frames=args.frames)
    w.acq = gen.family_acq(w.acq, args.kernel, args.nu)
    p_true = gen.phantom(w).astype(np.float32)
    T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device=dev)  # noqa: E731
    tmpl = T(w.tmpl)
    e_all = gen.perturb_euler(w.euler_true, 1.0, 0.5, seed=w.seed + 100)
    # frames by greedy longest-processing-time on the exact per-frame in-window counts of the initial poses
    # (every rank computes the same counts, so the partition needs no communication)
    _, per_frame = ctx.count(w.grid, w.acq, tmpl, T(gen.poses_from_euler(e_all)))
    frames = shard_frames(w.F, world, rank, cost=per_frame if world > 1 else None)
    Fl = len(frames)
    poses_true = T(w.poses_true()[frames])
    meas = ctx.forward(w.grid, w.acq, tmpl, poses_true, T(p_true))           # synthetic measurements
    e_init = e_all[frames]
    p_init = np.full(p_true.shape, 0.05, dtype=np.float32)
    nvox = p_true.size
    n_local = int(per_frame[frames].sum())                                   # exact in-window count
    cnt = torch.tensor([float(n_local)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(cnt)
    U = float(cnt.item())                                                    # updates per pass, all ranks
    radius = float(np.max(np.linalg.norm(w.tmpl, axis=1)))
    cfg = dict(lr_p0=1e-3, lr_trans=1e-2, lr_rot=1e-2 / max(radius, 1.0), beta1=0.9, beta2=0.999, eps=1e-8,
               step=1, loss_kind=0)
    ar = make_allreduce() if world > 1 else None

    p = T(p_init)
    eu = T(e_init)
    adam_p = torch.zeros(2 * nvox, device=dev)
    adam_q = torch.zeros(2 * 6 * Fl, device=dev)
    gbuf = torch.empty(nvox, device=dev)
    loss = torch.empty(2, device=dev)
    flush = torch.empty(64 * 1024 * 1024, device=dev)  # 256 MiB > 126 MB L2

    def one_step(s):
        cfg["step"] = s
        ctx.step(w.grid, w.acq, tmpl, meas, p, eu, adam_p, adam_q, gbuf, loss, cfg, allreduce=ar, stream=stream)

    for s in range(1, args.warmup + 1):
        one_step(s)
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- device-timed region
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    fwd_ms, adj_ms = [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n_launch0 = ctx.launch_count()
    with ClockSampler(dev.index) as clk:
        # the steps are enqueued back to back (pa_step does not synchronise the host), so host work between
        # steps never leaves the device idle inside a timed step; the pass times are read once at the end
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            one_step(args.warmup + 1 + i)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        fm, am = ctx.last_kernel_ms()  # forward / adjoint+pose pass of the last timed step (CUDA events)
        fwd_ms.append(fm)
        adj_ms.append(am)
    n_launch = ctx.launch_count() - n_launch0  # libpa kernels enqueued in the timed region
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / args.steps
    tmax = torch.tensor([ms, sum(fwd_ms) / len(fwd_ms), sum(adj_ms) / len(adj_ms)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms, fms, ams = (float(x) for x in tmax.tolist())
    value = 2.0 * U / (ms / 1e3)

    # ---------------------------------------------------------------- e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        meas_h = meas.cpu().pin_memory()
        p_h = p.cpu().pin_memory()
        e_h = eu.cpu().pin_memory()
        out_p = torch.empty_like(p_h).pin_memory()
        out_e = torch.empty_like(e_h).pin_memory()
        out_l = torch.empty(2).pin_memory()
        meas_d = torch.empty_like(meas)
        h2d = meas_h.numel() * 4 + p_h.numel() * 4 + e_h.numel() * 4
        d2h = out_p.numel() * 4 + out_e.numel() * 4 + out_l.numel() * 4
        k = 3  # >= 3 steps: the copies (~10 ms) resolve against seconds of compute
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(k):
            meas_d.copy_(meas_h, non_blocking=True)
            p.copy_(p_h, non_blocking=True)
            eu.copy_(e_h, non_blocking=True)
            cfg["step"] = args.warmup + args.steps + 1 + i
            ctx.step(w.grid, w.acq, tmpl, meas_d, p, eu, adam_p, adam_q, gbuf, loss, cfg, allreduce=ar, stream=stream)
            out_p.copy_(p, non_blocking=True)
            out_e.copy_(eu, non_blocking=True)
            out_l.copy_(loss, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([a.elapsed_time(b) / k], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": 2.0 * U / (float(e_ms.item()) / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(e_ms.item())}

    if rank != 0:
        dist.destroy_process_group()
        return
    clocks = clk.summary()
    # roofline of the dominant kernel: algorithmic lane-ops per pair (OPS_PAIR) x pairs / its live time, vs
    # 148 SM x 128 lanes x clock; the per-rank share of the work (frames are LPT-balanced)
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        peaks = json.load(fh)
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    f_meas = clocks["sm_mhz"] * 1e6 if clocks.get("sm_mhz") else None
    fam = FAMILIES[args.kernel]
    from paper_2604_09643_b200 import build as pa_build
    from paper_2604_09643_b200._pa import plan_info
    plan = plan_info(w.grid, w.acq, w.E)  # host-only: the kernels this geometry runs
    W = 2.0 * w.acq["kappa"] * w.acq["sigma"] / (w.acq["c"] * w.acq["dt"])  # in-window samples per pair
    U_rank = float(n_local)  # updates per pass on this rank (rank 0 prints; LPT keeps ranks within a frame)
    if plan["fwd_deposit"]:
        fwd_name = f"k_fwd_dep (K1d, deposit-form forward + fused loss/cotangent, rank {plan['dep_rank']})"
        fwd_ops = (47.5 + 5.0 * plan["dep_rank"]) / W
    else:
        fwd_name, fwd_ops = "k_forward (K1, direct forward + fused loss/cotangent)", fam["fwd"]
    if plan["adj_kernel"] == 2:
        adj_name, adj_ops = "k_adj_svd_filter + k_adjoint_svd (K2s, rank-R-basis adjoint + pose gradient)", OPS_PAIR["k_adjoint_svd"] / W
    elif plan["adj_kernel"] == 1:
        nf = 8 if plan["tay_order"] == 5 else 12
        adj_name = f"k_adj_filter + k_adjoint_tay2 (K2a/K2c, moment-filter adjoint + pose gradient, {4 * nf}-B records)"
        adj_ops = OPS_PAIR[f"k_adjoint_tay2_{nf}"] / W
    else:
        adj_name, adj_ops = "k_adjoint (K2, direct adjoint + pose gradient)", fam["adj"]
    lanes = fam["lanes"] if not (plan["fwd_deposit"] or plan["adj_kernel"]) else LANES
    peak = N_SM * lanes * f_max / 1e12

    def kinfo(name, ops, ms_):
        ach = U_rank * ops / (ms_ / 1e3) / 1e12 if ms_ > 0 else None
        return {"kernel": name, "achieved": ach, "frac": ach / peak if ach else None, "ops_per_update": ops,
                "ops_per_pair": ops * W, "ms_per_step": ms_,
                "frac_at_measured_clock": (ach * 1e12 / (N_SM * lanes * f_meas)) if (ach and f_meas) else None}

    k_fwd, k_adj = kinfo(fwd_name, fwd_ops, fms), kinfo(adj_name, adj_ops, ams)
    dom, other = (k_fwd, k_adj) if fms >= ams else (k_adj, k_fwd)
    # hardware-side check of the same kernels: warp instructions per update from an ncu capture of THIS build
    # (profiles/*_issue_c4.json stamped with libpa's source hash; a capture of another build is refused)
    issue, issue_note = None, None
    src_hash = pa_build.source_hash()
    caps = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_issue_c4.json"))
    for fname in reversed(caps):
        try:
            with open(os.path.join(ROOT, "profiles", fname)) as fh:
                iss = json.load(fh)
        except (OSError, ValueError):
            continue
        if iss.get("libpa_hash") != src_hash:
            issue_note = f"no ncu capture of this build (libpa {src_hash}); latest {fname} is of {iss.get('libpa_hash')}"
            continue
        if args.config == "c4" and args.kernel == "gauss":
            ipk = N_SM * 4 * f_max / 1e12
            issue = {"unit": "T warp-instr/s", "peak": ipk, "source": f"profiles/{fname} (libpa {src_hash})"}
            for key, kk in (("forward", k_fwd), ("adjoint", k_adj)):
                ipu = iss[key]["warp_inst_per_update"]
                ach = U_rank * ipu / (kk["ms_per_step"] / 1e3) / 1e12
                issue[key] = {"achieved": ach, "frac": ach / ipk, "warp_inst_per_update": ipu,
                              "lane_instr_per_pair": 32 * ipu * W}
            issue["frac"] = issue["adjoint" if dom is k_adj else "forward"]["frac"]
            issue_note = None
        break
    # measured DRAM bytes per launch (ncu launch list of the default C4 command, same build)
    traffic, traffic_note = None, None
    for fname in sorted((f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_traffic_c4.json")),
                        reverse=True):
        try:
            with open(os.path.join(ROOT, "profiles", fname)) as fh:
                tr = json.load(fh)
        except (OSError, ValueError):
            continue
        if tr.get("libpa_hash") == src_hash and args.config == "c4" and args.kernel == "gauss" and world == 1:
            t = tr["forward" if dom is k_fwd else "adjoint"]
            traffic = t["dram_read_bytes"] + t["dram_write_bytes"]
            traffic_note = tr.get("note")
        break
    roofline = {"bound": "alu", "kernel": dom["kernel"], "achieved": dom["achieved"], "peak": peak,
                "unit": fam["unit"] if lanes != LANES else "T lane-op/s", "frac": dom["frac"], "traffic": traffic,
                "traffic_unit": "bytes/launch",
                "peak_basis": f"148 SM x {lanes} lanes x sm_max {f_max / 1e6:.0f} MHz (MEASURED_PEAKS.json): the FP32-pipe "
                              f"peak = the issue peak (4 warp-instr/clk/SM x 32 lanes)",
                "ops_basis": "algorithmic lane-ops per (voxel, element) pair of the running kernel (DESIGN.md §7) / "
                             f"W = {W:.2f} in-window samples per pair",
                "ops_per_update": dom["ops_per_update"], "ops_per_pair": dom["ops_per_pair"],
                "kernel_ms_per_step": dom["ms_per_step"],
                "kernel_share_of_step": dom["ms_per_step"] / ms if ms > 0 else None,
                "frac_at_measured_clock": dom["frac_at_measured_clock"], "other_kernel": other,
                "step_frac": (U_rank * (fwd_ops + adj_ops) / (ms / 1e3) / 1e12) / peak if ms > 0 else None,
                "traffic_note": traffic_note, "issue": issue, "issue_note": issue_note,
                "dense_equivalent": {"value": value * w.acq["nt"] / W, "unit": "voxel·element·sample terms/s",
                                     "note": f"secondary figure: the same work counted on all N_t = {w.acq['nt']} samples "
                                             f"per pair, the paper's O(N_s N_d N_t) framing (P:347) = value x N_t / W"}}
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(w, p_true.astype(np.float64), w.poses_true())
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "s_per_iteration": ms / 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded vascular phantom, freehand sweep; meas = forward at true poses)",
        "config": {"workload": describe(w), "kernel": args.kernel, "frames_per_rank": Fl, "updates_per_pass": U,
                   "parallelism": f"frame-sharded x{world} (LPT on exact per-frame counts), "
                                  f"{'NCCL' if backend == 'nccl' or world == 1 else backend + ' (functional check)'} all-reduce of dL/dp0",
                   "plan": {k: plan[k] for k in ("lmin", "fwd_deposit", "dep_rank", "adj_kernel", "tay_order")},
                   "libpa_hash": src_hash,
                   "l2": "inputs larger than L2 (meas + cotangent per step) and a 256 MiB L2 flush before every timed step"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
        "gpu_launches": n_launch,
        "loss": float(loss[0].item()),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
