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
# Algorithmic FP32 lane-ops per in-window update: forward 4 + 0.5
# amortised setup; fused adjoint + pose 8 + 1 LDS (amortised setup included).
OPS_FWD = 4.5
OPS_ADJ = 8.5
N_SM = 148
LANES = 128
# kernel families (f3): algorithmic ops per in-window update and the pipe that bounds them.
#   exp: E = min(A K_i, B/K_i) -> 2 FMUL + 1 MIN + D + FFMA (+0.5 setup) forward; adjoint + pose adds
#        g E, |D| and three sums (SE, SD, SX)
#   pow: MUFU-bound: lg2 + ex2 per update forward, + ex2(-lg2 x) for the pose sum; 16 XU lanes/SM
FAMILIES = {
    "gauss": dict(fwd=OPS_FWD, adj=OPS_ADJ, lanes=LANES, unit="T FP32-lane-op/s", pipe="128 FP32 lanes"),
    "exp": dict(fwd=5.5, adj=9.5, lanes=LANES, unit="T FP32-lane-op/s", pipe="128 FP32 lanes"),
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


def cpu_oracle_sample(w, p0, poses, target_s=12.0):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload: frame 0, the first
    E_s elements: forward + adjoint + element gradient.  Returns (updates/s, cores, sample string)."""
    import oracle

    oracle.build()
    E_s = 1
    tmpl = w.tmpl
    cot = None
    # grow the element count until the sample is ~target_s of CPU work
    while True:
        t0 = time.perf_counter()
        sel = tmpl[:E_s]
        pz = poses[:1]
        y = oracle.forward(w.grid, w.acq, sel, pz, p0)
        cot = np.random.default_rng(0).normal(size=y.shape)
        oracle.adjoint(w.grid, w.acq, sel, pz, cot)
        oracle.elem_grad(w.grid, w.acq, sel, pz, p0, cot)
        dt = time.perf_counter() - t0
        n, _ = oracle.count(w.grid, w.acq, sel, pz)
        if dt * 2 > target_s or E_s * 2 > w.E:
            break
        E_s *= 2
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return 2.0 * n / dt, cores, f"frame 0, elements 0..{E_s - 1} of {w.E}: forward + adjoint + element gradient ({2 * n:.3e} updates, {dt:.1f} s)"


def run_reference(args):
    """--impl reference: the fp64 oracle on host cores, each step a bounded sample (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2604_09643_b200 import gen
    import oracle

    w = gen.workload(args.config)
    w.acq = gen.family_acq(w.acq, args.kernel, args.nu)
    p0 = gen.phantom(w)
    poses = w.poses_true()
    # size the per-step sample once (about 10-20 s of CPU work)
    E_s = 1
    while True:
        t0 = time.perf_counter()
        y = oracle.forward(w.grid, w.acq, w.tmpl[:E_s], poses[:1], p0)
        dt = time.perf_counter() - t0
        if dt * 3 * 2 > 15.0 or E_s * 2 > w.E:
            break
        E_s *= 2
    sel, pz = w.tmpl[:E_s], poses[:1]
    n, _ = oracle.count(w.grid, w.acq, sel, pz)
    cot = np.random.default_rng(0).normal(size=(1, E_s, w.acq["nt"]))

    def step():
        y = oracle.forward(w.grid, w.acq, sel, pz, p0)
        oracle.adjoint(w.grid, w.acq, sel, pz, cot)
        oracle.elem_grad(w.grid, w.acq, sel, pz, p0, cot)
        return y

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    value = 2.0 * n / dt
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    sample = f"frame 0, elements 0..{E_s - 1} of {w.E}: forward + adjoint + element gradient per step"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": describe(w), "kernel": args.kernel, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
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
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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
    frames = shard_frames(w.F, world, rank)
    Fl = len(frames)
    T = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device=dev)  # noqa: E731
    tmpl = T(w.tmpl)
    poses_true = T(w.poses_true()[frames])
    meas = ctx.forward(w.grid, w.acq, tmpl, poses_true, T(p_true))           # synthetic measurements
    e_init = gen.perturb_euler(w.euler_true, 1.0, 0.5, seed=w.seed + 100)[frames]
    p_init = np.full(p_true.shape, 0.05, dtype=np.float32)
    nvox = p_true.size
    n_local, _ = ctx.count(w.grid, w.acq, tmpl, poses_true)                 # exact in-window count
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
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            one_step(args.warmup + 1 + i)
            ev[i][1].record(stream)
            fm, am = ctx.last_kernel_ms()
            fwd_ms.append(fm)
            adj_ms.append(am)
        torch.cuda.synchronize()
    n_launch = ctx.launch_count() - n_launch0  # libpa kernels enqueued in the timed region
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / args.steps
    tmax = torch.tensor([ms, sum(fwd_ms) / args.steps, sum(adj_ms) / args.steps], device=dev, dtype=torch.float64)
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
        k = 1
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
    # roofline of the dominant kernel (adjoint+pose): FP32 lane-ops / s vs 148 SM x 128 lanes x clock
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        peaks = json.load(fh)
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    fam = FAMILIES[args.kernel]
    ops_fwd, ops_adj, lanes = fam["fwd"], fam["adj"], fam["lanes"]
    peak = N_SM * lanes * f_max / 1e12
    U_local_max = U / world  # frames are balanced; per-GPU roofline uses the per-rank share
    adj_achieved = U_local_max * ops_adj / (ams / 1e3) / 1e12 if ams > 0 else None
    fwd_achieved = U_local_max * ops_fwd / (fms / 1e3) / 1e12 if fms > 0 else None
    fwd_frac = fwd_achieved / peak if fwd_achieved else None
    adj_frac = adj_achieved / peak if adj_achieved else None
    f_meas = clocks["sm_mhz"] * 1e6 if clocks.get("sm_mhz") else None
    gauss = args.kernel == "gauss"
    # the kernels this geometry ran with (host-only plan query; env overrides included)
    from paper_2604_09643_b200._pa import plan_info
    plan = plan_info(w.grid, w.acq, w.E)
    fwd_name = ("k_fwd_dep (K1d, deposit-form forward + fused loss/cotangent)" if plan["fwd_deposit"]
                else "k_forward (K1, direct forward + fused loss/cotangent)")
    adj_name = ("k_adj_svd_filter + k_adjoint_svd (K2s, rank-R-basis adjoint + pose gradient)" if plan["adj_svd"]
                else "k_adj_filter + k_adjoint_tay2 (K2a/K2c, moment-filter adjoint + pose gradient)" if plan["adj_taylor"]
                else "k_adjoint (K2, direct adjoint + pose gradient)")
    k_fwd = {"kernel": fwd_name, "achieved": fwd_achieved, "frac": fwd_frac, "ops_per_update": ops_fwd, "ms_per_step": fms}
    k_adj = {"kernel": adj_name, "achieved": adj_achieved, "frac": adj_frac, "ops_per_update": ops_adj, "ms_per_step": ams}
    dom, other = (k_fwd, k_adj) if fms >= ams else (k_adj, k_fwd)
    # measured DRAM bytes per launch (ncu, default C4 command; profiles/r1_traffic_c4.json) — only for
    # the workload it was measured on
    traffic, traffic_note = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic_c4.json")) as fh:
            tr = json.load(fh)
        if args.config == "c4" and gauss and Fl == 400:
            t = tr["forward" if dom is k_fwd else "adjoint"]
            traffic = t["dram_read_bytes"] + t["dram_write_bytes"]
            traffic_note = tr.get("note")
    except (OSError, KeyError, ValueError):
        traffic = None
    # hardware-side check of the same kernel: warp instructions it issues per in-window update (ncu
    # smsp__inst_executed.sum / exact updates of the captured launch, profiles/r1_issue_c4.json) x this
    # run's updates / its live kernel time, against the issue peak 148 SM x 4 warp-instr/clk x sm_max
    issue = None
    try:
        with open(os.path.join(ROOT, "profiles", "r1_issue_c4.json")) as fh:
            iss = json.load(fh)
        if args.config == "c4" and gauss:
            key = "forward" if dom is k_fwd else "adjoint"
            ipu = iss[key]["warp_inst_per_update"]
            t_s = dom["ms_per_step"] / 1e3
            ach = U_local_max * ipu / t_s / 1e12
            ipk = N_SM * 4 * f_max / 1e12
            issue = {"achieved": ach, "peak": ipk, "unit": "T warp-instr/s", "frac": ach / ipk,
                     "warp_inst_per_update": ipu, "source": iss[key]["source"]}
    except (OSError, KeyError, ValueError):
        issue = None
    roofline = {"bound": "alu", "kernel": dom["kernel"], "achieved": dom["achieved"], "peak": peak,
                "unit": fam["unit"], "frac": dom["frac"], "traffic": traffic, "traffic_unit": "bytes/launch",
                "peak_basis": f"148 SM x {fam['pipe']} x sm_max {f_max / 1e6:.0f} MHz (MEASURED_PEAKS.json)",
                "ops_per_update": dom["ops_per_update"], "kernel_ms_per_step": dom["ms_per_step"],
                "kernel_share_of_step": dom["ms_per_step"] / ms if ms > 0 else None,
                "frac_at_measured_clock": (dom["achieved"] * 1e12 / (N_SM * lanes * f_meas)) if (dom["achieved"] and f_meas) else None,
                "other_kernel": other,
                "step_frac": (U_local_max * (ops_fwd + ops_adj) / (ms / 1e3) / 1e12) / peak if ms > 0 else None,
                "traffic_note": traffic_note, "issue": issue}
    cpu = None
    if world == 1 and not args.no_cpu:
        v, cores, sample = cpu_oracle_sample(w, p_true.astype(np.float64), w.poses_true())
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "s_per_iteration": ms / 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded vascular phantom, freehand sweep; meas = forward at true poses)",
        "config": {"workload": describe(w), "kernel": args.kernel, "frames_per_rank": Fl, "updates_per_pass": U,
                   "parallelism": f"frame-sharded x{world}, NCCL all-reduce of dL/dp0",
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
