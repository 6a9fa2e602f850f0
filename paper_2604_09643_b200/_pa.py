"""Thin ctypes binding of libpa (include/pa.h) — argument marshalling only.

Every step of the operator runs in libpa's CUDA kernels; torch is used for device memory,
streams and (in dist.py) the NCCL process group.  There is no CPU fallback: if libpa.so is
missing or no CUDA device is present, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PA_LIB_PATH", os.path.join(_HERE, "libpa.so"))

PA_OK, PA_EINVAL, PA_ESHAPE, PA_EDEGENERATE, PA_ECUDA, PA_ENOMEM, PA_EUNSUPPORTED = range(7)
_NAMES = {1: "PA_EINVAL", 2: "PA_ESHAPE", 3: "PA_EDEGENERATE", 4: "PA_ECUDA", 5: "PA_ENOMEM", 6: "PA_EUNSUPPORTED"}
EXPORTS = ("pa_create", "pa_destroy", "pa_last_error", "pa_version", "pa_forward", "pa_adjoint", "pa_pose_grad",
           "pa_adjoint_pose", "pa_count", "pa_loss", "pa_tgv", "pa_step", "pa_last_kernel_ms", "pa_launch_count",
           "pa_get_plan_info", "pa_ctx_plan_info", "pa_set_policy", "pa_step_status")

# kernel-selection policy bits of a context (pa_set_policy, include/pa.h)
POLICY = {"default": 0, "fwd_direct": 1, "adj_direct": 2, "adj_svd": 4, "adj_taylor": 8}


class PlanInfo(ctypes.Structure):
    """pa_plan_info (include/pa.h): the kernels the library runs for a geometry."""
    _fields_ = [("lmin", ctypes.c_int32), ("fwd_deposit", ctypes.c_int32), ("dep_rank", ctypes.c_int32),
                ("dep_warps", ctypes.c_int32), ("dep_err", ctypes.c_double), ("adj_taylor", ctypes.c_int32),
                ("tay_order", ctypes.c_int32), ("tay_err", ctypes.c_double), ("adj_svd", ctypes.c_int32),
                ("svd_derr", ctypes.c_double), ("dep_groups", ctypes.c_int32), ("dep_ring", ctypes.c_int32),
                ("adj_kernel", ctypes.c_int32), ("direct_class", ctypes.c_int32),
                ("dep_round", ctypes.c_int32), ("generic", ctypes.c_int32)]


def plan_info(grid, acq, E: int) -> dict:
    """pa_get_plan_info: host-only (no GPU needed)."""
    out = PlanInfo()
    _check(load().pa_get_plan_info(ctypes.byref(make_grid(grid)), ctypes.byref(make_acq(acq)), int(E), ctypes.byref(out)))
    return {k: getattr(out, k) for k, _ in PlanInfo._fields_}


class PAError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_NAMES.get(status, status)}: {msg}")
        self.status = status


class Grid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("origin", ctypes.c_float * 3), ("pitch", ctypes.c_float)]


class Acq(ctypes.Structure):
    _fields_ = [("c", ctypes.c_float), ("t0", ctypes.c_float), ("dt", ctypes.c_float), ("nt", ctypes.c_int32),
                ("sigma", ctypes.c_float), ("kappa", ctypes.c_float), ("kernel", ctypes.c_int32),
                ("nu", ctypes.c_float)]


# pa_kernel: families of the designated kernel K (reading R23)
KERNELS = {"gauss": 0, "exp": 1, "pow": 2}


class StepCfg(ctypes.Structure):
    _fields_ = [("lr_p0", ctypes.c_float), ("lr_rot", ctypes.c_float), ("lr_trans", ctypes.c_float),
                ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float),
                ("step", ctypes.c_int32), ("loss_kind", ctypes.c_int32), ("update_p0", ctypes.c_int32),
                ("update_pose", ctypes.c_int32), ("tgv_lambda", ctypes.c_float), ("tgv_alpha1", ctypes.c_float),
                ("tgv_alpha0", ctypes.c_float), ("tgv_eps", ctypes.c_float)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpa.so (raises if it is missing — no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(f"libpa.so not built at {path}; run __graft_entry__.build()")
            lib = ctypes.CDLL(path)
            vp, i32, st = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int
            lib.pa_last_error.restype = ctypes.c_char_p
            lib.pa_version.restype = ctypes.c_char_p
            for name in EXPORTS:
                if name not in ("pa_last_error", "pa_version", "pa_destroy", "pa_launch_count"):
                    getattr(lib, name).restype = st
            lib.pa_launch_count.restype = ctypes.c_longlong
            lib.pa_launch_count.argtypes = []
            lib.pa_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
            lib.pa_destroy.argtypes = [vp]
            lib.pa_destroy.restype = None
            g, a = ctypes.POINTER(Grid), ctypes.POINTER(Acq)
            lib.pa_forward.argtypes = [vp, g, a, vp, i32, vp, i32, vp, vp, vp]
            lib.pa_adjoint.argtypes = [vp, g, a, vp, i32, vp, i32, vp, vp, vp]
            lib.pa_pose_grad.argtypes = [vp, g, a, vp, i32, vp, i32, vp, vp, vp, vp, vp]
            lib.pa_adjoint_pose.argtypes = [vp, g, a, vp, i32, vp, i32, vp, vp, vp, vp, vp, vp]
            lib.pa_count.argtypes = [vp, g, a, vp, i32, vp, i32, ctypes.POINTER(ctypes.c_int64), vp, vp]
            lib.pa_loss.argtypes = [vp, i32, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp]
            lib.pa_step.argtypes = [vp, g, a, vp, i32, i32, vp, vp, vp, vp, vp, vp, ctypes.POINTER(StepCfg),
                                    ALLREDUCE_FN, vp, vp, vp, vp, vp, vp, vp, vp]
            lib.pa_tgv.argtypes = [vp, g, vp, vp, ctypes.c_float, ctypes.c_float, ctypes.c_float, vp, vp, vp, vp]
            lib.pa_last_kernel_ms.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
            lib.pa_get_plan_info.argtypes = [g, a, i32, ctypes.POINTER(PlanInfo)]
            lib.pa_ctx_plan_info.argtypes = [vp, g, a, i32, ctypes.POINTER(PlanInfo)]
            lib.pa_set_policy.argtypes = [vp, i32]
            lib.pa_step_status.argtypes = [vp]
            _lib = lib
    return _lib


def _check(status: int):
    if status != PA_OK:
        raise PAError(status, load().pa_last_error().decode())


def make_grid(grid: dict) -> Grid:
    g = Grid()
    g.nx, g.ny, g.nz = int(grid["nx"]), int(grid["ny"]), int(grid["nz"])
    for i in range(3):
        g.origin[i] = float(grid["origin"][i])
    g.pitch = float(grid["pitch"])
    return g


def make_acq(acq: dict) -> Acq:
    a = Acq()
    a.c, a.t0, a.dt = float(acq["c"]), float(acq["t0"]), float(acq["dt"])
    a.nt = int(acq["nt"])
    a.sigma, a.kappa = float(acq["sigma"]), float(acq["kappa"])
    k = acq.get("kernel", "gauss")
    a.kernel = KERNELS[k] if isinstance(k, str) else int(k)
    a.nu = float(acq.get("nu", 0.0))
    return a


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libpa takes CUDA tensors")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _f32(t):
    if t.dtype != torch.float32:
        raise TypeError(f"expected float32, got {t.dtype}")
    return _ptr(t)


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_allreduce_callback(tensors, allreduce):
    """C callback for pa_step: maps the raw pointer libpa passes back to the torch tensor that
    owns it and calls `allreduce(tensor)` (in place, e.g. torch.distributed SUM) with libpa's
    stream made torch's current stream, so the collective is ordered after the kernels that
    produced the buffer and before the ones pa_step enqueues next (pa.h).  Non-zero return =
    failure (pa_step then returns PA_ECUDA)."""
    views = {t.data_ptr(): t for t in tensors}

    def _cb(buf, n, stream_ptr, user):
        try:
            t = views[buf]
            if t.numel() != n:
                return 2
            if t.is_cuda:
                ext = torch.cuda.ExternalStream(int(stream_ptr or 0), device=t.device) if stream_ptr else \
                    torch.cuda.default_stream(t.device)
                with torch.cuda.stream(ext):
                    allreduce(t)
            else:
                allreduce(t)
            return 0
        except Exception:  # noqa: BLE001 - reported through the status code
            return 1

    cb = ALLREDUCE_FN(_cb)
    cb._views = views  # keep the tensors alive with the callback
    return cb


class Context:
    """Owns a pa_ctx (libpa's internal workspace) for one device; use one per stream."""

    def __init__(self, device: int | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("libpa needs a CUDA device (no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.lib = load()
        h = ctypes.c_void_p()
        _check(self.lib.pa_create(ctypes.byref(h), self.device))
        self.h = h

    def set_policy(self, policy):
        """Kernel-selection policy of this context: an int of PA_POLICY_* bits or names from POLICY."""
        if isinstance(policy, str):
            policy = POLICY[policy]
        elif not isinstance(policy, int):
            policy = sum(POLICY[p] for p in policy)
        _check(self.lib.pa_set_policy(self.h, int(policy)))

    def plan_info(self, grid, acq, E: int) -> dict:
        """pa_ctx_plan_info: the kernels this context runs for a geometry (its policy applied)."""
        out = PlanInfo()
        _check(self.lib.pa_ctx_plan_info(self.h, ctypes.byref(make_grid(grid)), ctypes.byref(make_acq(acq)), int(E),
                                         ctypes.byref(out)))
        return {k: getattr(out, k) for k, _ in PlanInfo._fields_}

    def step_status(self):
        """pa_step_status: raises PAError(PA_EDEGENERATE) if the last step's geometry was degenerate."""
        _check(self.lib.pa_step_status(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.pa_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- operator
    def forward(self, grid, acq, tmpl, poses, p0, out=None, stream=None):
        F, E = poses.shape[0], tmpl.shape[0]
        if out is None:
            out = torch.empty((F, E, int(acq["nt"])), device=p0.device, dtype=torch.float32)
        _check(self.lib.pa_forward(self.h, ctypes.byref(make_grid(grid)), ctypes.byref(make_acq(acq)), _f32(tmpl), E,
                                   _f32(poses), F, _f32(p0), _f32(out), _stream(stream)))
        return out

    def adjoint(self, grid, acq, tmpl, poses, cot, out=None, stream=None):
        F, E = poses.shape[0], tmpl.shape[0]
        if out is None:
            out = torch.empty((grid["nz"], grid["ny"], grid["nx"]), device=cot.device, dtype=torch.float32)
        _check(self.lib.pa_adjoint(self.h, ctypes.byref(make_grid(grid)), ctypes.byref(make_acq(acq)), _f32(tmpl), E,
                                   _f32(poses), F, _f32(cot), _f32(out), _stream(stream)))
        return out

    def pose_grad(self, grid, acq, tmpl, poses, p0, cot, want_elem=True, stream=None):
        F, E = poses.shape[0], tmpl.shape[0]
        gp = torch.empty((F, 12), device=cot.device, dtype=torch.float32)
        ge = torch.empty((F, E, 3), device=cot.device, dtype=torch.float32) if want_elem else None
        _check(self.lib.pa_pose_grad(self.h, ctypes.byref(make_grid(grid)), ctypes.byref(make_acq(acq)), _f32(tmpl), E,
                                     _f32(poses), F, _f32(p0), _f32(cot), _f32(gp), _ptr(ge), _stream(stream)))
        return gp, ge

    def adjoint_pose(self, grid, acq, tmpl, poses, p0, cot, want_elem=True, stream=None):
        F, E = poses.shape[0], tmpl.shape[0]
        gz = torch.empty((grid["nz"], grid["ny"], grid["nx"]), device=cot.device, dtype=torch.float32)
        gp = torch.empty((F, 12), device=cot.device, dtype=torch.float32)
        ge = torch.empty((F, E, 3), device=cot.device, dtype=torch.float32) if want_elem else None
        _check(self.lib.pa_adjoint_pose(self.h, ctypes.byref(make_grid(grid)), ctypes.byref(make_acq(acq)), _f32(tmpl),
                                        E, _f32(poses), F, _f32(p0), _f32(cot), _f32(gz), _f32(gp), _ptr(ge),
                                        _stream(stream)))
        return gz, gp, ge

    def count(self, grid, acq, tmpl, poses, stream=None):
        import numpy as np

        F, E = poses.shape[0], tmpl.shape[0]
        tot = ctypes.c_int64(0)
        pf = np.zeros(max(F, 1), dtype=np.int64)
        _check(self.lib.pa_count(self.h, ctypes.byref(make_grid(grid)), ctypes.byref(make_acq(acq)), _f32(tmpl), E,
                                 _f32(poses), F, ctypes.byref(tot), pf.ctypes.data_as(ctypes.c_void_p),
                                 _stream(stream)))
        return int(tot.value), pf[:F]

    def loss(self, kind, y, S, row_mask=None, cot=None, row_loss=False, stream=None):
        F, E, nt = y.shape
        if cot is None:
            cot = torch.empty_like(y)
        L = torch.empty(2, device=y.device, dtype=torch.float32)
        rl = torch.empty((F, E), device=y.device, dtype=torch.float32) if row_loss else None
        m = None
        if row_mask is not None:
            m = row_mask.to(torch.uint8).contiguous()
        _check(self.lib.pa_loss(self.h, int(kind), _f32(y), _f32(S), _ptr(m), F, E, nt, _f32(cot), _f32(L), _ptr(rl),
                                _stream(stream)))
        return (L[0], cot, rl) if row_loss else (L[0], cot)

    def tgv(self, grid, P, w, alpha1=1.0, alpha0=2.0, eps=1e-6, stream=None):
        """TGV^2 value and gradients (pa_tgv): returns (value tensor[1], grad_P, grad_w)."""
        val = torch.empty(1, device=P.device, dtype=torch.float32)
        gP = torch.empty_like(P)
        gw = torch.empty_like(w)
        _check(self.lib.pa_tgv(self.h, ctypes.byref(make_grid(grid)), _f32(P), _f32(w), float(alpha1), float(alpha0),
                               float(eps), _f32(val), _f32(gP), _f32(gw), _stream(stream)))
        return val, gP, gw

    def step(self, grid, acq, tmpl, meas, p0, euler_t, adam_p0, adam_pose, grad_p0, loss, cfg: dict, row_mask=None,
             allreduce=None, grad_euler=None, row_loss=None, tgv_w=None, adam_w=None, stream=None, check=False):
        """One SfM iteration (pa_step).  `allreduce(tensor)` (optional) sums a CUDA tensor in place across ranks;
        it is called for grad_p0 and for the global loss slot, on libpa's stream.  pa_step does not synchronise
        the host; check=True reads the step's degenerate-geometry verdict (pa_step_status) before returning."""
        F, E = euler_t.shape[0], tmpl.shape[0]
        c = StepCfg()
        c.lr_p0, c.lr_rot, c.lr_trans = float(cfg["lr_p0"]), float(cfg["lr_rot"]), float(cfg["lr_trans"])
        c.beta1, c.beta2, c.eps = float(cfg.get("beta1", 0.9)), float(cfg.get("beta2", 0.999)), float(cfg.get("eps", 1e-8))
        c.step = int(cfg["step"])
        c.loss_kind = int(cfg.get("loss_kind", 0))
        c.update_p0, c.update_pose = int(cfg.get("update_p0", 1)), int(cfg.get("update_pose", 1))
        c.tgv_lambda = float(cfg.get("tgv_lambda", 0.0))
        c.tgv_alpha1, c.tgv_alpha0 = float(cfg.get("tgv_alpha1", 1.0)), float(cfg.get("tgv_alpha0", 2.0))
        c.tgv_eps = float(cfg.get("tgv_eps", 1e-6))
        cb = ALLREDUCE_FN(0)
        if allreduce is not None:
            cb = make_allreduce_callback([grad_p0.view(-1), loss[1:2]], allreduce)
        m = None if row_mask is None else row_mask.to(torch.uint8).contiguous()
        _check(self.lib.pa_step(self.h, ctypes.byref(make_grid(grid)), ctypes.byref(make_acq(acq)), _f32(tmpl), E, F,
                                _f32(meas), _ptr(m), _f32(p0), _f32(euler_t), _f32(adam_p0), _f32(adam_pose),
                                ctypes.byref(c), cb, None, _f32(grad_p0), _f32(loss), _ptr(grad_euler),
                                _ptr(row_loss), _ptr(tgv_w), _ptr(adam_w), _stream(stream)))
        if check:
            self.step_status()
        return loss

    def launch_count(self):
        """Running count of kernels libpa enqueued from this thread (pa_launch_count)."""
        return int(self.lib.pa_launch_count())

    def last_kernel_ms(self):
        fw, ad = ctypes.c_float(0), ctypes.c_float(0)
        _check(self.lib.pa_last_kernel_ms(self.h, ctypes.byref(fw), ctypes.byref(ad)))
        return float(fw.value), float(ad.value)
