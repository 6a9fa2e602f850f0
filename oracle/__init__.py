"""fp64 CPU oracle for the PA-SFM acoustic radiation operator — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path
(``paper_2604_09643_b200``) never imports it and shares no code with it.

The arithmetic lives in ``pa_oracle.c`` (plain C, fp64, OpenMP); this module only builds
and marshals.  Closed forms from the paper's appendix used as pins live in
``oracle/closed_forms.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pa_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile pa_oracle.c -> liboracle.so (gcc -O2, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _Grid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("origin", ctypes.c_double * 3), ("pitch", ctypes.c_double)]


class _Acq(ctypes.Structure):
    _fields_ = [("c", ctypes.c_double), ("t0", ctypes.c_double), ("dt", ctypes.c_double),
                ("nt", ctypes.c_int32), ("sigma", ctypes.c_double), ("kappa", ctypes.c_double),
                ("kernel", ctypes.c_int32), ("nu", ctypes.c_double)]


# kernel families of the designated kernel function K (R23)
KERNELS = {"gauss": 0, "exp": 1, "pow": 2}


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            _lib = ctypes.CDLL(_LIB)
            _lib.oracle_count.restype = ctypes.c_int64
            _lib.oracle_mse.restype = ctypes.c_double
            _lib.oracle_nc.restype = ctypes.c_double
            _lib.oracle_step.restype = ctypes.c_double
    return _lib


def _grid(grid) -> _Grid:
    g = _Grid()
    g.nx, g.ny, g.nz = int(grid["nx"]), int(grid["ny"]), int(grid["nz"])
    for i in range(3):
        g.origin[i] = float(grid["origin"][i])
    g.pitch = float(grid["pitch"])
    return g


def _acq(acq) -> _Acq:
    a = _Acq()
    a.c, a.t0, a.dt = float(acq["c"]), float(acq["t0"]), float(acq["dt"])
    a.nt = int(acq["nt"])
    a.sigma, a.kappa = float(acq["sigma"]), float(acq["kappa"])
    k = acq.get("kernel", "gauss")
    a.kernel = KERNELS[k] if isinstance(k, str) else int(k)
    a.nu = float(acq.get("nu", 0.0))
    return a


def _d(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _p(x):
    return x.ctypes.data_as(ctypes.c_void_p) if x is not None else None


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's loops (bench.py's cpu_baseline: the 1-thread and all-core rates)."""
    _load().oracle_set_threads(ctypes.c_int32(int(n)))


def threads() -> int:
    return int(_load().oracle_get_threads())


def place(tmpl, poses):
    tmpl, poses = _d(tmpl), _d(poses)
    E, F = tmpl.shape[0], poses.shape[0]
    out = np.zeros((F, E, 3))
    _load().oracle_place(_p(tmpl), ctypes.c_int32(E), _p(poses), ctypes.c_int32(F), _p(out))
    return out


def forward(grid, acq, tmpl, poses, p0):
    """traces[F][E][nt] (Eq. gpu_forward_model)."""
    tmpl, poses, p0 = _d(tmpl), _d(poses), _d(p0).reshape(-1)
    E, F = tmpl.shape[0], poses.shape[0]
    out = np.zeros((F, E, int(acq["nt"])))
    g, a = _grid(grid), _acq(acq)
    _load().oracle_forward(ctypes.byref(g), ctypes.byref(a), _p(tmpl), ctypes.c_int32(E), _p(poses),
                           ctypes.c_int32(F), _p(p0), _p(out))
    return out


def adjoint(grid, acq, tmpl, poses, cot):
    """grad_p0[nz][ny][nx] = A^T cot."""
    tmpl, poses, cot = _d(tmpl), _d(poses), _d(cot)
    E, F = tmpl.shape[0], poses.shape[0]
    out = np.zeros((int(grid["nz"]), int(grid["ny"]), int(grid["nx"])))
    g, a = _grid(grid), _acq(acq)
    _load().oracle_adjoint(ctypes.byref(g), ctypes.byref(a), _p(tmpl), ctypes.c_int32(E), _p(poses),
                           ctypes.c_int32(F), _p(cot), _p(out))
    return out


def adjoint_abs(grid, acq, tmpl, poses, cot):
    """Per-voxel error scale of the adjoint: sum of |terms| (test infrastructure; see pa_oracle.c)."""
    tmpl, poses, cot = _d(tmpl), _d(poses), _d(cot)
    E, F = tmpl.shape[0], poses.shape[0]
    out = np.zeros((int(grid["nz"]), int(grid["ny"]), int(grid["nx"])))
    g, a = _grid(grid), _acq(acq)
    _load().oracle_adjoint_abs(ctypes.byref(g), ctypes.byref(a), _p(tmpl), ctypes.c_int32(E), _p(poses),
                               ctypes.c_int32(F), _p(cot), _p(out))
    return out


def elem_grad(grid, acq, tmpl, poses, p0, cot):
    """dL/dx_fe [F][E][3]."""
    tmpl, poses, p0, cot = _d(tmpl), _d(poses), _d(p0).reshape(-1), _d(cot)
    E, F = tmpl.shape[0], poses.shape[0]
    out = np.zeros((F, E, 3))
    g, a = _grid(grid), _acq(acq)
    _load().oracle_elem_grad(ctypes.byref(g), ctypes.byref(a), _p(tmpl), ctypes.c_int32(E), _p(poses),
                             ctypes.c_int32(F), _p(p0), _p(cot), _p(out))
    return out


def pose_grad_from_elem(tmpl, grad_elem):
    """[F][12] = dL/dR (row-major), dL/dt."""
    tmpl, ge = _d(tmpl), _d(grad_elem)
    F, E = ge.shape[0], ge.shape[1]
    out = np.zeros((F, 12))
    _load().oracle_pose_grad_from_elem(_p(tmpl), ctypes.c_int32(E), ctypes.c_int32(F), _p(ge), _p(out))
    return out


def pose_grad(grid, acq, tmpl, poses, p0, cot):
    ge = elem_grad(grid, acq, tmpl, poses, p0, cot)
    return pose_grad_from_elem(tmpl, ge), ge


def count(grid, acq, tmpl, poses):
    """Exact in-window (voxel, element, sample) count; returns (total, per_frame)."""
    tmpl, poses = _d(tmpl), _d(poses)
    E, F = tmpl.shape[0], poses.shape[0]
    pf = np.zeros(F, dtype=np.int64)
    g, a = _grid(grid), _acq(acq)
    tot = _load().oracle_count(ctypes.byref(g), ctypes.byref(a), _p(tmpl), ctypes.c_int32(E), _p(poses),
                               ctypes.c_int32(F), pf.ctypes.data_as(ctypes.c_void_p))
    return int(tot), pf


def mse(y, S):
    y, S = _d(y), _d(S)
    cot = np.zeros_like(y)
    L = _load().oracle_mse(_p(y), _p(S), ctypes.c_int64(y.size), _p(cot))
    return L, cot


def nc(y, S, mask=None):
    """Rows along the last axis; mask (nullable) per row."""
    y, S = _d(y), _d(S)
    n = y.shape[-1]
    rows = y.size // n
    cot = np.zeros_like(y)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
    L = _load().oracle_nc(_p(y), _p(S), ctypes.c_int64(rows), ctypes.c_int32(n), _p(m), _p(cot))
    return L, cot


def adam(x, m, v, grad, lr, b1=0.9, b2=0.999, eps=1e-8, t=1, clamp=None):
    x, m, v, grad = _d(x).copy(), _d(m).copy(), _d(v).copy(), _d(grad)
    lr_vec = None
    lr_s = 0.0
    if np.ndim(lr) == 0:
        lr_s = float(lr)
    else:
        lr_vec = _d(np.broadcast_to(lr, x.shape))
    _load().oracle_adam(_p(x), _p(m), _p(v), _p(grad), ctypes.c_int64(x.size), ctypes.c_double(lr_s), _p(lr_vec),
                        ctypes.c_double(b1), ctypes.c_double(b2), ctypes.c_double(eps), ctypes.c_int32(t),
                        ctypes.c_int32(0 if clamp is None else 1), ctypes.c_double(0.0 if clamp is None else clamp))
    return x, m, v


def euler_zyx(euler):
    e = _d(euler)
    R = np.zeros(9)
    dR = np.zeros(27)
    _load().oracle_euler_zyx(_p(e), _p(R), _p(dR))
    return R.reshape(3, 3), dR.reshape(3, 3, 3)


def step(grid, acq, tmpl, meas, p0, euler_t, adam_p0, adam_pose, *, lr_p0, lr_rot, lr_trans, b1=0.9, b2=0.999,
         eps=1e-8, t=1, loss_kind=0, mask=None, update_p0=True, update_pose=True):
    """One SfM iteration (see pa_oracle.c oracle_step). Returns dict with updated state + diagnostics."""
    tmpl, meas = _d(tmpl), _d(meas)
    p0, euler_t = _d(p0).copy(), _d(euler_t).copy()
    adam_p0, adam_pose = _d(adam_p0).copy(), _d(adam_pose).copy()
    E, F = tmpl.shape[0], euler_t.shape[0]
    nvox = p0.size
    gp0, gpose, geul = np.zeros(nvox), np.zeros((F, 12)), np.zeros((F, 6))
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
    g, a = _grid(grid), _acq(acq)
    L = _load().oracle_step(ctypes.byref(g), ctypes.byref(a), _p(tmpl), ctypes.c_int32(E), ctypes.c_int32(F),
                            _p(meas), _p(p0), _p(euler_t), _p(adam_p0), _p(adam_pose), ctypes.c_double(lr_p0),
                            ctypes.c_double(lr_rot), ctypes.c_double(lr_trans), ctypes.c_double(b1),
                            ctypes.c_double(b2), ctypes.c_double(eps), ctypes.c_int32(t), ctypes.c_int32(loss_kind),
                            _p(m), ctypes.c_int32(int(update_p0)), ctypes.c_int32(int(update_pose)), _p(gp0),
                            _p(gpose), _p(geul))
    return dict(loss=L, p0=p0, euler_t=euler_t, adam_p0=adam_p0, adam_pose=adam_pose, grad_p0=gp0,
                grad_pose=gpose, grad_euler=geul)
