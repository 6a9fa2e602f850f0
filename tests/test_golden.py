"""Golden pins (-m "not gpu"): the oracle against values worked out by hand from the paper's equations.

tests/golden/closed_form_points.txt — the appendix closed forms at hand-chosen points,
pinning the transcriptions in oracle/closed_forms.py that P1-P4 compare the discrete oracle with.
tests/golden/single_blob_trace.txt — samples of Eq. gpu_forward_model for one voxel,
pinning oracle.forward directly (amplitude, 1/2r, sign of Delta, Gaussian width, window).
P:n = /root/reference/PAPER.md line n (citations only; nothing here reads that file).
"""
import os

import numpy as np
import pytest

import oracle
from oracle import closed_forms as cf

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rows(name):
    out = []
    with open(os.path.join(GOLD, name)) as fh:
        for ln in fh:
            if ln.strip() and not ln.startswith("#"):
                out.append(ln.split())
    return out


def params(s):
    return {k: float(v) for k, v in (kv.split("=") for kv in s.split(","))}


def closed_form(form, r, t, c, p):
    if form == "uniform_sphere":
        return cf.uniform_sphere(r, t, p["p0"], p["a0"], c)
    if form == "gaussian_far":
        return cf.gaussian_far_field(r, t, p["pc"], p["s"], c)
    if form == "gaussian_sol":
        return cf.gaussian_solution(r, t, p["pc"], p["s"], c)
    if form == "exponential_sol":
        return cf.exponential_solution(r, t, p["pc"], p["a"], c)
    if form == "power_law_sol":
        return cf.power_law_solution(r, t, p["A"], p["a"], p["nu"], c)
    raise KeyError(form)


CF_ROWS = rows("closed_form_points.txt")


@pytest.mark.parametrize("row", CF_ROWS, ids=[f"{r[0]}-r{r[1]}-t{r[2]}" for r in CF_ROWS])
def test_closed_forms_match_worked_values(row):
    form, r, t, c, p, want = row[0], float(row[1]), float(row[2]), float(row[3]), params(row[4]), float(row[5])
    got = float(closed_form(form, r, t, c, p))
    assert abs(got - want) <= 1e-12 * max(1.0, abs(want)), (form, got, want)


def test_uniform_sphere_boxed_form_matches_worked_values():
    """The boxed unified solution with p0(r) = p0 U(a0 - r) reduces to P:303-305 for r > a0."""
    for row in CF_ROWS:
        if row[0] != "uniform_sphere":
            continue
        r, t, c, p, want = float(row[1]), float(row[2]), float(row[3]), params(row[4]), float(row[5])
        got = float(cf.boxed(r, t, lambda x: np.where(np.asarray(x) < p["a0"], p["p0"], 0.0), c))
        assert abs(got - want) <= 1e-12, (r, t, got, want)


def test_oracle_forward_single_voxel_matches_worked_samples():
    g = dict(nx=1, ny=1, nz=1, origin=[0.0, 0.0, 0.0], pitch=0.2)
    a = dict(c=1.5, t0=0.0, dt=0.025, nt=256, sigma=0.5, kappa=5.0)
    pose = np.zeros((1, 12))
    pose[0, :9] = np.eye(3).reshape(-1)
    y = oracle.forward(g, a, np.array([[0.0, 0.0, 2.0]]), pose, np.array([1.0]))[0, 0]
    for row in rows("single_blob_trace.txt"):
        j, want = int(row[0]), float(row[1])
        assert abs(y[j] - want) <= 1e-12 * max(abs(want), 1e-3), (j, y[j], want)
