"""Closed-form solutions from the paper's appendix — TEST INFRASTRUCTURE (oracle pins).

Every function is a literal transcription of a displayed equation of PAPER.md
(P:n = /root/reference/PAPER.md line n).  These are independent of the discrete
model (Eq. gpu_forward_model) that ``pa_oracle.c`` evaluates; tests use them to pin
the oracle.  Units: mm, µs, mm/µs.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf


def boxed(r, t, p0_of, c):
    """Unified spherically-symmetric solution, boxed Eq. final_expression:
    p(r,t) = 1/(2r) [ (r + c t) p0(r + c t) + (r - c t) p0(|r - c t|) ]."""
    r = np.asarray(r, dtype=np.float64)
    ct = c * np.asarray(t, dtype=np.float64)
    return ((r + ct) * p0_of(r + ct) + (r - ct) * p0_of(np.abs(r - ct))) / (2.0 * r)


def far_field(r, t, p0_of, c):
    """Unified far-field approximation, Eq. far_field_general:
    p(r,t) ~ 1/(2r) (r - c t) p0(|r - c t|)."""
    r = np.asarray(r, dtype=np.float64)
    ct = c * np.asarray(t, dtype=np.float64)
    return (r - ct) * p0_of(np.abs(r - ct)) / (2.0 * r)


def uniform_sphere(r, t, p0, a0, c):
    """Uniform sphere p0(r) = p0 U(a0 - r), observation point r > a0:
    p = p0/(2r) (r - c t) when r - a0 <= c t <= r + a0, else 0."""
    r = np.asarray(r, dtype=np.float64)
    ct = c * np.asarray(t, dtype=np.float64)
    inside = (r - a0 <= ct) & (ct <= r + a0)
    return np.where(inside, p0 / (2.0 * r) * (r - ct), 0.0)


def gaussian_solution(r, t, pc, s, c):
    """Gaussian distribution p0(r) = pc exp(-r^2/2s^2), Eq. gaussian_solution."""
    r = np.asarray(r, dtype=np.float64)
    ct = c * np.asarray(t, dtype=np.float64)
    return pc / (2.0 * r) * ((r + ct) * np.exp(-(r + ct) ** 2 / (2 * s * s))
                             + (r - ct) * np.exp(-(r - ct) ** 2 / (2 * s * s)))


def gaussian_far_field(r, t, pc, s, c):
    """Outgoing Gaussian pulse, Eq. gaussian_far_field."""
    r = np.asarray(r, dtype=np.float64)
    ct = c * np.asarray(t, dtype=np.float64)
    return pc / (2.0 * r) * (r - ct) * np.exp(-(r - ct) ** 2 / (2 * s * s))


def exponential_solution(r, t, pc, a, c):
    """Exponential distribution p0 = pc e^{-r/a}, Eq. exponential_solution."""
    r = np.asarray(r, dtype=np.float64)
    ct = c * np.asarray(t, dtype=np.float64)
    return pc / (2.0 * r) * ((r + ct) * np.exp(-(r + ct) / a) + (r - ct) * np.exp(-np.abs(r - ct) / a))


def power_law_solution(r, t, A, a, nu, c):
    """Power law p0 = A/(r^2 + a^2)^nu, Eq. power_law_solution."""
    r = np.asarray(r, dtype=np.float64)
    ct = c * np.asarray(t, dtype=np.float64)
    return A / (2.0 * r) * ((r + ct) / ((r + ct) ** 2 + a * a) ** nu + (r - ct) / ((r - ct) ** 2 + a * a) ** nu)


def smoothed_ball_profile(rho, R, p0, sigma):
    """Radial profile of a uniform ball (radius R, density p0) convolved with a normalised
    isotropic Gaussian of std sigma (the blob lattice's smoothing, R2/R3):
    p~0(rho) = p0 { 1/2 [erf((R-rho)/(sqrt2 s)) + erf((R+rho)/(sqrt2 s))]
                    - s/(rho sqrt(2 pi)) [e^{-(R-rho)^2/2s^2} - e^{-(R+rho)^2/2s^2}] }.
    (Standard result: 3-D Gaussian blur of an indicator of a ball, evaluated radially.)"""
    rho = np.maximum(np.asarray(rho, dtype=np.float64), 1e-12)
    s = sigma
    a = 0.5 * (erf((R - rho) / (np.sqrt(2) * s)) + erf((R + rho) / (np.sqrt(2) * s)))
    b = s / (rho * np.sqrt(2 * np.pi)) * (np.exp(-(R - rho) ** 2 / (2 * s * s)) - np.exp(-(R + rho) ** 2 / (2 * s * s)))
    return p0 * (a - b)


def shell_integral_pressure(r, t, p0_of, c, n=20001, h=1e-4):
    """Numerical route (independent of the boxed closed form): Eq. pressure_simplified
    p = 1/(2 c r) d/dt int_{|r-ct|}^{r+ct} r' p0(r') dr', integral by composite Simpson,
    time derivative by a central difference of step h (µs)."""
    def inner(tt):
        lo, hi = abs(r - c * tt), r + c * tt
        x = np.linspace(lo, hi, n)
        w = np.ones(n)
        w[1:-1:2] = 4.0
        w[2:-1:2] = 2.0
        return (hi - lo) / (3.0 * (n - 1)) * np.sum(w * x * p0_of(x))
    return (inner(t + h) - inner(t - h)) / (2 * h) / (2.0 * c * r)
