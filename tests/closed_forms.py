"""Independent closed forms used to PIN the oracle (never used by the oracle itself).

* scalar φ-functions φ_q(z), complex z, by power series (|z| < 1) or the upward
  recurrence φ_{q+1}(z) = (φ_q(z) - 1/q!)/z (|z| >= 1) — no matrix exponential;
* the circulant diagonalisation of the periodic central-difference operator:
  A e_k = λ_k e_k, e_k(x_i) = exp(2πi k i/n),
  λ_k = -(4ν/Δx²) sin²(πk/n) - i (a/Δx) sin(2πk/n);
* the exact solution of the periodic ADE with a piecewise-cubic source, mode by
  mode (SURVEY §8(c).4 "One linear EBK (interpolated source)").
"""
from __future__ import annotations

import math

import numpy as np


def phi_scalar(q: int, z: np.ndarray) -> np.ndarray:
    """φ_q(z) elementwise for complex/real arrays, q >= 0."""
    z = np.asarray(z, dtype=np.complex128)
    out = np.empty_like(z)
    small = np.abs(z) < 1.0
    if np.any(small):
        zs = z[small]
        acc = np.zeros_like(zs)
        term = np.ones_like(zs) / math.factorial(q)
        for j in range(60):
            acc = acc + term
            term = term * zs / (q + j + 1)
        out[small] = acc
    big = ~small
    if np.any(big):
        zb = z[big]
        p = np.exp(zb)
        for r in range(q):
            p = (p - 1.0 / math.factorial(r)) / zb
        out[big] = p
    return out


def periodic_eigs(n: int, nu: float, a: float) -> np.ndarray:
    dx = 1.0 / n
    k = np.arange(n)
    return -(4 * nu / dx ** 2) * np.sin(np.pi * k / n) ** 2 - 1j * (a / dx) * np.sin(2 * np.pi * k / n)


def periodic_forced_solution(n, nu, a, coef_phys, h, z0=None):
    """Exact y at every node for y' = A y + s(τ), y(0) = z0, A periodic ADE, s piecewise
    cubic with physical-space Taylor coefficients coef_phys [npieces][4][n].
    Uses numpy's FFT only to change basis (a library primitive)."""
    lam = periodic_eigs(n, nu, a)
    # FFT convention: A acts diagonally on np.fft.fft coefficients with eigenvalue λ_k
    npieces = coef_phys.shape[0]
    c = np.zeros(n, dtype=np.complex128) if z0 is None else np.fft.fft(z0)
    e0 = np.exp(lam * h)
    ph = [phi_scalar(q + 1, lam * h) for q in range(4)]
    out = [np.real(np.fft.ifft(c))]
    for i in range(npieces):
        c = e0 * c
        for q in range(4):
            c = c + h ** (q + 1) * ph[q] * np.fft.fft(coef_phys[i, q])
        out.append(np.real(np.fft.ifft(c)))
    return np.array(out)


def periodic_propagate(n, nu, a, v, t):
    """exp(tA) v for the periodic ADE operator (circulant closed form)."""
    lam = periodic_eigs(n, nu, a)
    return np.real(np.fft.ifft(np.exp(lam * t) * np.fft.fft(v)))


def pulse_semidiscrete(x, t, nu, a, n):
    """Exact solution of the periodic semi-discrete f1 problem (Eq.(ade)/(manusol) P:555-563)
    u' = (νD2 - aD1)u + f(t), f = -50π²ν cos(10π(x - a t)), u(0) = 1/2 - 1/2 cos(10πx).
    Single circulant mode k = 10π: u = 1/2 + Re(c(t) e^{ikx}), c' = λc + F e^{-iωt},
    λ = ν(2cos(kΔx) - 2)/Δx² - i a sin(kΔx)/Δx, F = -50π²ν, ω = k a, c(0) = -1/2:
        c(t) = e^{λt} c(0) + F (e^{-iωt} - e^{λt}) / (-iω - λ)."""
    k = 10 * np.pi
    dx = 1.0 / n
    lam = nu * (2 * np.cos(k * dx) - 2) / dx ** 2 - 1j * a * np.sin(k * dx) / dx
    F = -50 * np.pi ** 2 * nu
    w = k * a
    c = np.exp(lam * t) * (-0.5) + F * (np.exp(-1j * w * t) - np.exp(lam * t)) / (-1j * w - lam)
    return 0.5 + np.real(c * np.exp(1j * k * x))
