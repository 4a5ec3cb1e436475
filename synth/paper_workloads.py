"""Seeded-free manufactured workloads of the paper's own experiments.

Like ``configs.py`` this module holds NO arithmetic of the method: it evaluates closed-form
manufactured solutions u(x, t) and their sources f = u_t + (PDE terms) at grid points and sample
nodes.  Two kinds of source:

  * ``continuous``: f from the exact derivatives of u (the semi-discrete solution then differs from
    u by the spatial discretisation error, "error converges to a value that depends on the
    mesh width");
  * ``discrete``: f such that the *semi-discrete* system reproduces u exactly ("the source
    term accounts for the error by the spatial discretization").  Every manufactured solution here
    is a finite Fourier series on the periodic unit interval, so its central-difference derivatives
    are evaluated per mode from the difference symbols in closed form,
        D1 e^{2πikx} = i sin(2πkΔx)/Δx e^{2πikx},   D2 e^{2πikx} = (2cos(2πkΔx) - 2)/Δx² e^{2πikx},
    never by applying a stencil to grid data.

Workloads (citations: PAPER.md line numbers):
  pulse_ade         f1: five travelling pulses u = 1/2 - 1/2 cos(10π(x - t)) of Eq.(ade)/(manusol)
                    (P:555-564), n = 1000 (Δx = 1e-3), a = 1, ν = 1e-2, tol = 1e-4, rank-2
                    source ("retain only the first two").
  sawtooth_burgers  f2: smoothed sawtooth Eq.(modifiedSawtooth), ξ = x - t/2 + 1/2
                    (P:651), k_max = 100, ε = 0.1, ν = 1e-2.
  multiscale_burgers f2: Eq.(multiscale_solution), k0 ∈ {4, 16}.
"""
from __future__ import annotations

import numpy as np

from .configs import PERIODIC, LinearProblem, BurgersProblem, grid_x, node_times


def _symbols(k, dx):
    """Central-difference symbols of the mode sin/cos(2πkx) on a periodic grid of width dx:
    D1 cos = -s1 sin, D1 sin = s1 cos with s1 = sin(2πkΔx)/Δx;  D2 = s2 with s2 = (2cos(2πkΔx)-2)/Δx²."""
    th = 2 * np.pi * k * dx
    return np.sin(th) / dx, (2 * np.cos(th) - 2) / dx ** 2


# ------------------------------------------------------------------------------------------ f1
def pulse_exact(x, t, a=1.0):
    """u(x, t) = 1/2 - 1/2 cos(10π(x - a t))  (Eq.(manusol), a = 1)."""
    return 0.5 - 0.5 * np.cos(10 * np.pi * (x - a * t))


def pulse_ade(P=2, dT=0.5, n=1000, s=64, tol=1e-4, nu=1e-2, a=1.0, T=None, node_rule=0) -> LinearProblem:
    """f1 workload: Eq.(ade) u_t + a u_x = ν u_xx + f with the five-pulse solution Eq.(manusol).

    f = u_t + a u_x - ν u_xx of the exact solution (continuous source):
      θ = 10π(x - a t):  u_t = -5πa sin θ,  u_x = 5π sin θ,  u_xx = 50π² cos θ
      f = -5πa sin θ + 5πa sin θ - 50π²ν cos θ = -50π²ν cos θ.
    Readings (f1): T = P·ΔT (the paper's τ0 grows ∝ P, Table 1), ΔT = 0.5;
    s = 64 (the paper's 100 samples exceed the library's s ≤ 64; the source is exactly rank 2 in
    x, so only the spline error of sin(10πt) changes, ~1e-8 relative)."""
    T = P * dT if T is None else T
    x = grid_x(n, PERIODIC)
    t = node_times(T, P, s, node_rule)                             # [P][s]
    th = 10 * np.pi * (x[None, None, :] - a * t[:, :, None])
    src = -50 * np.pi ** 2 * nu * np.cos(th)
    u0 = pulse_exact(x, 0.0, a)
    return LinearProblem("F1", n, PERIODIC, np.array([nu]), np.array([a]), T, P, s, tol,
                         u0[None].copy(), src[None].copy(), np.array([0]))


# ------------------------------------------------------------------------------------------ f2
def sawtooth_modes(kmax=100, eps=0.1):
    """Amplitudes b_k = Φ(k, ε)/(πk), Φ = (πkε/2)/sinh(πkε/2) (the printed bracket
    has no exponent, reading #19)."""
    k = np.arange(1, kmax + 1, dtype=np.float64)
    z = np.pi * k * eps / 2
    return k, (z / np.sinh(z)) / (np.pi * k)


def sawtooth_exact(x, t, kmax=100, eps=0.1):
    """u = 1/2 - Σ_k b_k sin(2πkξ), ξ = x - t/2 + 1/2 (Eq.(modifiedSawtooth))."""
    k, b = sawtooth_modes(kmax, eps)
    xi = np.asarray(x)[..., None] - 0.5 * np.asarray(t)[..., None] + 0.5
    return 0.5 - np.sum(b * np.sin(2 * np.pi * k * xi), axis=-1)


def _sawtooth_source(x, t, nu, kmax, eps, discrete, dx):
    """f = u_t + u u_x - ν u_xx on the grid at times t (array), continuous or discrete (module doc)."""
    k, b = sawtooth_modes(kmax, eps)
    xi = x[None, :] - 0.5 * t[:, None] + 0.5                       # [nt][n]
    arg = 2 * np.pi * k[None, None, :] * xi[:, :, None]            # [nt][n][K]
    S, C = np.sin(arg), np.cos(arg)
    u = 0.5 - np.einsum("k,tnk->tn", b, S)
    w = 2 * np.pi * k
    u_t = 0.5 * np.einsum("k,tnk->tn", b * w, C)                   # dξ/dt = -1/2
    if discrete:
        s1, s2 = _symbols(k, dx)
        ux = -np.einsum("k,tnk->tn", b * s1, C)
        uxx = -np.einsum("k,tnk->tn", b * s2, S)
    else:
        ux = -np.einsum("k,tnk->tn", b * w, C)
        uxx = np.einsum("k,tnk->tn", b * w * w, S)
    return u_t + u * ux - nu * uxx


def sawtooth_burgers(P=2, dT=0.1, n=400, s=50, tol=1e-4, nu=1e-2, kmax=100, eps=0.1,
                     forcing="continuous", T=None, max_wr_iters=30, wr_tol=1e-6) -> BurgersProblem:
    """f2 travelling sawtooth: Eq.(burgersEq) with f making Eq.(modifiedSawtooth) the solution.

    Defaults follow P:672-677 (tol 1e-4, s = 50, Δx = 2.5e-3, ΔT = 0.1, T = PΔT); the efficiency
    protocol is ``forcing="discrete", n=500, dT=0.2/P, s=128/P`` (s ≤ 64 here)."""
    T = P * dT if T is None else T
    x = grid_x(n, PERIODIC)
    t = node_times(T, P, s)
    f = _sawtooth_source(x, t.ravel(), nu, kmax, eps, forcing == "discrete", 1.0 / n).reshape(P, s, n)
    u0 = sawtooth_exact(x, 0.0 * x, kmax, eps)
    pb = BurgersProblem("F2-sawtooth", n, nu, T, P, s, tol, u0, max_wr_iters, wr_tol)
    pb.f = f
    return pb


def multiscale_exact(x, t, k0):
    """u = sin(2πx) sin(2πt) + (1/k0) sin(2k0πx) sin(2k0πt)  (Eq.(multiscale_solution))."""
    return (np.sin(2 * np.pi * x) * np.sin(2 * np.pi * t)
            + np.sin(2 * k0 * np.pi * x) * np.sin(2 * k0 * np.pi * t) / k0)


def multiscale_burgers(P=2, k0=4, dT=0.1, n=400, s=50, tol=1e-4, nu=1e-2, forcing="continuous",
                       T=None, max_wr_iters=30, wr_tol=1e-6) -> BurgersProblem:
    """f2 multiscale example: the Fig. error_dtfix protocol (ΔT = 0.1, T = PΔT) with
    the two-scale solution.  ν and Δx are not printed for it: those of the travelling-wave runs
    (ν = 1e-2, Δx = 2.5e-3) are used (reading)."""
    T = P * dT if T is None else T
    x = grid_x(n, PERIODIC)
    t = node_times(T, P, s).ravel()[:, None]
    X = x[None, :]
    modes = [(1.0, 1.0), (float(k0), 1.0 / k0)]                    # (wavenumber q, amplitude c)
    u = sum(c * np.sin(2 * np.pi * q * X) * np.sin(2 * np.pi * q * t) for q, c in modes)
    u_t = sum(c * 2 * np.pi * q * np.sin(2 * np.pi * q * X) * np.cos(2 * np.pi * q * t) for q, c in modes)
    if forcing == "discrete":
        syms = [_symbols(q, 1.0 / n) for q, _ in modes]
        ux = sum(c * s1 * np.cos(2 * np.pi * q * X) * np.sin(2 * np.pi * q * t)
                 for (q, c), (s1, _) in zip(modes, syms))
        uxx = sum(c * s2 * np.sin(2 * np.pi * q * X) * np.sin(2 * np.pi * q * t)
                  for (q, c), (_, s2) in zip(modes, syms))
    else:
        ux = sum(c * 2 * np.pi * q * np.cos(2 * np.pi * q * X) * np.sin(2 * np.pi * q * t) for q, c in modes)
        uxx = sum(-c * (2 * np.pi * q) ** 2 * np.sin(2 * np.pi * q * X) * np.sin(2 * np.pi * q * t)
                  for q, c in modes)
    f = (u_t + u * ux - nu * uxx).reshape(P, s, n)
    u0 = multiscale_exact(x, 0.0, k0)
    pb = BurgersProblem(f"F2-multiscale-k{k0}", n, nu, T, P, s, tol, u0, max_wr_iters, wr_tol)
    pb.f = f
    return pb
