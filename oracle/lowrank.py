"""Low-rank source approximation g(t) ≈ U p(t) (oracle; test infrastructure only).

PAPER.md:64-78 (§2.1): sample G = [g(t_1) … g(t_s)], thin SVD G = Ũ Σ̃ Ṽᵀ,
keep the m largest singular values, U = first m columns of Ũ, p(t) by
interpolation of the coefficients — "cubic piecewise polynomials".
Readings: m = #{σ_i > τ_svd·σ_1}, τ_svd = 0.01·tol (#7);
p(t) = not-a-knot cubic spline through the s uniform nodes (#8, #9).
"""
from __future__ import annotations

import numpy as np


def truncated_svd(G: np.ndarray, tau_rel: float):
    """Return (U [n][m], C [m][s], sigma [s]) with C = Uᵀ G (P:69-77 Eq.(svd_appr)).

    The thin SVD itself is a library primitive (LAPACK gesdd via numpy)."""
    Ut, sig, Vt = np.linalg.svd(G, full_matrices=False)
    if sig.size == 0 or sig[0] == 0.0:
        return np.zeros((G.shape[0], 0)), np.zeros((0, G.shape[1])), sig
    m = int(np.count_nonzero(sig > tau_rel * sig[0]))
    U = Ut[:, :m].copy()
    C = sig[:m, None] * Vt[:m]
    return U, C, sig


def notaknot_taylor(Y: np.ndarray, h: float) -> np.ndarray:
    """Not-a-knot cubic spline through uniform nodes τ_i = i·h, i = 0..s-1, for each
    row of Y [m][s].  Returns per-piece Taylor coefficients at the left node,
    shape [s-1][4][m]: (p, p', p'', p''') so that on piece i,
        p(τ_i + σ) = c0 + c1 σ + c2 σ²/2 + c3 σ³/6,  0 <= σ <= h.

    Unknowns M_i = p''(τ_i).  Interior rows (C² continuity):
        M_{i-1} + 4 M_i + M_{i+1} = 6 (y_{i+1} - 2 y_i + y_{i-1}) / h²
    Not-a-knot (p''' continuous at τ_1 and τ_{s-2}):
        M_0 - 2 M_1 + M_2 = 0,   M_{s-3} - 2 M_{s-2} + M_{s-1} = 0.
    The s×s solve is a library primitive (numpy.linalg.solve)."""
    Y = np.atleast_2d(Y)
    m, s = Y.shape
    if s < 4:
        raise ValueError("not-a-knot spline needs s >= 4")
    K = np.zeros((s, s))
    R = np.zeros((s, m))
    K[0, 0:3] = [1.0, -2.0, 1.0]
    K[s - 1, s - 3:s] = [1.0, -2.0, 1.0]
    for i in range(1, s - 1):
        K[i, i - 1:i + 2] = [1.0, 4.0, 1.0]
        R[i] = 6.0 * (Y[:, i + 1] - 2.0 * Y[:, i] + Y[:, i - 1]) / h ** 2
    M = np.linalg.solve(K, R).T              # [m][s]
    out = np.empty((s - 1, 4, m))
    for i in range(s - 1):
        out[i, 0] = Y[:, i]
        out[i, 1] = (Y[:, i + 1] - Y[:, i]) / h - h * (2.0 * M[:, i] + M[:, i + 1]) / 6.0
        out[i, 2] = M[:, i]
        out[i, 3] = (M[:, i + 1] - M[:, i]) / h
    return out


def cheb_taylor(Y: np.ndarray, dT: float, npieces: int) -> np.ndarray:
    """Higher-order p(t) on Chebyshev nodes ("Chebyshev nodes ... other types of
    p(t) are possible", DESIGN.md §3 reading #23).

    Each row of Y [m][s] holds the values at the Chebyshev-Lobatto nodes
    τ_i = (dT/2)(1 - cos(π i/(s-1))), i = 0..s-1, of the subinterval [0, dT].  p is THE polynomial
    of degree s-1 through them.  It is returned as its exact Taylor re-expansion about the uniform
    piece starts σ_i = i·dT/npieces (a polynomial of degree s-1 equals its s-term Taylor series):
        out[i][q] = p^{(q)}(σ_i),  shape [npieces][s][m],
        p(σ_i + σ) = Σ_{q<s} out[i][q] σ^q/q!.
    Interpolation, differentiation and evaluation in the Chebyshev basis are library primitives
    (numpy.polynomial.chebyshev: chebfit on s points with degree s-1 is interpolation)."""
    from numpy.polynomial import chebyshev as Ch
    Y = np.atleast_2d(Y)
    m, s = Y.shape
    x = -np.cos(np.pi * np.arange(s) / (s - 1))              # nodes mapped to [-1, 1]
    c = Ch.chebfit(x, Y.T, s - 1)                             # [s][m] Chebyshev coefficients
    xs = 2.0 * (np.arange(npieces) * (dT / npieces)) / dT - 1.0
    out = np.zeros((npieces, s, m))
    for q in range(s):
        cq = c if q == 0 else Ch.chebder(c, m=q, scl=2.0 / dT, axis=0)   # d^q/dτ^q
        out[:, q, :] = Ch.chebval(xs, cq).T if cq.shape[0] > 0 else 0.0
    return out


def eval_taylor(coef: np.ndarray, h: float, tau: float) -> np.ndarray:
    """Evaluate the piecewise cubic at local time tau in [0, (s-1)h]."""
    npieces = coef.shape[0]
    i = min(int(tau // h), npieces - 1)
    sg = tau - i * h
    c = coef[i]
    return c[0] + c[1] * sg + c[2] * sg ** 2 / 2 + c[3] * sg ** 3 / 6
