"""Exact integration of z' = X z + Y p(σ) with a cubic p over one step h (oracle).

Variation of constants: with p(σ) = Σ_{q=0}^{3} c_q σ^q/q!,
    z(h) = e^{hX} z(0) + Σ_{q=0}^{3} h^{q+1} φ_{q+1}(hX) Y c_q,
φ_0 = exp, φ_{q+1}(x) = (φ_q(x) - 1/q!)/x.  The blocks φ_{q+1}(hX)·hY come from the
exponential of the augmented matrix ("augmented-matrix exponential")
    [[hX, hY, 0, 0, 0],
     [0,  0,  I, 0, 0],
     [0,  0,  0, I, 0],
     [0,  0,  0, 0, I],
     [0,  0,  0, 0, 0]]
whose first block row is [e^{hX}, φ_1(hX)hY, φ_2(hX)hY, φ_3(hX)hY, φ_4(hX)hY]
(top-right block = ∫_0^1 e^{(1-σ)hX} hY e^{σN} dσ).  The matrix exponential is a
library primitive (scipy.linalg.expm, Padé scaling-and-squaring).
Test infrastructure only (oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import expm


def phi_blocks(X: np.ndarray, Y: np.ndarray, h: float, nq: int = 4):
    """Return (F0 = e^{hX}, [B_0..B_{nq-1}]) with B_q = φ_{q+1}(hX)·hY (nq = 4: cubic pieces;
    nq = s: the degree-(s-1) pieces of lowrank.cheb_taylor — the same augmented matrix with
    nq - 1 identity blocks on its superdiagonal)."""
    k = X.shape[0]
    m = Y.shape[1]
    if m == 0:
        return expm(h * X), [np.zeros((k, 0))] * nq
    N = k + nq * m
    M = np.zeros((N, N))
    M[:k, :k] = h * X
    M[:k, k:k + m] = h * Y
    for q in range(nq - 1):
        r0 = k + q * m
        M[r0:r0 + m, r0 + m:r0 + 2 * m] = np.eye(m)
    E = expm(M)
    F0 = E[:k, :k]
    B = [E[:k, k + q * m:k + (q + 1) * m] for q in range(nq)]
    return F0, B


def chain(F0, B, coef, h, z0, npieces):
    """z_{i+1} = F0 z_i + Σ_q h^q B_q c_{i,q} over npieces pieces; returns [npieces+1][k].

    coef: [npieces][nq][m] Taylor coefficients (or None for the homogeneous case)."""
    k = F0.shape[0]
    Z = np.empty((npieces + 1, k))
    Z[0] = z0
    for i in range(npieces):
        z = F0 @ Z[i]
        if coef is not None:
            for q in range(coef.shape[1]):
                z = z + (h ** q) * (B[q] @ coef[i, q])
        Z[i + 1] = z
    return Z
