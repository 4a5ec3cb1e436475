"""Semi-discrete operators (oracle; test infrastructure only — see oracle/__init__.py).

PAPER.md:465 (§3.1): "discretized in space with a second-order central finite
difference scheme"; PAPER.md:458-462 periodic BCs; PAPER.md:636 Burgers
u_t + u u_x = nu u_xx.  Grids (reading #15): periodic x_i = i/n, dx = 1/n;
Dirichlet x_i = i/(n+1), i = 1..n, dx = 1/(n+1), zero boundary values.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def grid_dx(n: int, bc: str) -> float:
    if bc == "periodic":
        return 1.0 / n
    if bc == "dirichlet":
        return 1.0 / (n + 1)
    raise ValueError(bc)


def d1_matrix(n: int, bc: str = "periodic") -> sp.csr_matrix:
    """Central first difference (u_{i+1} - u_{i-1}) / (2 dx)."""
    dx = grid_dx(n, bc)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i + 1, 1.0)):
            if bc == "periodic":
                j %= n
            elif not (0 <= j < n):
                continue
            rows.append(i); cols.append(j); vals.append(v / (2 * dx))
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def d2_matrix(n: int, bc: str = "periodic") -> sp.csr_matrix:
    """Central second difference (u_{i-1} - 2 u_i + u_{i+1}) / dx^2."""
    dx = grid_dx(n, bc)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j, v in ((i - 1, 1.0), (i, -2.0), (i + 1, 1.0)):
            if bc == "periodic":
                j %= n
            elif not (0 <= j < n):
                continue
            rows.append(i); cols.append(j); vals.append(v / dx ** 2)
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def ade_matrix(n: int, bc: str, nu: float, a: float) -> sp.csr_matrix:
    """A = nu*D2 - a*D1 for u_t + a u_x = nu u_xx."""
    return (nu * d2_matrix(n, bc) - a * d1_matrix(n, bc)).tocsr()


def burgers_N(u: np.ndarray, n: int) -> np.ndarray:
    """Nonlinear term g(u) = -u∘(D1 u), advective form of PAPER.md:636 (reading #16)."""
    return -u * (d1_matrix(n) @ u)


def burgers_J(ubar: np.ndarray, n: int) -> sp.csr_matrix:
    """Jacobian of g(u) = -u∘(D1 u) at ubar: J = -diag(D1 ubar) - diag(ubar) D1.

    Used as J(ū_j) = (1/ΔT)∫ ∂g/∂u dt of Eq.(piecewiseJac) PAPER.md:297-301 —
    J is linear in u, so the time average of J equals J of the time average
    (reading #3)."""
    D1 = d1_matrix(n)
    return (-sp.diags(D1 @ ubar) - sp.diags(ubar) @ D1).tocsr()
