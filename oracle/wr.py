"""Burgers waveform relaxation with Paraexp-EBK inside (oracle; test infrastructure only).

Follows Fig. 5 and §2.4:
  0. u_0(t) ≡ u0 at every node                                   (Fig. 5 "Initialize u_0(t)", reading #14)
  1. per subinterval j: ū_j = (1/ΔT)∫ u_k dt (trapezoid over the s nodes),
     J_{k,j} = J(ū_j)                                            (Eq.(piecewiseJac), reading #3)
  2. operator A_j = ν D2 + J_{k,j}; shifted source at the nodes
        ĝ_{j,k}(t) = A u0 + g_k(t) - J_{k,j} û_k(t)
                   = ν D2 u0 - u_k∘D1 u_k - J_{k,j}(u_k - u0) + f(t)
                                                                 (Eq.(sourceParallel), corrected: reading #2;
                                                                  forcing f of Eq.(burgersEq), f2 workloads)
  3. nonhomogeneous parts v_{j,k+1} on [T_{j-1}, T_j] by EBK      (Eq.(ivpSubproblem))
  4. homogeneous parts: v_j continued over later subintervals with each subinterval's own
     operator; summed first (linearity), this is the scan
        û(t) = exp((t - T_{i-1}) A_i) û(T_{i-1}) + v_i(t),  t ∈ [T_{i-1}, T_i]   (Fig. 5 line 4, reading #11)
  5. u_{k+1} = u0 + û at all nodes                                (Eq.(updateSolution))
  6. δ_k = max |u_{k+1} - u_k| over all nodes; stop if δ_k < wr_tol or at max_wr_iters (reading #13);
     error if δ non-finite or grows by > 1e3.
γ_j = min(ΔT/10, 0.5/max_i(-(D1 ū_j)_i)) (reading #4).
"""
from __future__ import annotations

import numpy as np

from .operators import d1_matrix, d2_matrix, burgers_J
from .lowrank import truncated_svd, notaknot_taylor
from .ebk import ebk_dense, ebk_krylov


class OracleDiverged(RuntimeError):
    pass


def trapezoid_mean(Uk_j: np.ndarray) -> np.ndarray:
    """(1/ΔT)∫ u dt by the composite trapezoid rule over s uniform nodes; Uk_j: [s][n]."""
    s = Uk_j.shape[0]
    return (0.5 * Uk_j[0] + Uk_j[1:s - 1].sum(axis=0) + 0.5 * Uk_j[s - 1]) / (s - 1)


def wr_gamma(ubar: np.ndarray, D1, dT: float) -> float:
    mx = float(np.max(-(D1 @ ubar)))
    g = dT / 10
    if mx > 0:
        g = min(g, 0.5 / mx)
    return g


def wr_map(Uk, u0, nu, n, T, P, s, tol, *, eta=1e-12, dense_max=1024, svd_tau_factor=0.01, info=None,
           f=None):
    """One WR iteration u_k -> u_{k+1} on all nodes; Uk: [P][s][n]; f: forcing [P][s][n] or None."""
    dT = T / P
    h = dT / (s - 1)
    D1 = d1_matrix(n)
    D2 = d2_matrix(n)
    A0 = nu * D2
    A0u0 = A0 @ u0
    dense = n <= dense_max
    Unew = np.empty_like(Uk)
    uhat_prev = np.zeros(n)                         # û(T_0) = 0
    V = np.empty((P, s, n))
    ops = []
    for j in range(P):                              # steps 1-3 (independent per j)
        ubar = trapezoid_mean(Uk[j])
        J = burgers_J(ubar, n)
        Aj = (A0 + J).tocsr()
        gam = wr_gamma(ubar, D1, dT)
        ops.append((Aj, gam))
        Ukj = Uk[j]                                 # [s][n]
        G = np.empty((n, s))
        for i in range(s):
            u = Ukj[i]
            G[:, i] = A0u0 - u * (D1 @ u) - J @ (u - u0)
            if f is not None:
                G[:, i] += f[j, i]
        U, C, _ = truncated_svd(G, svd_tau_factor * tol)
        if info is not None:
            info.setdefault("m", []).append(U.shape[1])
        if U.shape[1] == 0:
            V[j] = 0.0
            continue
        coef = notaknot_taylor(C, h)
        if dense:
            V[j] = ebk_dense(Aj, U, coef, h, s - 1)
        else:
            V[j] = ebk_krylov(Aj, U, coef, h, s - 1, gamma=gam, eta=eta)
    for i in range(P):                              # step 4: scan over subintervals
        Aj, gam = ops[i]
        if i == 0 or not np.any(uhat_prev):
            Wh = np.zeros((s, n))
        elif dense:
            Wh = ebk_dense(Aj, None, None, h, s - 1, y0=uhat_prev)
        else:
            Wh = ebk_krylov(Aj, None, None, h, s - 1, gamma=gam, y0=uhat_prev, eta=eta)
        uh = Wh + V[i]
        Unew[i] = u0[None, :] + uh                  # step 5
        uhat_prev = uh[-1]
    return Unew


def solve_burgers(n, nu, u0, T, P, s, tol, max_wr_iters=30, wr_tol=1e-6, *, eta=1e-12,
                  dense_max=1024, svd_tau_factor=0.01, return_info=False, fixed_iters=None, f=None):
    """Returns out [P][n] = u_K(T_1..T_P) (reading #12) and optionally info
    {"iters": K, "delta": [...], "U": final waveform [P][s][n], "out_hist": [u_k(T_1..T_P)]}.
    f: forcing samples [P][s][n] at the nodes (Eq.(burgersEq)), None for f = 0."""
    u0 = np.asarray(u0, dtype=np.float64)
    Uk = np.broadcast_to(u0, (P, s, n)).copy()      # step 0
    deltas = []
    info = {"m": []}
    kmax = max_wr_iters if fixed_iters is None else fixed_iters
    for k in range(kmax):
        Un = wr_map(Uk, u0, nu, n, T, P, s, tol, eta=eta, dense_max=dense_max,
                    svd_tau_factor=svd_tau_factor, info=info, f=f)
        info.setdefault("out_hist", []).append(Un[:, -1, :].copy())
        d = float(np.max(np.abs(Un - Uk)))
        deltas.append(d)
        Uk = Un
        if not np.isfinite(d) or d > 1e3 * deltas[0]:
            raise OracleDiverged(f"WR diverged at iteration {k + 1}: delta={d}")
        if fixed_iters is None and d < wr_tol:
            break
    out = Uk[:, -1, :].copy()
    if return_info:
        info.update({"iters": len(deltas), "delta": deltas, "U": Uk})
        return out, info
    return out
