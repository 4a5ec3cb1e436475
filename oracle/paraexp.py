"""Linear Paraexp-EBK (PEBK) solve (oracle; test infrastructure only).

Follows Fig. 2 and §2.2 step by step:
  1. shift to homogeneous IC: u = u0 + û, ĝ(t) = A u0 + g(t)          (Eq.(linivp_shift))
  2. partition [0,T] into P subintervals, ĝ_j = ĝ on [T_{j-1}, T_j)     (Eq.(piecewiseSource_linivp))
  3. per subinterval: sample ĝ at the s nodes, truncated SVD, spline p
  4. nonhomogeneous part v_j on [T_{j-1}, T_j], v_j(T_{j-1}) = 0           (Eq.(linivpSubproblem))
  5. homogeneous part v_j(T_i) = exp((T_i - T_j)A) v_j(T_j), i > j        (Fig. 2 line 3)
  6. superposition u(T_i) = u0 + Σ_{j<=i} v_j(T_i)                        (Eq.(superposition))
Returns out[b][i] = u(T_{i+1}) (0-based i; reading #12).
"""
from __future__ import annotations

import numpy as np

from .operators import ade_matrix
from .lowrank import truncated_svd, notaknot_taylor, cheb_taylor
from .ebk import ebk_dense, ebk_krylov


def solve_linear(n, bc, nu, a, u0, src, T, P, s, tol, *, eta=1e-12, dense_max=1024,
                 i_max=None, svd_tau_factor=0.01, return_info=False, node_rule=0):
    """u0: [batch][n]; src: [batch][P][s][n] (g at the nodes of synth.node_times);
    nu, a: [batch].  Returns out [batch][P'][n], P' = P or i_max.
    node_rule 0: uniform nodes, not-a-knot cubic p(t) (readings #8, #9); node_rule 1 (row f3):
    Chebyshev-Lobatto nodes, p(t) = the degree-(s-1) interpolant (reading #23)."""
    u0 = np.atleast_2d(u0)
    batch = u0.shape[0]
    nu = np.broadcast_to(np.asarray(nu, dtype=np.float64), (batch,))
    a = np.broadcast_to(np.asarray(a, dtype=np.float64), (batch,))
    Pout = P if i_max is None else i_max
    dT = T / P
    h = dT / (s - 1)
    tau = svd_tau_factor * tol
    out = np.empty((batch, Pout, n))
    info = {"m": np.zeros((batch, Pout), dtype=int), "k": np.zeros((batch, Pout), dtype=int)}
    for b in range(batch):
        A = ade_matrix(n, bc, nu[b], a[b])
        Au0 = A @ u0[b]
        dense = n <= dense_max
        if dense:
            from scipy.linalg import expm
            EdT = expm(dT * A.toarray())
        vend = np.empty((Pout, n))                  # v_j(T_j)
        for j in range(Pout):
            G = Au0[:, None] + src[b, j].T          # step 1/3: Ĝ_j = A u0 + g(t_{j,i})
            U, C, _ = truncated_svd(G, tau)         # step 3
            info["m"][b, j] = U.shape[1]
            if U.shape[1] == 0:
                vend[j] = 0.0
                continue
            coef = notaknot_taylor(C, h) if node_rule == 0 else cheb_taylor(C, dT, s - 1)
            if dense:                               # step 4
                Y = ebk_dense(A, U, coef, h, s - 1)
            else:
                Y, inf = ebk_krylov(A, U, coef, h, s - 1, gamma=dT / 10, eta=eta, return_info=True)
                info["k"][b, j] = inf["k"]
            vend[j] = Y[-1]
        acc = u0[b][None, :] + vend                 # step 6, own term v_i(T_i)
        for j in range(Pout - 1):                   # step 5: leg of v_j over [T_j, T_P]
            nleg = Pout - 1 - j
            if dense:
                W = np.empty((nleg + 1, n))
                W[0] = vend[j]
                for q in range(nleg):
                    W[q + 1] = EdT @ W[q]
            else:
                W = ebk_krylov(A, None, None, dT, nleg, gamma=T / 10, y0=vend[j], eta=eta)
            acc[j + 1:] += W[1:]                    # W[q] = exp(qΔT A) v_j(T_j) → T_{j+q}
        out[b] = acc
    return (out, info) if return_info else out
