"""One EBK evaluation on one subinterval (oracle; test infrastructure only).

Solves   y'(τ) = A y(τ) + U p(τ),  y(0) = y0,   τ ∈ [0, npieces·h]
where p is the per-piece Taylor cubic from lowrank.notaknot_taylor (or p ≡ 0,
the homogeneous leg of Fig. 2), and returns y at every node τ_i = i·h.

Two routes to the same object:
  * ebk_dense  (n small): the definition written out — e^{hA} and φ_q(hA)U by the
    augmented exponential (expm.py), chained over the pieces.
  * ebk_krylov (any n): the paper's method: block Krylov
    subspace K_l(B, U) of the shift-and-invert operator B = (I - γA)^{-1},
    classical Gram-Schmidt applied twice, NO restart (reading #5: the oracle keeps
    one large space), projected matrix Â = (I - H^{-1})/γ, the projected IVP
    z' = Â z + E p(τ) integrated exactly per cubic piece (replaces ode15s),
    stop when the residual at every node is below eta (default 1e-12, 100x under
    the GPU's eta = 0.01·tol).

Residual (derived from the SaI Arnoldi relation B V_k = V_k H + Ṽ H_tail):
    r(τ) = A V_k z - V_k z' + U p = (1/γ)(I - γA) Ṽ H_tail H^{-1} z(τ).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from .expm import phi_blocks, chain


class OracleNoConvergence(RuntimeError):
    pass


def ebk_dense(A, U, coef, h, npieces, y0=None):
    n = A.shape[0]
    Ad = A.toarray() if sp.issparse(A) else np.asarray(A)
    Uc = U if U is not None else np.zeros((n, 0))
    F0, B = phi_blocks(Ad, Uc, h, nq=coef.shape[1] if (coef is not None and Uc.shape[1]) else 4)
    z0 = np.zeros(n) if y0 is None else y0
    return chain(F0, B, coef if Uc.shape[1] else None, h, z0, npieces)


def ebk_krylov(A, U, coef, h, npieces, gamma, y0=None, eta=1e-12, kmax=900,
               scale=None, return_info=False):
    """SaI block Arnoldi EBK.  Exactly one of (U, coef) or y0 drives the problem:
    forced (U, coef, y0 = None) or homogeneous (U = None, y0 given)."""
    n = A.shape[0]
    A = sp.csr_matrix(A)
    forced = y0 is None
    if forced:
        V0 = U
        m = U.shape[1]
        if m == 0:
            Z = np.zeros((npieces + 1, n))
            return (Z, {"k": 0}) if return_info else Z
        # criterion scale: max over nodes of ||U p(τ_i)|| = ||c_{i,0}|| (U orthonormal)
        import math
        last = sum(coef[-1, q] * h ** q / math.factorial(q) for q in range(coef.shape[1]))   # p at the end node
        nodes = np.concatenate([coef[:, 0, :], last[None]])
        tgt = eta * (scale if scale is not None else np.max(np.linalg.norm(nodes, axis=1)))
    else:
        beta = np.linalg.norm(y0)
        if beta == 0.0:
            Z = np.zeros((npieces + 1, n))
            return (Z, {"k": 0}) if return_info else Z
        V0 = (y0 / beta)[:, None]
        m = 1
        tgt = eta * beta / (npieces * h)
    M = (sp.identity(n, format="csc") - gamma * A).tocsc()
    lu = splu(M)
    V = np.zeros((n, kmax + m + 1))
    V[:, :m] = V0
    H = np.zeros((kmax + m + 1, kmax + m))
    nb, c = m, 0
    while True:
        stop_c = min(c + m, nb)
        while c < stop_c:                           # one block step
            w = lu.solve(V[:, c].copy())
            n0 = np.linalg.norm(w)
            for _ in range(2):                      # CGS2
                hh = V[:, :nb].T @ w
                w = w - V[:, :nb] @ hh
                H[:nb, c] += hh
            nw = np.linalg.norm(w)
            if nw > 1e-12 * n0:
                V[:, nb] = w / nw
                H[nb, c] = nw
                nb += 1
            c += 1
            if nb > kmax:
                raise OracleNoConvergence(f"oracle Krylov dimension exceeded {kmax}")
        k = c
        Hs = H[:k, :k]
        Ht = H[k:nb, :k]
        Hinv = np.linalg.inv(Hs)
        Ahat = (np.eye(k) - Hinv) / gamma
        if forced:
            E = np.zeros((k, m)); E[:m, :m] = np.eye(m)
            F0, B = phi_blocks(Ahat, E, h, nq=coef.shape[1])
            Z = chain(F0, B, coef, h, np.zeros(k), npieces)
        else:
            F0, B = phi_blocks(Ahat, np.zeros((k, 0)), h)
            z0 = np.zeros(k); z0[0] = beta
            Z = chain(F0, B, None, h, z0, npieces)
        if nb == k:
            res = 0.0                               # invariant subspace: exact
        else:
            Wt = (M @ V[:, k:nb]) / gamma
            X = Ht @ (Hinv @ Z.T)                   # [(nb-k)][nodes]
            res = float(np.max(np.linalg.norm(Wt @ X, axis=0)))
        if res <= tgt or nb == k:
            Y = Z @ V[:, :k].T
            if return_info:
                return Y, {"k": k, "res": res, "tgt": tgt}
            return Y
