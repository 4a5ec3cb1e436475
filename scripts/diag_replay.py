import sys, os, glob
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from oracle.operators import ade_matrix
p = synth.config4(indices=[0], P=16, s=32); dT=p.T/p.P; gam = dT/10
A = ade_matrix(p.n,p.bc,p.nu[0],p.a[0]).toarray(); M = np.eye(p.n) - gam*A
raw = open("/tmp/pe_K12.bin","rb").read()
n, kcap, K, m, nout = np.frombuffer(raw[:20], np.int32); o = 20
live = np.frombuffer(raw[o:o+4*kcap], np.int32); o += 4*kcap
V = np.frombuffer(raw[o:o+8*kcap*n], np.float64).reshape(kcap, n).T.copy()
def block_chol(G, norm0=None, defl=1e-10):
    N = G.shape[0]; g = np.diag(G).copy()
    dead = [not (g[k] > 0) or (norm0 is not None and not (g[k] > defl*defl*norm0[k])) for k in range(N)]
    d = np.where(g > 0, 1/np.sqrt(np.maximum(g, 1e-300)), 0.0)
    L = (d[:, None]*d[None, :])*0.5*(G + G.T)
    piv = []
    for k in range(N):
        pk = L[k, k]
        if dead[k] or not (pk > 1e-14):
            dead[k] = True; L[k:, k] = 0; piv.append(pk); continue
        L[k, k] = np.sqrt(pk); L[k+1:, k] /= L[k, k]; piv.append(pk)
        for i in range(k+1, N):
            for j in range(k+1, i+1):
                L[i, j] -= L[i, k]*L[j, k]
    X = np.zeros((N, N))
    for j in range(N):
        if dead[j]: continue
        for k in range(j, -1, -1):
            if dead[k]: continue
            s_ = (1.0 if k == j else 0.0) - sum(L[q, k]*X[q, j] for q in range(k+1, j+1))
            X[k, j] = s_/L[k, k]
    Rinv = d[:, None]*X
    R = np.array([[L[j, k]/d[j] if (j >= k and d[j] > 0) else 0 for j in range(N)] for k in range(N)])
    return R, Rinv, dead, piv
Vp = V[:, :12]            # blocks 0,1 (as stored)
W0 = np.linalg.solve(M, V[:, 6:12])
G0 = W0.T @ W0
H1 = Vp.T @ W0; W = W0 - Vp @ H1
G1 = W.T @ W
print("pass1 rel norms", np.sqrt(np.diag(G1)/np.diag(G0)))
R1, R1i, dead1, piv1 = block_chol(G1, np.diag(G0))
print("pass1 dead", dead1, "scaled pivots", np.array(piv1))
Q1 = W @ R1i
print("recon err pass1", np.linalg.norm(W - Q1 @ R1, axis=0) / np.linalg.norm(W0, axis=0))
T = Vp.T @ Q1; W2 = Q1 - Vp @ T
R2, R2i, dead2, piv2 = block_chol(W2.T @ W2)
print("pass2 dead", dead2, "scaled pivots", np.array(piv2))
Q2 = W2 @ R2i
print("GPU block2 live", live[12:18].tolist(), "max |Q2 - V_gpu| over live", np.abs(Q2[:, [k for k in range(6) if not dead2[k]]] - V[:, [12+k for k in range(6) if not dead2[k]]]).max())
H = H1 + T @ R1; Rt = R2 @ R1
rel = np.linalg.norm(W0 - Vp @ H - Q2 @ Rt, axis=0)/np.linalg.norm(W0, axis=0)
print("relation err per col (replay)", rel)
# what a rank-revealing SVD says about the pass-1 block
sv = np.linalg.svd(W / np.linalg.norm(W0, axis=0), compute_uv=False)
print("sv of W1 (normalized by |W0|)", sv)
