import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1509_04567_b200 import pexp
from oracle.operators import ade_matrix
from oracle.lowrank import truncated_svd, notaknot_taylor
from tests.closed_forms import periodic_forced_solution
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
p = synth.config4(indices=[0], P=16, s=32); dT=p.T/p.P; h=dT/(p.s-1)
for j in (12, 13):
    src = p.src[:, j:j+1].copy()
    A = ade_matrix(p.n,p.bc,p.nu[0],p.a[0]); G=(A@p.u0[0])[:,None]+src[0,0].T
    U,C,sv = truncated_svd(G, 1e-10); coef = notaknot_taylor(C,h)
    Y = []
    for k in range(U.shape[1]):
        cpk = np.einsum("n,iq->iqn", U[:,k], coef[:,:,k])
        Y.append(periodic_forced_solution(p.n,p.nu[0],p.a[0],cpk,h)[-1])
    Y = np.array(Y).T
    yref = Y.sum(axis=1)
    c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512)
    out, st = c.solve_linear(t(p.u0), t(src), dT, 1, p.tol)
    yg = out.cpu().numpy()[0, 0] - p.u0[0]
    e = yg - yref
    coeffs, res, *_ = np.linalg.lstsq(Y, e, rcond=None)
    print("j", j, "err", np.linalg.norm(e)/np.linalg.norm(yref), "e = Y @", np.round(coeffs, 4).tolist(),
          "unexplained", np.linalg.norm(e - Y @ coeffs)/np.linalg.norm(yref))
