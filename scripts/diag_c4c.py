import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1509_04567_b200 import pexp
from oracle.operators import ade_matrix
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
p = synth.config4(indices=[0], P=16, s=32)
dT = p.T / p.P; j = 13
A = ade_matrix(p.n, p.bc, p.nu[0], p.a[0])
G = (A @ p.u0[0])[None, :] + p.src[0, j]
U, C, sv = oracle.truncated_svd(G.T, 1e-10)
print("numpy sigma/sigma1:", (sv[:8] / sv[0]).tolist())
c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512)
m, sig, proj = c.source_svd(t(G[None]), p.tol)
sg = sig.cpu().numpy()[0]
print("gpu m", m, "sigma/sigma1:", (sg[:8] / sg[0]).tolist())
print("proj err", np.linalg.norm(proj.cpu().numpy()[0].T - U @ C) / sv[0])
src = p.src[:, j:j+1].copy()
ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, src, dT, 1, p.s, p.tol)
for rule in (0, 1):
    for tol in (1e-8, 1e-6):
        cc = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512, stop_rule=rule)
        out, st = cc.solve_linear(t(p.u0), t(src), dT, 1, tol)
        r2 = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, src, dT, 1, p.s, tol)
        print("rule", rule, "tol", tol, "err %.2e" % rel(out.cpu().numpy() - p.u0[:, None], r2 - p.u0[:, None]), "k", st["max_k"], "m", st["max_m"])
