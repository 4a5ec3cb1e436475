import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1509_04567_b200 import pexp
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for P in (2, 3, 5, 9):
    p = synth.generic_linear(n=300, bc="dirichlet", nu=1e-3, a=1.0, P=P, s=8, T=0.1 * P, seed=3)
    c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=256)
    out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol)
    ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol)
    o = out.cpu().numpy()
    print("P", P, "err", "%.2e" % rel(o, ref), "per-i", ["%.1e" % rel(o[0, i], ref[0, i]) for i in range(P)], st["max_k"], flush=True)
