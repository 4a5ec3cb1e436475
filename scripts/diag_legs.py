import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1509_04567_b200 import pexp
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
p = synth.config2(n=1200, P=16, T=0.25, s=64)
c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512)
out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol)
ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol)
print(st, "err", np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref))
