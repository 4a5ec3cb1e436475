import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1509_04567_b200 import pexp
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
p = synth.config4(indices=[0], P=16, s=32)
dT = p.T / p.P
c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512)
for j in range(p.P):
    src = p.src[:, j:j+1].copy()
    ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, src, dT, 1, p.s, p.tol)
    out, st = c.solve_linear(t(p.u0), t(src), dT, 1, p.tol)
    o = out.cpu().numpy()
    print(j, "nonhom err %.2e" % rel(o - p.u0[:, None], ref - p.u0[:, None]), "max_k", st["max_k"], "m", st["max_m"], flush=True)
# homogeneous: zero source, u0 -> exp(T A) u0 via P subintervals (legs carry everything)
src0 = np.zeros_like(p.src)
ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, src0, p.T, p.P, p.s, p.tol)
out, st = c.solve_linear(t(p.u0), t(src0), p.T, p.P, p.tol)
print("unforced P=16 err", rel(out.cpu().numpy(), ref), st)
