import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1509_04567_b200 import pexp
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
p = synth.config4(indices=[0, 1, 511], P=16, s=32)
ref, info = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol, return_info=True)
print("oracle m per (b,j):", info["m"].tolist())
c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512)
out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol); o = out.cpu().numpy()
for b in range(3):
    print("batched b", b, "err", rel(o[b], ref[b]), "per-i", [f"{rel(o[b,i], ref[b,i]):.1e}" for i in range(p.P)])
for b in range(3):
    c1 = pexp.Context(p.n, p.bc, [p.nu[b]], [p.a[b]], s=p.s, k_max=512)
    o1, st1 = c1.solve_linear(t(p.u0[b:b+1]), t(p.src[b:b+1]), p.T, p.P, p.tol)
    print("single b", b, "err", rel(o1.cpu().numpy()[0], ref[b]), st1["max_m"], st1["max_k"])
# stage check: source SVD per subinterval vs numpy
A = [oracle.ade_matrix(p.n, p.bc, p.nu[b], p.a[b]) for b in range(3)]
G = np.stack([(A[b] @ p.u0[b])[None, :] + p.src[b, j] for b in range(3) for j in range(p.P)])
m, sig, proj = c.source_svd(t(G), p.tol)
print("gpu m:", m)
