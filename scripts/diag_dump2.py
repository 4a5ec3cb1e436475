import sys, os, glob
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1509_04567_b200 import pexp
from oracle.operators import ade_matrix
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
p = synth.config4(indices=[0], P=16, s=32); dT=p.T/p.P; j=13
for f in glob.glob("/tmp/pe_K*.bin"): os.remove(f)
os.environ["PEXP_DUMP"] = "/tmp/pe"
src = p.src[:, j:j+1].copy()
c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512)
out, st = c.solve_linear(t(p.u0), t(src), dT, 1, p.tol)
gam = dT / 10
A = ade_matrix(p.n,p.bc,p.nu[0],p.a[0]).toarray(); M = np.eye(p.n) - gam*A
f = "/tmp/pe_K12.bin"
raw = open(f, "rb").read()
n, kcap, K, m, nout = np.frombuffer(raw[:20], np.int32)
o = 20
live = np.frombuffer(raw[o:o+4*kcap], np.int32); o += 4*kcap
V = np.frombuffer(raw[o:o+8*kcap*n], np.float64).reshape(kcap, n).T; o += 8*kcap*n
H = np.frombuffer(raw[o:o+8*kcap*kcap], np.float64).reshape(kcap, kcap).T
print("live[:18]", live[:18].tolist())
idx = np.where(live[:K+m] > 0)[0]
for cidx in range(K):
    if not live[cidx]: continue
    bv = np.linalg.solve(M, V[:, cidx])
    rec = V[:, :K+m] @ H[:K+m, cidx]
    coef_true = V[:, :K+m].T @ bv
    print(cidx, "relerr %.2e" % (np.linalg.norm(bv - rec)/np.linalg.norm(bv)),
          "H vs true proj max diff %.2e" % np.abs(H[:K+m, cidx] - coef_true * (live[:K+m] > 0)).max(),
          "resid outside span %.2e" % (np.linalg.norm(bv - V[:, idx] @ (V[:, idx].T @ bv))/np.linalg.norm(bv)))
