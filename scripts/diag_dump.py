import sys, os, glob
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1509_04567_b200 import pexp
from oracle.operators import ade_matrix
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
p = synth.config4(indices=[0], P=16, s=32); dT=p.T/p.P; j=int(sys.argv[1]) if len(sys.argv)>1 else 13
os.environ["PEXP_DUMP"] = "/tmp/pd"
src = p.src[:, j:j+1].copy()
c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512)
out, st = c.solve_linear(t(p.u0), t(src), dT, 1, p.tol)
gam = dT / 10
A = ade_matrix(p.n,p.bc,p.nu[0],p.a[0]).toarray(); M = np.eye(p.n) - gam*A
for f in sorted(glob.glob("/tmp/pd_K*.bin"), key=lambda x: int(x.split("_K")[1][:-4])):
    raw = open(f, "rb").read()
    n, kcap, K, m, nout = np.frombuffer(raw[:20], np.int32)
    o = 20
    live = np.frombuffer(raw[o:o+4*kcap], np.int32); o += 4*kcap
    V = np.frombuffer(raw[o:o+8*kcap*n], np.float64).reshape(kcap, n).T; o += 8*kcap*n
    H = np.frombuffer(raw[o:o+8*kcap*kcap], np.float64).reshape(kcap, kcap).T; o += 8*kcap*kcap
    idx = np.where(live[:K+m] > 0)[0]
    Vl = V[:, idx]
    orth = np.abs(Vl.T @ Vl - np.eye(len(idx))).max()
    cols = np.where(live[:K] > 0)[0]
    lhs = np.linalg.solve(M, V[:, cols])
    rhs = V[:, idx] @ H[np.ix_(idx, cols)]
    arn = np.linalg.norm(lhs - rhs, axis=0).max()
    print(f"K={K} live={len(idx)} orth={orth:.2e} arnoldi={arn:.2e} |H|={np.abs(H[:K+m,:K]).max():.2e}", flush=True)
