import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1509_04567_b200 import pexp
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
B = int(sys.argv[1])
p = synth.config4(indices=np.arange(B))
c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=128)
try:
    out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol); torch.cuda.synchronize()
    print("B", B, "ok", st, flush=True)
except Exception as e:
    print("B", B, "EXC", str(e)[:200], flush=True)
