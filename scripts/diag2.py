import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1509_04567_b200 import pexp
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
which = sys.argv[1]
if which == "c4":
    p = synth.config4(indices=[0], P=4, s=16)
    c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=256)
else:
    p = synth.config2()
    c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512)
try:
    out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol); print(st)
except Exception as e:
    print("EXC", e)
