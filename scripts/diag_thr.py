import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1509_04567_b200 import pexp
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for name, p in [("C1", synth.config1()), ("C4sub", synth.config4(indices=[0, 1, 511], P=16, s=32))]:
    ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol)
    c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512, stop_factor=0.1)
    out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol)
    print(name, os.environ.get("PEXP_PIVTOL"), os.environ.get("PEXP_DEFL"), "err %.2e" % rel(out.cpu().numpy(), ref), "k", st["max_k"], flush=True)
