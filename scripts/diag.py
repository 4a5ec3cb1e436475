"""Developer diagnostics on the GPU box: per-problem stats and errors vs the oracle."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
from paper_1509_04567_b200 import build; build.build()
from paper_1509_04567_b200 import pexp

def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c4":
    for idx in [0, 1, 511]:
        p = synth.config4(indices=[idx], P=4, s=16)
        ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol)
        for rule in (0, 1):
            c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=256, stop_rule=rule)
            try:
                out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol)
                print(idx, "nu=%.2e a=%.2f" % (p.nu[0], p.a[0]), "rule", rule, "err %.2e" % rel(out.cpu().numpy(), ref), st, flush=True)
            except Exception as e:
                print(idx, "nu=%.2e a=%.2f" % (p.nu[0], p.a[0]), "rule", rule, "EXC", e, flush=True)
elif which == "c2":
    p = synth.config2()
    ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol, i_max=2)
    for rule in (0, 1):
        c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512, stop_rule=rule)
        try:
            t0 = time.time(); out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol); torch.cuda.synchronize()
            print("C2 rule", rule, "err(first 2) %.2e" % rel(out.cpu().numpy()[0, :2], ref[0]), st, "wall %.3f" % (time.time() - t0), flush=True)
        except Exception as e:
            print("C2 rule", rule, "EXC", e, flush=True)
