"""Error vs oracle and Krylov size as a function of stop_factor (eta = stop_factor*tol)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1509_04567_b200 import pexp
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
cases = {
  "C1": (synth.config1(), {}),
  "C2red": (synth.config2(n=1200, P=16, T=0.25, s=64), {}),
  "C2full": (synth.config2(), {"i_max": 2}),
  "gen_per": (synth.generic_linear(n=777, nu=5e-3, a=1.3, P=5, s=12, T=0.5, seed=7), {}),
  "gen_dir": (synth.generic_linear(n=600, bc="dirichlet", nu=1e-3, a=1.0, P=5, s=12, T=0.5, seed=7), {}),
  "C4sub": (synth.config4(indices=[0, 1, 511], P=16, s=32), {}),
}
for name, (p, kw) in cases.items():
    ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol, **kw)
    for sf in (0.01, 0.1, 1.0):
        c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=512, stop_factor=sf)
        out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol)
        o = out.cpu().numpy()
        if "i_max" in kw: o = o[:, :kw["i_max"]]
        print(f"{name:8s} sf={sf:5.2f} err={rel(o, ref):.2e} max_k={st['max_k']} ms={st['ms_total']:.1f}", flush=True)
for sf in (0.01, 1.0):
    p = synth.config3()
    ref, info = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, p.P, p.s, p.tol, return_info=True)
    c = pexp.Context(p.n, "periodic", p.nu, 0.0, s=p.s, k_max=512, stop_factor=sf)
    out, st = c.solve_burgers(t(p.u0), p.nu, p.T, p.P, p.tol, 30)
    print(f"C3       sf={sf:5.2f} err={rel(out.cpu().numpy(), ref):.2e} max_k={st['max_k']} iters={st['wr_iters']}/{info['iters']} ms={st['ms_total']:.1f}", flush=True)
