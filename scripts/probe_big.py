import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1509_04567_b200 import pexp
def t(x): return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")
which = sys.argv[1]
if which == "C4":
    p = synth.config4()
    c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=128)
    u0, src = t(p.u0), t(p.src)
    for it in range(2):
        t0 = time.time(); out, st = c.solve_linear(u0, src, p.T, p.P, p.tol); torch.cuda.synchronize()
        print("C4", st, "wall %.2f" % (time.time() - t0), flush=True)
else:
    p = synth.config5()
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    kmax = int(sys.argv[3]) if len(sys.argv) > 3 else 768
    bcols = int(sys.argv[4]) if len(sys.argv) > 4 else 256
    chunk = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    c = pexp.Context(p.n, "periodic", p.nu, 0.0, s=p.s, k_max=kmax, basis_cols=bcols, restart_blocks=-1,
                     eval_chunk=chunk)
    print("workspace GiB", c.workspace_bytes(p.P, 1) / 2**30, flush=True)
    t0 = time.time(); out, st = c.solve_burgers(t(p.u0), p.nu, p.T, p.P, p.tol, iters); torch.cuda.synchronize()
    print("C5", st, "wall %.2f" % (time.time() - t0), flush=True)
