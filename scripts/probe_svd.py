import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_04567_b200 import pexp
for E in [int(x) for x in sys.argv[1:]]:
    r = np.random.default_rng(0)
    n, s = 1024, 32
    G = torch.tensor(r.standard_normal((E, s, 4)) @ r.standard_normal((4, n)), device="cuda")
    c = pexp.Context(n, "periodic", [1e-3] * 16, [1.0] * 16, s=s, k_max=128)
    try:
        m, sig, proj = c.source_svd(G, 1e-8); torch.cuda.synchronize()
        print("E", E, "ok", set(m), flush=True)
    except Exception as e:
        print("E", E, "EXC", str(e)[:160], flush=True)
        break
