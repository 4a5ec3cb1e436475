import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_04567_b200 import pexp
s = int(sys.argv[1])
for E in [int(x) for x in sys.argv[2:]]:
    r = np.random.default_rng(0)
    n = 1024
    G = torch.tensor(r.standard_normal((E, s, 4)) @ r.standard_normal((4, n)), device="cuda")
    c = pexp.Context(n, "periodic", [1e-3] * 16, [1.0] * 16, s=s, k_max=128)
    try:
        m, sig, proj = c.source_svd(G, 1e-8); torch.cuda.synchronize()
        print("s", s, "E", E, "ok", flush=True)
    except Exception as e:
        print("s", s, "E", E, "EXC", str(e)[-60:], flush=True)
        break
