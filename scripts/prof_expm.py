"""Profile target: one batched Pade-13 expm launch (E=64, N=246) through the stage API."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_04567_b200 import pexp
E, N = int(os.environ.get("E", 64)), int(os.environ.get("N", 246))
c = pexp.Context(16, "periodic", 1e-2, 1.0)
r = np.random.default_rng(0)
A = torch.tensor(r.standard_normal((E, N, N)) * 3.0 / np.sqrt(N), device="cuda")
for _ in range(3):
    c.expm_batched(A)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); c.expm_batched(A); e1.record(); e1.synchronize()
print(f"E={E} N={N}: {e0.elapsed_time(e1):.3f} ms")
