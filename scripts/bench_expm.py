import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_04567_b200 import pexp
c = pexp.Context(16, "periodic", 1e-2, 1.0)
for E, N in [(64, 64), (64, 128), (64, 246), (148, 246)]:
    r = np.random.default_rng(0)
    A = torch.tensor(r.standard_normal((E, N, N)) * 3.0 / np.sqrt(N), device="cuda")
    c.expm_batched(A); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c.expm_batched(A); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    fl = E * (12 + 2.7) * 2 * N**3 / 2   # ~ (6 GEMMs + solve) flops, 2 flops/FMA counted once
    print(f"E={E} N={N}: {ms:.2f} ms, ~{E*22*N**3/ms/1e9:.2f} TFLOP/s (22N^3 model)", flush=True)
