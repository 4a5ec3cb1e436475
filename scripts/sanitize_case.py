"""Small solves for compute-sanitizer runs (one tool per gpurun call; logs under profiles/):

    compute-sanitizer --tool memcheck  python scripts/sanitize_case.py linear
    compute-sanitizer --tool racecheck python scripts/sanitize_case.py burgers
    compute-sanitizer --tool synccheck python scripts/sanitize_case.py linear

linear : C1 (fused cluster Arnoldi step, DSMEM reductions, cluster projected problems, grouped legs)
         and a generic Dirichlet problem on the streaming route (TMA ring + DMMA kernels, restart).
burgers: a Burgers WR solve with n = 2048 (8 scan workers + the checker CTA: the stamped exchanges,
         the cooperative scan, k_scan_output) on both Arnoldi routes, 3 WR iterations.
Each result is compared with a second run of itself (determinism up to the eta level) -- the oracle
comparison of the same cases is in tests/test_gpu_parity.py.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1509_04567_b200 import pexp  # noqa: E402
import synth  # noqa: E402

dev = "cuda"


def t(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=dev)


what = sys.argv[1] if len(sys.argv) > 1 else "linear"
if what == "linear":
    p = synth.config1()
    c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s)
    out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol)
    print("C1 fused", st["max_k"], st["kernel_launches"], float(out.abs().max()))
    q = synth.generic_linear(n=600, bc="dirichlet", nu=1e-3, a=1.0, P=3, s=12, T=0.3, seed=7)
    c2 = pexp.Context(q.n, q.bc, list(q.nu), list(q.a), s=q.s, k_max=512, route=1, restart_blocks=6)
    out2, st2 = c2.solve_linear(t(q.u0), t(q.src), q.T, q.P, q.tol)
    print("generic streaming", st2["max_k"], st2["restarts"], st2["kernel_launches"], float(out2.abs().max()))
else:
    p = synth.config3(n=2048, P=4, s=12, T=0.05)
    for route in (0, 1):
        c = pexp.Context(p.n, "periodic", p.nu, 0.0, s=p.s, route=route)
        out, st = c.solve_burgers(t(p.u0), p.nu, p.T, p.P, p.tol, 3)
        print("burgers route", route, st["wr_iters"], st["max_k"], st["kernel_launches"], st["delta_hist"])
torch.cuda.synchronize()
print("done")
