"""f1: the paper's parallel-efficiency study (Table 1)
on one B200 through the C ABI.

Workload: Eq.(ade) with the travelling pulses Eq.(manusol): n = 1000, a = 1, nu = 1e-2,
tol = 1e-4, retained rank m = 2, T = P * 0.5 (tau_0 grows in proportion to P in Table 1), s = 64
samples per subinterval (the paper's 100 exceed the library's s <= 64).

Per P in {2, 4, 8, 16, 32}:
  serial   tau_0 : the serial PEBK march -- P successive single-subinterval solves (P = 1 each,
                   u0 := the previous end value), device time summed (CUDA events in pexp_stats);
  parallel tau_1 : nonhomogeneous parts of ALL P subintervals in one batched call (pexp_stats.ms_nonhom)
           tau_2 : homogeneous legs + superposition (pexp_stats.ms_hom)
  speedup = tau_0 / (tau_1 + tau_2), efficiency = speedup / P  (the paper emulates
  P processors on a serial machine by timing each subproblem, here the P subproblems really run
  concurrently on one GPU, so "efficiency" is the fraction of the ideal P-fold gain one GPU delivers).
Errors: relative l2 error Eq.(relerr) at t = T against the exact PDE solution.
Every number is the median of --repeat runs after one warm-up.  Prints one JSON object.

    python scripts/f1_efficiency.py [--repeat 5] [--check-oracle]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1509_04567_b200 import build  # noqa: E402

build.build()
from paper_1509_04567_b200 import pexp  # noqa: E402
import synth  # noqa: E402

# Table 1, PEBK rows: P, tau_0, serial error, max tau_1, max tau_2, parallel error, efficiency %
TABLE1 = {2: (1.43, 3.05e-4, 7.22e-1, 6.44e-2, 2.70e-4, 91), 4: (2.81, 3.05e-4, 7.23e-1, 7.06e-2, 2.68e-4, 89),
          8: (5.59, 3.05e-4, 7.40e-1, 6.21e-2, 2.88e-4, 87), 16: (11.4, 3.05e-4, 7.30e-1, 6.28e-2, 3.22e-4, 90),
          32: (22.7, 3.05e-4, 7.33e-1, 6.63e-2, 3.65e-4, 89)}

ap = argparse.ArgumentParser()
ap.add_argument("--repeat", type=int, default=5)
ap.add_argument("--check-oracle", action="store_true", help="also compare the P = 2, 8 results with the oracle (CPU)")
a = ap.parse_args()
dev = torch.device("cuda")


def t(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=dev)


def relerr(u, ue):
    return float(np.linalg.norm(u - ue) / np.linalg.norm(ue))


rows = []
for P in (2, 4, 8, 16, 32):
    p = synth.pulse_ade(P=P, s=64, tol=1e-4)
    x = synth.grid_x(p.n, p.bc)
    ue = synth.pulse_exact(x, p.T)
    u0, src = t(p.u0), t(p.src)
    cpar = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=256)
    cser = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=256)
    srcs = [src[:, j:j + 1].contiguous() for j in range(P)]
    tau0, tau1, tau2, tot = [], [], [], []
    for it in range(a.repeat + 1):
        out, st = cpar.solve_linear(u0, src, p.T, P, p.tol, records=(it == 0))
        if it == 0:
            m_par = sorted(set(st["m_j"]))
            k_par = max(st["k_j"])
        # serial march
        u = u0
        ms = 0.0
        for j in range(P):
            o1, s1 = cser.solve_linear(u, srcs[j], p.T / P, 1, p.tol)
            u = o1[:, 0].contiguous()
            ms += s1["ms_total"]
        if it > 0:
            tau0.append(ms)
            tau1.append(st["ms_nonhom"])
            tau2.append(st["ms_hom"])
            tot.append(st["ms_total"])
    e_par = relerr(out[0, -1].cpu().numpy(), ue)
    e_ser = relerr(u[0].cpu().numpy(), ue)
    t0, t1, t2 = float(np.median(tau0)), float(np.median(tau1)), float(np.median(tau2))
    row = {"P": P, "T": p.T, "tau0_ms": t0, "tau1_ms": t1, "tau2_ms": t2, "err_serial": e_ser, "err_parallel": e_par,
           "speedup": t0 / (t1 + t2), "efficiency_pct": 100.0 * t0 / (t1 + t2) / P, "m": m_par, "k_max": k_par,
           "evals_per_s_parallel": P / (float(np.median(tot)) / 1e3),
           "paper_table1": dict(zip(("tau0_s", "err_serial", "tau1_s", "tau2_s", "err_parallel", "efficiency_pct"),
                                    TABLE1[P]))}
    if a.check_oracle and P in (2, 8):
        import oracle
        ref = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol)
        row["rel_vs_oracle"] = relerr(out.cpu().numpy(), ref)
    rows.append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
print(json.dumps({"workload": "F1 travelling-pulse ADE (PAPER.md:555-565), n=1000, s=64, tol=1e-4, T=0.5P",
                  "gpu": torch.cuda.get_device_name(0), "repeat": a.repeat, "rows": rows,
                  "paper_hardware": "not named in the paper (MATLAB, serial machine, emulated processors; P:571)"}))
