"""Developer tool: one solve of a workload with the live per-kernel profiler and the
per-evaluation records (pexp_stats m_j / k_j / gamma_j), printed as JSON.

    python scripts/run_profile.py C5 [--route 1] [--iters K]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1509_04567_b200 import build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", default="C5", nargs="?")
ap.add_argument("--route", type=int, default=0)
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--scan-gamma", type=float, default=0.0, help="pexp_options.scan_gamma_factor")
ap.add_argument("--gamma", type=float, default=0.0, help="pexp_options.gamma_factor")
ap.add_argument("--eval-chunk", type=int, default=0)
ap.add_argument("--basis-cols", type=int, default=0)
ap.add_argument("--plain-only", action="store_true", help="one plain solve (ncu target), no profiler pass")
a = ap.parse_args()
build.build()
from paper_1509_04567_b200 import pexp  # noqa: E402

p, cfg = bench.workload(a.config)
dev = torch.device("cuda")
kw = {k: cfg[k] for k in ("basis_cols", "eval_chunk") if k in cfg}
if a.eval_chunk:
    kw["eval_chunk"] = a.eval_chunk
if a.basis_cols:
    kw["basis_cols"] = a.basis_cols
if not a.gamma:
    a.gamma = cfg.get("gamma_factor", 0.0)
if not a.scan_gamma:
    a.scan_gamma = cfg.get("scan_gamma_factor", 0.0)
if cfg["kind"] == "linear":
    ctx = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=cfg["s"], k_max=cfg["k_max"], route=a.route,
                       gamma_factor=a.gamma, **kw)
    u0 = torch.tensor(p.u0, device=dev)
    src = torch.tensor(p.src, device=dev)
    run = lambda rec: ctx.solve_linear(u0, src, p.T, p.P, p.tol, records=rec)
else:
    ctx = pexp.Context(p.n, "periodic", p.nu, 0.0, s=cfg["s"], k_max=cfg["k_max"], route=a.route,
                       scan_gamma_factor=a.scan_gamma, gamma_factor=a.gamma, **kw)
    u0 = torch.tensor(p.u0, device=dev)
    its = a.iters or p.max_wr_iters
    run = lambda rec: ctx.solve_burgers(u0, p.nu, p.T, p.P, p.tol, its, records=rec)
for _ in range(a.repeat):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, st = run(False)
    torch.cuda.synchronize()
    print("plain solve", round(time.perf_counter() - t0, 3), "s", {k: st[k] for k in ("ms_total", "ms_hom", "wr_iters", "max_m", "max_k", "host_syncs", "kernel_launches", "scan_steps", "scan_checks", "scan_check_cycles")}, flush=True)
if a.plain_only:
    sys.exit(0)
pexp.profile_enable(True)
out, st = run(True)
prof = pexp.profile_read()
pexp.profile_enable(False)
res = {"stats": {k: v for k, v in st.items() if k not in ("m_j", "k_j", "gamma_j", "kscan_j")},
       "profile": {k: {"ms": round(v["ms"], 2), "launches": v["launches"],
                       "GBps": round(v["bytes"] / v["ms"] / 1e6, 1) if v["ms"] else None,
                       "TFps": round(v["flops"] / v["ms"] / 1e9, 3) if v["ms"] else None} for k, v in prof.items()}}
if cfg["kind"] == "burgers":
    res["per_iter"] = [{"m_mean": float(np.mean(m)), "m_max": int(max(m)), "k_mean": float(np.mean(k)),
                        "k_max": int(max(k)), "gamma_min": float(min(g)), "kscan_mean": float(np.mean(ks)),
                        "kscan_max": int(max(ks))}
                       for m, k, g, ks in zip(st["m_j"], st["k_j"], st["gamma_j"], st["kscan_j"])]
else:
    res["m"] = st["m_j"][:64]
    res["k"] = st["k_j"][:64]
print(json.dumps(res, indent=1))
