"""Write the stored oracle references used by the GPU parity tests (tests/golden/*.npz).

Test infrastructure only: this script imports ONLY `oracle/` (the method) and `synth/` (the
seeded inputs); nothing here touches the CUDA path.  Re-run it to regenerate a reference:

    python scripts/gen_oracle_refs.py c5proxy   # C5-shaped Burgers WR to convergence (~30-60 min)
    python scripts/gen_oracle_refs.py c2full    # C2 at full size, all 64 outputs (~15 min)

c5proxy: SURVEY.md §8(d).2 C5 generator (seed 5, ν = 1e-3, s = 64, tol = 1e-8) at n = 8192 with
ΔT = 1/256 and T = 0.25 (P = 64): the front forms inside the window (SURVEY A.3 shows the ν = 1e-3
front is already resolved at n = 8192, the trajectory equal to the full n = 65536 one), so the WR
iterations that carry m up to ~25 and the steep per-subinterval Jacobians are all in it.
c2full: BASELINE configs[1] exactly (synth.config2()), every output u(T_1..T_64).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def c5proxy():
    p = synth.config5(n=8192, P=64, T=0.25)
    t0 = time.time()
    out, info = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, p.P, p.s, p.tol, max_wr_iters=30,
                                     return_info=True)
    dt = time.time() - t0
    m = np.asarray(info["m"], dtype=np.int32).reshape(info["iters"], p.P)
    np.savez_compressed(os.path.join(GOLD, "c5proxy_oracle.npz"), out=out, m=m,
                        delta=np.asarray(info["delta"]), iters=np.int32(info["iters"]))
    meta = {"case": "c5proxy", "generator": "synth.config5(n=8192, P=64, T=0.25)",
            "oracle": "oracle.solve_burgers(..., max_wr_iters=30) eta=1e-12 Krylov branch (n > 1024)",
            "iters": info["iters"], "delta": info["delta"], "max_m_per_iter": m.max(axis=1).tolist(),
            "seconds": dt}
    with open(os.path.join(GOLD, "c5proxy_oracle.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta))


def c2full():
    p = synth.config2()
    t0 = time.time()
    out, info = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol,
                                    return_info=True)
    dt = time.time() - t0
    np.savez_compressed(os.path.join(GOLD, "c2full_oracle.npz"), out=out, m=info["m"], k=info["k"])
    meta = {"case": "c2full", "generator": "synth.config2()",
            "oracle": "oracle.solve_linear eta=1e-12 Krylov branch (n > 1024)",
            "m": info["m"][0].tolist(), "k": info["k"][0].tolist(), "seconds": dt}
    with open(os.path.join(GOLD, "c2full_oracle.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta))


if __name__ == "__main__":
    for name in sys.argv[1:]:
        {"c5proxy": c5proxy, "c2full": c2full}[name]()
