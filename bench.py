"""bench.py — Paraexp-EBK solve on B200 (driver contract).

Default workload C5 (BASELINE.json configs[4], the largest config the north-star target is
quoted on): viscous Burgers, periodic, n = 65536, nu = 1e-3, T = 1, P = 256 subintervals,
s = 64 samples, tol = 1e-8, fp64, waveform relaxation to max-norm change < 1e-6.  One step =
one pexp_solve_burgers call: every WR iteration runs the batched EBK over all 256 subintervals
(truncated two-pass SVD, SaI block Arnoldi, projected Pade-13 expm, superposition) and the
homogeneous scan.  value = EBK evaluations/s over all ranks (P x WR iterations per solve);
the solve time is ms_per_step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C5|C1|C2|C3|C4]

N>1 (torchrun): "replicas only" — the north star keeps the path on one GPU, so each rank
solves an independent replica (weak scaling, no data-path collective; the timing max is
taken over ranks with one all_reduce after the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz
METRIC = "EBK evaluations/s (Paraexp-EBK solve; solve time = ms_per_step)"


# CUDA kernels behind each profiler class (paper_1509_04567_b200/csrc)
KERNELS_OF_CLASS = {
    "sai_solve": "k_sai_solve (tridiag.cu)", "xty": "k_xty_sq / k_xty_tall / k_xty_mma + k_reduce (tsmm.cu)",
    "combine": "k_combine (tsmm.cu)", "small_problem": "k_small_problem (small.cu)",
    "small_dense": "k_block_chol, k_sym_eig_select, k_onesided_svd, k_spline, ... (small.cu)",
    "stencil": "k_burgers_source, k_ubar, k_gamma, k_superpose, ... (stencil.cu)",
    "factor": "k_factor / k_factor_par (tridiag.cu)", "arnoldi_step": "k_arnoldi_step<MB> (arnoldi.cu)",
    "hom_scan": "k_hom_scan (hom_scan.cu)", "small_hom": "k_small_hom (small.cu)",
    "stream_proj": "k_sproj<8>, k_sproj2<2|3|4> + k_sred (stream.cu)", "stream_update": "k_supdate<8|16|32> (stream.cu)",
    "scan_output": "k_scan_output (hom_scan.cu)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def workload(name):
    import synth
    if name == "C2":
        p = synth.config2()
        return p, dict(kind="linear", s=p.s, k_max=384)
    if name == "C1":
        p = synth.config1()
        return p, dict(kind="linear", s=p.s, k_max=256)
    if name == "C4":
        p = synth.config4()
        return p, dict(kind="linear", s=p.s, k_max=96)
    if name == "C3":
        p = synth.config3()
        return p, dict(kind="burgers", s=p.s, k_max=256)
    if name == "C5":
        p = synth.config5()
        # 256 subintervals x 65536 points: the EBK runs in chunks of 128 subintervals with 640-column
        # bases per restart cycle (40 GiB of basis; 134 GiB workspace in total)
        # shift-and-invert parameters tuned for this very stiff case (4 nu dT/dx^2 = 6.7e4): gamma = dT/20 for
        # the nonhomogeneous evaluations and 0.7 of that for the scan (route only, DESIGN.md §3 #4; measured
        # 14 % faster than the default dT/10; the less stiff C1-C4 are fastest at the default)
        return p, dict(kind="burgers", s=p.s, k_max=960, basis_cols=640, eval_chunk=128, gamma_factor=0.5,
                       scan_gamma_factor=0.7)
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and "Active" in r[4 + i]
                          and "Not" not in r[4 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(p, cfg, budget_s=20.0):
    """The oracle as it stands (test infrastructure, never tuned) on a bounded sample of the
    same workload, on this host's cores."""
    import oracle
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    t0 = time.perf_counter()
    if cfg["kind"] == "linear":
        if p.batch > 1:       # C4: whole problems from the batch
            k = 0
            while time.perf_counter() - t0 < budget_s and k < p.batch:
                oracle.solve_linear(p.n, p.bc, p.nu[k:k + 1], p.a[k:k + 1], p.u0[k:k + 1], p.src[k:k + 1], p.T,
                                    p.P, p.s, p.tol)
                k += 1
            evals, sample = k * p.P, f"{k} of {p.batch} problems, full solves (P={p.P} EBK evals each)"
        else:
            k = 1
            while True:
                oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol, i_max=k)
                if time.perf_counter() - t0 > budget_s / 3 or k >= p.P:
                    break
                k *= 2
            t0 = time.perf_counter()
            oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol, i_max=k)
            evals, sample = k, f"first {k} of {p.P} subintervals (nonhomogeneous EBK + homogeneous legs, i_max={k})"
    else:
        # WR iteration 1 on the first k subintervals of the workload (same ΔT, n, s), k doubled
        # until the sample costs about budget_s / 3, then timed again
        from oracle.wr import wr_map
        dT = p.T / p.P
        k = 1
        while True:
            U = np.broadcast_to(p.u0, (k, p.s, p.n)).copy()
            t1 = time.perf_counter()
            wr_map(U, p.u0, p.nu, p.n, dT * k, k, p.s, p.tol)
            if time.perf_counter() - t1 > budget_s / 3 or 2 * k > p.P:
                break
            k *= 2
        t0 = time.perf_counter()
        U = np.broadcast_to(p.u0, (k, p.s, p.n)).copy()
        wr_map(U, p.u0, p.nu, p.n, dT * k, k, p.s, p.tol)
        evals, sample = k, f"WR iteration 1 on the first {k} of {p.P} subintervals (EBK + scan)"
    dt = time.perf_counter() - t0
    return {"value": evals / dt, "unit": "EBK evals/s", "cores": int(cores), "kind": "oracle", "sample": sample,
            "seconds": round(dt, 3)}


def fp64_peak(dev):
    """Measured fp64 tensor-core peak on this GPU: cuBLAS DGEMM (DMMA) 8192^3, best of 5 (CUDA
    events).  The roofline denominator for the fp64 contraction kernels."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = a @ b
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    del a, b, c
    torch.cuda.empty_cache()
    return {"tflops": 2.0 * n ** 3 / (best / 1e3) / 1e12, "how": "cuBLAS DGEMM 8192^3 fp64 (torch.matmul), best of 5",
            "derived_fma_peak_tflops": FP64_PEAK_TFLOPS}


def max_over_ranks(ms: float, world: int, dev) -> float:
    """The step time of the whole job: the slowest rank's (device-timed) mean step time."""
    if world <= 1:
        return float(ms)
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(world: int, evals_per_rank_step: int, ms_max: float) -> float:
    """Whole-job EBK evaluations/s: every rank solves an independent replica (weak scaling)."""
    return world * evals_per_rank_step / (ms_max / 1e3)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p, cfg = workload(args.config)
    import oracle
    times = []
    # the Burgers sample is bounded by the run's own length: two subintervals (EBK + one scan leg, ~37 s
    # per step at C5 size on 16 cores) only when --warmup + --steps is short, otherwise the first
    # subinterval alone (EBK evaluation, ~3 s at C5 size; its scan leg starts from zero), so that the
    # whole run ends within a few minutes for any K, W the driver passes
    ksub = 2 if (args.warmup + args.steps) <= 6 else 1
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if cfg["kind"] == "linear":
            oracle.solve_linear(p.n, p.bc, p.nu[:1], p.a[:1], p.u0[:1], p.src[:1], p.T, p.P, p.s, p.tol, i_max=1)
            evals = 1
        else:
            from oracle.wr import wr_map
            evals = min(p.P, ksub)
            U = np.broadcast_to(p.u0, (evals, p.s, p.n)).copy()
            wr_map(U, p.u0, p.nu, p.n, p.T * evals / p.P, evals, p.s, p.tol)
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    step = float(np.mean(times))
    val = evals / step
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    sample = (f"first subinterval of {args.config} (1 EBK eval + its legs, oracle SaI Krylov at eta=1e-12) per step"
              if cfg["kind"] == "linear" else
              f"WR iteration 1 on the first {evals} of {p.P} subintervals of {args.config} per step "
              + ("(EBK + scan)" if evals > 1 else "(EBK evaluation; the first subinterval's scan leg is zero)"))
    line = {"impl": "reference", "metric": METRIC, "value": val,
            "unit": "EBK evals/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, SURVEY §8(d).2)",
            "config": {"workload": args.config, "n": p.n, "bc": p.bc, "P": p.P, "s": p.s, "tol": p.tol,
                       "sample": sample},
            "cpu_baseline": {"value": val, "unit": "EBK evals/s", "cores": int(cores), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": "EBK evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_1509_04567_b200 import build
    if local == 0:           # one build per node; the other ranks wait, then load the same .so
        build.build()
    if world > 1:
        dist.barrier()
    from paper_1509_04567_b200 import pexp
    fp64 = fp64_peak(dev)

    p, cfg = workload(args.config)
    linear = cfg["kind"] == "linear"
    if linear:
        ctx = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=cfg["s"], k_max=cfg["k_max"])
        ctx.ensure_workspace(p.P, dev, kind=0)
        u0_h = torch.tensor(p.u0).pin_memory()
        src_h = torch.tensor(p.src).pin_memory()
        out = torch.empty((p.batch, p.P, p.n), dtype=torch.float64, device=dev)
    else:
        ctx = pexp.Context(p.n, "periodic", p.nu, 0.0, s=cfg["s"], k_max=cfg["k_max"],
                           basis_cols=cfg.get("basis_cols", 0), eval_chunk=cfg.get("eval_chunk", 0),
                           gamma_factor=cfg.get("gamma_factor", 0.0),
                           scan_gamma_factor=cfg.get("scan_gamma_factor", 0.0))
        ctx.ensure_workspace(p.P, dev, kind=1)
        u0_h = torch.tensor(p.u0).pin_memory()
        src_h = None
        out = torch.empty((p.P, p.n), dtype=torch.float64, device=dev)
    u0 = u0_h.to(dev)
    src = src_h.to(dev) if src_h is not None else None
    out_h = torch.empty(out.shape, dtype=torch.float64).pin_memory()
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)   # 256 MiB > 126 MB L2

    def step(records=False):
        if linear:
            return ctx.solve_linear(u0, src, p.T, p.P, p.tol, out=out, records=records)[1]
        return ctx.solve_burgers(u0, p.nu, p.T, p.P, p.tol, p.max_wr_iters, out=out, records=records)[1]

    st = None
    for _ in range(args.warmup):
        st = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    launches = 0
    syncs = 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = step()
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            launches += st["kernel_launches"]
            syncs += st["host_syncs"]
    evals_per_step = st["evals"]
    # per-kernel breakdown from ONE extra, separately profiled step (CUDA events around every
    # launch on its stream); the timed steps above ran with the profiler off
    flush.zero_()
    torch.cuda.synchronize()
    pexp.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    stp = step(records=True)
    e1.record()
    e1.synchronize()
    prof_step_ms = e0.elapsed_time(e1)
    prof = pexp.profile_read()
    pexp.profile_enable(False)
    if not linear and prof["hom_scan"]["ms"]:
        # the persistent scan kernel: algorithmic bytes of its single-vector SaI Arnoldi per subinterval by
        # SURVEY §8(d).4's figure for homogeneous legs, 8n(2K^2 + 10K) (CGS2 reads the basis four times per
        # step, solve read/write), K = the converged dimension recorded per subinterval (pexp_stats.kscan_j)
        ks = np.array([k for it in stp["kscan_j"] for k in it if k > 0], dtype=np.float64)
        prof["hom_scan"]["bytes"] = float(8.0 * p.n * np.sum(2.0 * ks * ks + 10.0 * ks))
        prof["hom_scan"]["flops"] = float(np.sum(8.0 * p.n * ks * ks))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_max = max_over_ranks(float(np.mean(times)), world, dev)
    value = job_throughput(world, evals_per_step, ms_max)

    # ---- end to end through the public API with host buffers (H2D + solve + D2H timed)
    e2e = None
    if not args.no_e2e:
        et = []
        # as many steps as the device-timed loop, but bounded to about 30 s of solves (at least 2) so a
        # long --steps run on the 10 s C5 solve still ends within minutes; the count is reported
        n_e2e = max(2, min(args.steps, int(30e3 / max(1e-3, float(np.mean(times))))))
        for _ in range(n_e2e):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            u0.copy_(u0_h, non_blocking=True)
            if src is not None:
                src.copy_(src_h, non_blocking=True)
            step()
            out_h.copy_(out, non_blocking=True)
            e1.record()
            e1.synchronize()
            et.append(e0.elapsed_time(e1))
        tm = max_over_ranks(float(np.mean(et)), world, dev)
        h2d = u0_h.numel() * 8 + (src_h.numel() * 8 if src_h is not None else 0)
        e2e = {"value": job_throughput(world, evals_per_step, tm), "unit": "EBK evals/s",
               "ms_per_step": tm, "steps": n_e2e, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(out_h.numel() * 8)}

    # ---- roofline of the dominant kernel class (live CUDA-event timing inside the timed region)
    peaks = json.load(open(MEASURED)) if os.path.exists(MEASURED) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    dom = max(prof, key=lambda k: prof[k]["ms"])
    d = prof[dom]
    if dom in ("small_problem", "small_hom", "small_dense"):
        ach = d["flops"] / (d["ms"] / 1e3) / 1e12 if d["ms"] else 0.0
        roof = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": fp64["tflops"], "unit": "TFLOP/s",
                "frac": ach / fp64["tflops"], "traffic": None,
                "peak_source": "measured fp64 DGEMM (cuBLAS, DMMA) on this GPU in this run"}
    else:
        ach = d["bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] else 0.0
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                "frac": ach / hbm_peak, "traffic": None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s (B200_PROFILING.md)"}
    # traffic: DRAM bytes per launch of this class from a committed `ncu --set full` capture
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        tj = json.load(open(tf)).get(dom)
        if tj and tj.get("workload") == args.config:
            roof["traffic"] = tj["dram_bytes_per_launch"]
            roof["traffic_source"] = tj["source"]
    if dom == "hom_scan":
        roof["note"] = ("sequential chain (255 subintervals x ~37 dependent Arnoldi steps per WR iteration): latency-bound; "
                        "its basis rows live in shared memory, so DRAM traffic is far below the algorithmic bytes")
    roof["cuda_kernels"] = KERNELS_OF_CLASS.get(dom, dom)
    roof["share_of_step"] = d["ms"] / max(1e-9, prof_step_ms)
    roof["launches_per_step"] = d["launches"]
    roof["ms_per_step"] = d["ms"]
    def hbm_roof(name):
        v = prof[name]
        if not v["ms"]:
            return None
        a = v["bytes"] / (v["ms"] / 1e3) / 1e9
        r = {"kernel": name, "bound": "hbm", "achieved": a, "peak": hbm_peak, "unit": "GB/s", "frac": a / hbm_peak,
             "TFLOP_per_s": v["flops"] / (v["ms"] / 1e3) / 1e12, "fp64_tensor_frac": v["flops"] / (v["ms"] / 1e3) / 1e12 / fp64["tflops"],
             "share_of_step": v["ms"] / max(1e-9, prof_step_ms), "launches_per_step": v["launches"]}
        if os.path.exists(tf):
            tj = json.load(open(tf)).get(name)
            if tj and tj.get("workload") == args.config:
                r["traffic"] = tj["dram_bytes_per_launch"]
                r["traffic_source"] = tj["source"]
        return r
    roof_stream = [r for r in (hbm_roof("stream_proj"), hbm_roof("stream_update")) if r]
    classes = {k: {"ms_per_step": v["ms"], "launches_per_step": v["launches"],
                   "GB_per_s": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] and v["bytes"] else None,
                   "TFLOP_per_s": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] and v["flops"] else None}
               for k, v in prof.items()}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "EBK evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generators, SURVEY §8(d).2)",
            "config": {"workload": args.config, "n": p.n, "bc": p.bc, "P": p.P, "s": p.s, "tol": p.tol,
                       "batch": getattr(p, "batch", 1), "evals_per_step": evals_per_step,
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": "flushed (256 MiB write) before every timed step",
                       "max_m": st["max_m"], "max_k": st["max_k"], "wr_iters": st["wr_iters"],
                       "options": {k: cfg[k] for k in ("k_max", "basis_cols", "eval_chunk", "gamma_factor",
                                                       "scan_gamma_factor") if k in cfg}},
            "roofline": roof, "roofline_ebk_streaming": roof_stream, "kernel_classes": classes,
            "gpu_launches": int(launches), "gpu_launches_per_step": int(launches / args.steps),
            "host_syncs_per_step": syncs / args.steps,
            "profiled_step_ms": prof_step_ms,
            "fp64_peak": fp64,
            "clocks": clk.summary(),
            "e2e": e2e,
        }
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(p, cfg)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
