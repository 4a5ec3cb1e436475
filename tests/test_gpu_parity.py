"""GPU parity: the CUDA path (through the C ABI) vs the oracle / library routines on the
same seeded inputs.  Tolerances: relative 2-norm 1e-8 for solves (BASELINE.json north_star);
stage tolerances from SURVEY.md §8(c).5 / DESIGN.md §7."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1509_04567_b200 import build  # noqa: E402

build.build()
from paper_1509_04567_b200 import pexp  # noqa: E402
import oracle  # noqa: E402
from oracle.operators import ade_matrix  # noqa: E402

DEV = "cuda"


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def t(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=DEV)


# ---------------------------------------------------------------- subsystem 1: SaI solves

@pytest.mark.parametrize("n,bc,nu,a,gamma", [
    (256, "periodic", 1e-2, 1.0, 1 / 80),
    (5000, "periodic", 1e-3, 1.0, 1 / 640),      # ragged: 2 full 2048-row chunks + tail
    (4096, "dirichlet", 1e-3, 1.0, 1 / 640),
    (1024, "periodic", 1e-4, 2.0, 1 / 160),      # C4 corner: cell Peclet ~20, M not dominant
    (6144, "periodic", 1e-5, 2.0, 1 / 160),      # parallel (Moebius-scan) factorisation, cell Peclet ~33
    (65536, "periodic", 1e-3, 0.3, 1 / 2560),    # C5-sized column, 32 tiles of the parallel factorisation
    (7, "dirichlet", 0.3, -1.0, 0.5),            # tiny
])
def test_sai_solve_vs_dense(n, bc, nu, a, gamma):
    import scipy.sparse as sp
    from scipy.sparse.linalg import splu
    r = np.random.default_rng(n)
    c = pexp.Context(n, bc, nu, a)
    B = r.standard_normal((5, n))
    X = c.sai_solve(0, gamma, t(B)).cpu().numpy()
    M = (sp.identity(n, format="csc") - gamma * ade_matrix(n, bc, nu, a)).tocsc()
    ref = splu(M).solve(B.T.copy()).T           # LAPACK-style sparse LU with pivoting
    assert rel(X, ref) < 1e-12
    # backward error: residual relative to ||M|| ||X|| (the scale of the rounding in M X)
    nM = abs(M).sum(axis=1).max()
    assert np.linalg.norm(M @ X.T - B.T) <= 1e-14 * nM * np.linalg.norm(X) + 1e-13 * np.linalg.norm(B)


# ---------------------------------------------------------------- subsystem 3: source SVD

def _svd_case(G, tol):
    c = pexp.Context(G.shape[2], "periodic", 1e-2, 1.0, s=G.shape[1])
    m, sig, proj = c.source_svd(t(G), tol)
    return m, sig.cpu().numpy(), proj.cpu().numpy()


def test_source_svd_config1_exact_rank():
    p = synth.config1()
    A = ade_matrix(p.n, p.bc, p.nu[0], p.a[0])
    G = np.stack([(A @ p.u0[0])[None, :] + p.src[0, j] for j in range(p.P)])  # [P][s][n]
    m, sig, proj = _svd_case(G, p.tol)
    for j in range(p.P):
        U, C, sv = oracle.truncated_svd(G[j].T, 0.01 * p.tol)
        assert m[j] == U.shape[1] == 4
        assert rel(proj[j].T, U @ C) < 1e-12
        np.testing.assert_allclose(sig[j][:4], sv[:4], rtol=1e-10)


def test_source_svd_noisy_no_gap():
    """C2-like spectrum: geometric decay, then a 1e-10 noise floor: the two-pass
    Gram SVD must find the same m as LAPACK and the same projection."""
    p = synth.config2(n=1500, P=3, s=64)
    G = p.src[0] + 0.0
    m, sig, proj = _svd_case(G, p.tol)
    for j in range(p.P):
        U, C, sv = oracle.truncated_svd(G[j].T, 0.01 * p.tol)
        assert m[j] == U.shape[1]
        assert np.linalg.norm(proj[j].T - U @ C) <= 1e-12 * sv[0]


def test_source_svd_zero_and_rank_one():
    n, s = 300, 9
    G = np.zeros((2, s, n))
    G[1] = np.outer(np.linspace(1, 2, s), np.sin(np.arange(n)))
    m, sig, proj = _svd_case(G, 1e-8)
    assert m == [0, 1]
    assert np.abs(proj[0]).max() == 0.0
    assert rel(proj[1], G[1]) < 1e-13


# ---------------------------------------------------------------- subsystem 4: batched expm

def test_expm_batched_vs_scipy():
    from scipy.linalg import expm
    r = np.random.default_rng(0)
    mats = [r.standard_normal((40, 40)) * s for s in (0.01, 1.0, 8.0)]
    mats.append(np.diag(-np.linspace(0, 300, 40)) + np.triu(r.standard_normal((40, 40)), 1))
    A = np.stack(mats)
    c = pexp.Context(16, "periodic", 1e-2, 1.0)
    X = c.expm_batched(t(A)).cpu().numpy()
    for k in range(len(mats)):
        ref = expm(A[k])
        assert rel(X[k], ref) < 1e-12, k


# ---------------------------------------------------------------- linear Paraexp-EBK solves

def _linear(p, k_max=256, records=False, **kw):
    c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=k_max, **kw)
    out, st = c.solve_linear(t(p.u0), t(p.src), p.T, p.P, p.tol, records=records)
    return out.cpu().numpy(), st


_ORACLE_MEMO = {}


def _memo_key(tag, p, kw, arrays):
    """Key of one oracle call: every scalar argument and a digest of every array argument."""
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return (tag, p.n, getattr(p, "bc", "periodic"), p.T, p.P, p.s, p.tol, tuple(sorted(kw.items())), h.hexdigest())


def _oracle_linear(p, **kw):
    """oracle.solve_linear, memoised per pytest process on its exact inputs: several tests compare
    different launch configurations of the CUDA path against the SAME oracle run (C2 reduced: ~170 s
    of CPU each), which is computed once.  Only oracle outputs are stored, keyed by oracle inputs."""
    want_info = kw.pop("return_info", False)
    key = _memo_key("linear", p, kw, (p.nu, p.a, p.u0, p.src))
    if key not in _ORACLE_MEMO:
        _ORACLE_MEMO[key] = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol,
                                                return_info=True, **kw)
    out, info = _ORACLE_MEMO[key]
    return (out, info) if want_info else out


def _oracle_burgers(p):
    """oracle.solve_burgers(..., return_info=True), memoised like _oracle_linear."""
    key = _memo_key("burgers", p, {}, ([p.nu], p.u0))
    if key not in _ORACLE_MEMO:
        _ORACLE_MEMO[key] = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, p.P, p.s, p.tol, return_info=True)
    return _ORACLE_MEMO[key]


ROUTES = [0, 1]  # pexp_options.route: 0 auto (fused cluster step where it fits), 1 streaming route


@pytest.mark.parametrize("route", ROUTES)
def test_linear_config1_full(route):
    p = synth.config1()
    out, st = _linear(p, route=route)
    ref = _oracle_linear(p)
    assert rel(out, ref) < 1e-8, st
    assert st["max_m"] == 4


@pytest.mark.parametrize("route", ROUTES)
@pytest.mark.parametrize("bc,n,nu,a", [("periodic", 777, 5e-3, 1.3), ("dirichlet", 600, 1e-3, 1.0)])
def test_linear_generic_deep_arnoldi(bc, n, nu, a, route):
    """Non-Fourier data: the Krylov space is not invariant; deep Arnoldi, ragged n."""
    p = synth.generic_linear(n=n, bc=bc, nu=nu, a=a, P=5, s=12, T=0.5, seed=7)
    out, st = _linear(p, route=route)
    ref = _oracle_linear(p)
    assert rel(out, ref) < 1e-8, st
    assert st["max_k"] > 20


@pytest.mark.parametrize("route", ROUTES)
def test_linear_config2_reduced(route):
    p = synth.config2(n=1200, P=16, T=0.25, s=64)     # same subinterval length dT = 1/64 as C2
    out, st = _linear(p, k_max=384, route=route)
    ref = _oracle_linear(p)
    assert rel(out, ref) < 1e-8, st


def test_linear_config4_subset():
    p = synth.config4(indices=[0, 1, 511], P=4, s=16)
    out, st = _linear(p, k_max=128)
    ref = _oracle_linear(p)
    for b in range(p.batch):
        assert rel(out[b], ref[b]) < 1e-8, (b, st)


def test_linear_config4_full_batch_sampled():
    """C4 at its full size (512 problems, one batched call, the bench's k_max); the oracle
    recomputes sampled problems, which are bit-identical rows of the full batch (synth streams)."""
    p = synth.config4()
    out, st = _linear(p, k_max=96)
    assert np.all(np.isfinite(out))
    for b in (0, 257, 511):
        q = synth.config4(indices=[b])
        ref = _oracle_linear(q)
        assert rel(out[b], ref[0]) < 1e-8, (b, st)


@pytest.mark.parametrize("route", ROUTES)
@pytest.mark.parametrize("restart_blocks,basis_cols", [(3, 0), (-1, 40), (20, 0)])
def test_linear_restart_nested_exact(restart_blocks, basis_cols, route):
    """Exact nested restart (DESIGN.md §3 #5): the cycle residual becomes the next cycle's
    source; the result must match the unrestarted oracle to the same 1e-8."""
    p = synth.generic_linear(n=777, bc="periodic", nu=5e-3, a=1.3, P=5, s=12, T=0.5, seed=7)
    out, st = _linear(p, k_max=512, restart_blocks=restart_blocks, basis_cols=basis_cols, route=route)
    ref = _oracle_linear(p)
    assert rel(out, ref) < 1e-8, st
    if restart_blocks != 20:
        assert st["restarts"] >= 1, st


def test_linear_config2_reduced_restarted():
    p = synth.config2(n=1200, P=16, T=0.25, s=64)
    out, st = _linear(p, k_max=512, restart_blocks=-1, basis_cols=72)
    ref = _oracle_linear(p)
    assert rel(out, ref) < 1e-8, st
    assert st["restarts"] >= 1, st


def test_linear_config2_reduced_chunked():
    """eval_chunk: the 16 subintervals run as EBK chunks 5, 5, 5, 1 sharing one basis buffer."""
    p = synth.config2(n=1200, P=16, T=0.25, s=64)
    out, st = _linear(p, k_max=384, eval_chunk=5)
    ref = _oracle_linear(p)
    assert rel(out, ref) < 1e-8, st


def test_linear_P1_and_unforced_and_zero():
    n = 300
    x = synth.grid_x(n, "periodic")
    u0 = np.exp(-((x - 0.5) / 0.08) ** 2)[None]
    src = np.zeros((1, 1, 6, n))
    c = pexp.Context(n, "periodic", 1e-2, 1.0, s=6)
    out, _ = c.solve_linear(t(u0), t(src), 1.0, 1, 1e-8)
    ref = oracle.solve_linear(n, "periodic", [1e-2], [1.0], u0, src, 1.0, 1, 6, 1e-8)
    assert rel(out.cpu().numpy(), ref) < 1e-8
    z, _ = c.solve_linear(t(np.zeros((1, n))), t(np.zeros((1, 3, 6, n))), 1.0, 3, 1e-8)
    assert torch.count_nonzero(z).item() == 0


def _golden(name):
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name)
    if not os.path.exists(path):
        pytest.fail(f"stored oracle reference {name} missing: run scripts/gen_oracle_refs.py")
    return np.load(path)


def test_linear_config2_full_size_all_outputs():
    """C2 at its full size (BASELINE configs[1]) in the bench's launch configuration: all 64
    outputs u(T_1..T_64) (every nonhomogeneous evaluation and all 8 homogeneous leg groups)
    against the stored oracle reference (tests/golden/c2full_oracle.npz, written by
    scripts/gen_oracle_refs.py, which calls only oracle/)."""
    p = synth.config2()
    out, st = _linear(p, k_max=384, records=True)
    ref = _golden("c2full_oracle.npz")
    assert rel(out, ref["out"]) < 1e-8, st
    for i in range(p.P):   # every output on its own, incl. the late legs of the last group
        assert rel(out[0, i], ref["out"][0, i]) < 1e-8, i
    assert st["m_j"] == ref["m"][0].tolist()     # retained ranks m_j equal the oracle's


@pytest.mark.parametrize("route", ROUTES)
@pytest.mark.parametrize("s,n,P,restart_blocks", [(20, 700, 4, 0), (20, 700, 4, 6), (40, 900, 3, 0)])
def test_linear_wide_blocks(s, n, P, restart_blocks, route):
    """Block widths 8 < m <= 32 and m > 32 (a rough 1e-6-noise source keeps every sample:
    m = s): the DMMA projections, the deferred-column in-block QR at m > 32 and nested restarts
    at wide blocks, on both Arnoldi routes."""
    p = synth.generic_linear(n=n, bc="periodic", nu=5e-3, a=1.3, P=P, s=s, T=0.5, seed=7, rank=3, noise=1e-6)
    out, st = _linear(p, k_max=880, restart_blocks=restart_blocks, route=route, records=True)
    ref, info = _oracle_linear(p, dense_max=0, return_info=True)
    assert st["m_j"] == info["m"][0].tolist() == [s] * P
    assert rel(out, ref) < 1e-8, st
    if restart_blocks:
        assert st["restarts"] >= 1, st


# ---------------------------------------------------------------- Burgers WR

def _burgers(p, k_max=256, records=False, **kw):
    c = pexp.Context(p.n, "periodic", p.nu, 0.0, s=p.s, k_max=k_max, **kw)
    out, st = c.solve_burgers(t(p.u0), p.nu, p.T, p.P, p.tol, p.max_wr_iters, records=records)
    return out.cpu().numpy(), st


@pytest.mark.parametrize("route", ROUTES)
def test_burgers_small(route):
    p = synth.config3(n=256, P=4, s=12, T=0.2, nu=0.02)
    out, st = _burgers(p, route=route)
    ref, info = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, p.P, p.s, p.tol, return_info=True)
    assert st["wr_iters"] == info["iters"], (st, info["delta"])
    assert rel(out, ref) < 1e-8, st
    assert abs(out.sum(axis=1) - p.u0.sum()).max() < 1e-9 * np.abs(p.u0).sum()


@pytest.mark.parametrize("route", ROUTES)
def test_burgers_config3_full(route):
    p = synth.config3()
    out, st = _burgers(p, route=route)
    ref, info = _oracle_burgers(p)
    assert st["wr_iters"] == info["iters"], (st, info["delta"])
    assert rel(out, ref) < 1e-8, st


@pytest.mark.parametrize("route", ROUTES)
def test_burgers_small_restarted(route):
    p = synth.config3(n=256, P=4, s=12, T=0.2, nu=0.02)
    out, st = _burgers(p, k_max=512, restart_blocks=-1, basis_cols=40, route=route)
    ref, info = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, p.P, p.s, p.tol, return_info=True)
    assert st["wr_iters"] == info["iters"], (st, info["delta"])
    assert rel(out, ref) < 1e-8, st
    assert st["restarts"] >= 1, st


# bench.py's launch configuration of C5 (bench.workload("C5")): capacities and the tuned shift parameters
C5_BENCH_OPTIONS = dict(k_max=960, basis_cols=640, eval_chunk=128, gamma_factor=0.5, scan_gamma_factor=0.7)


@pytest.mark.parametrize("route,tuned", [(0, False), (1, False), (1, True)])
def test_burgers_c5proxy_to_convergence(route, tuned):
    """C5-shaped WR run to convergence (SURVEY §8(d).2 C5 generator at n = 8192, ν = 1e-3,
    s = 64, ΔT = 1/256, T = 0.25): the steep front forms, block widths reach ~25 and the
    per-subinterval Jacobians differ, i.e. the iterations the C5 first-iterate check cannot
    see.  Reference: the oracle to convergence (tests/golden/c5proxy_oracle.npz, written by
    scripts/gen_oracle_refs.py); equal WR iteration counts and equal retained ranks m_j in
    every iteration."""
    p = synth.config5(n=8192, P=64, T=0.25)
    ref = _golden("c5proxy_oracle.npz")
    kw = dict(gamma_factor=0.5, scan_gamma_factor=0.7) if tuned else {}   # bench.py's C5 shift parameters
    c = pexp.Context(p.n, "periodic", p.nu, 0.0, s=p.s, k_max=960, route=route, **kw)
    out, st = c.solve_burgers(t(p.u0), p.nu, p.T, p.P, p.tol, p.max_wr_iters, records=True)
    out = out.cpu().numpy()
    assert st["wr_iters"] == int(ref["iters"]), (st["delta_hist"], ref["delta"])
    assert rel(out, ref["out"]) < 1e-8, st
    # retained ranks: equal except at threshold ties (reading #7: a sigma at tau*sigma_1 changes
    # the projection by <= tau), which may flip m_j by one in isolated subintervals
    K = st["wr_iters"]
    dm = np.abs(np.array(st["m_j"]) - ref["m"][:K])
    assert dm.max() <= 1 and (dm > 0).sum() <= max(2, dm.size // 100), np.argwhere(dm > 0)
    assert np.abs(out.sum(axis=1) - p.u0.sum()).max() < 1e-9 * np.abs(p.u0).sum()


def test_stats_records_linear():
    """pexp_stats per-evaluation records: m_j equal the oracle's ranks, k_j > 0, gamma_j = ΔT/10."""
    p = synth.config2(n=1200, P=16, T=0.25, s=64)
    out, st = _linear(p, k_max=384, records=True)
    ref, info = _oracle_linear(p, return_info=True)
    assert st["m_j"] == info["m"][0].tolist()
    assert min(st["k_j"]) > 0 and max(st["k_j"]) <= st["max_k"]
    assert np.allclose(st["gamma_j"], p.T / p.P / 10)
    assert st["host_syncs"] >= 1


def test_burgers_small_chunked():
    p = synth.config3(n=256, P=4, s=12, T=0.2, nu=0.02)
    out, st = _burgers(p, eval_chunk=3)
    ref, info = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, p.P, p.s, p.tol, return_info=True)
    assert st["wr_iters"] == info["iters"], (st, info["delta"])
    assert rel(out, ref) < 1e-8, st


def test_burgers_config5_full_size_first_iterate():
    """C5 at its full size (n = 65536, P = 256, s = 64) in the bench's launch configuration, one
    WR iteration: u_0 ≡ u0 makes the first iterate the closed form u_1(t) = u0 + t φ1(tB) c with
    B = νD2 + J(u0), c = νD2 u0 - u0∘D1 u0 (SURVEY §8(c).4 'WR iteration 1', pinned by
    test_wr_first_iterate_closed_form).  The reference evaluates it at all T_i with the oracle's
    SaI Krylov routine (η = 1e-12) on the constant rank-1 source."""
    from oracle.ebk import ebk_krylov
    from oracle.operators import burgers_J, d1_matrix, d2_matrix
    p = synth.config5()
    c = pexp.Context(p.n, "periodic", p.nu, 0.0, s=p.s, **C5_BENCH_OPTIONS)
    out, st = c.solve_burgers(t(p.u0), p.nu, p.T, p.P, p.tol, 1)
    out = out.cpu().numpy()
    assert st["wr_iters"] == 1
    B = (p.nu * d2_matrix(p.n) + burgers_J(p.u0, p.n)).tocsr()
    cv = p.nu * (d2_matrix(p.n) @ p.u0) - p.u0 * (d1_matrix(p.n) @ p.u0)
    beta = np.linalg.norm(cv)
    coef = np.zeros((p.P, 4, 1))
    coef[:, 0, 0] = beta
    Y = ebk_krylov(B, (cv / beta)[:, None], coef, p.T / p.P, p.P, gamma=0.1, eta=1e-12)
    ref = Y[1:] + p.u0[None, :]
    assert rel(out, ref) < 1e-8, st
    # mass is conserved by every WR iterate (periodic central differences)
    assert np.abs(out.sum(axis=1) - p.u0.sum()).max() < 1e-9 * np.abs(p.u0).sum()


@pytest.mark.parametrize("route", ROUTES)
def test_linear_width_buckets(route):
    """Retained ranks that differ across subintervals (a 1e-6-noise source on the second half:
    m_j = s there, 4 elsewhere): the evaluations run in two width buckets (own block widths,
    gathered into chunk slots and scattered back); equal to the oracle and to the unbucketed run."""
    p = synth.generic_linear(n=600, bc="periodic", nu=5e-3, a=1.3, P=32, s=12, T=2.0, seed=5, rank=3)
    r = np.random.default_rng(9)
    p.src[0, 16:] += 1e-6 * r.standard_normal(p.src[0, 16:].shape)
    out, st = _linear(p, k_max=512, route=route, records=True)
    ref, info = _oracle_linear(p, return_info=True)
    assert st["m_j"] == info["m"][0].tolist()
    assert len(set(st["m_j"])) >= 2
    assert rel(out, ref) < 1e-8, st
    out2, st2 = _linear(p, k_max=512, route=route, width_buckets=-1)
    assert rel(out2, ref) < 1e-8, st2


# ---------------------------------------------------------------- the paper's own workloads (f1, f2)

@pytest.mark.parametrize("P", [2, 8])
def test_f1_pulse_ade_table1(P):
    """f1 (Table 1): forced travelling pulses Eq.(ade)/(manusol), n = 1000,
    tol = 1e-4, T = P·0.5.  GPU = oracle to 1e-8, retained rank 2 (P:565 'retain only the first
    two'), and the error vs the exact PDE solution equals the printed serial PEBK error 3.05e-4
    (the semi-discrete model's own error) within 2 %, for every P (Table 1: 'error' column is
    P-independent to 3 digits for PEBK)."""
    p = synth.pulse_ade(P=P, s=64, tol=1e-4)
    out, st = _linear(p, k_max=256, records=True)
    ref = _oracle_linear(p)
    assert rel(out, ref) < 1e-8, st
    assert set(st["m_j"]) == {2}, st["m_j"]
    x = synth.grid_x(p.n, p.bc)
    ue = synth.pulse_exact(x, p.T)
    err = np.linalg.norm(out[0, -1] - ue) / np.linalg.norm(ue)
    assert abs(err - 3.05e-4) < 0.02 * 3.05e-4, err


def _burgers_forced(pb, k_max=256, **kw):
    c = pexp.Context(pb.n, "periodic", pb.nu, 0.0, s=pb.s, k_max=k_max, **kw)
    out, st = c.solve_burgers(t(pb.u0), pb.nu, pb.T, pb.P, pb.tol, pb.max_wr_iters, f=t(pb.f))
    return out.cpu().numpy(), st


F2_CASES = {
    "sawtooth-cont": lambda: synth.sawtooth_burgers(P=2, n=400, s=50, tol=1e-8, forcing="continuous"),
    "sawtooth-disc": lambda: synth.sawtooth_burgers(P=4, dT=0.05, n=500, s=32, tol=1e-8, forcing="discrete"),
    "multiscale-k4": lambda: synth.multiscale_burgers(P=4, k0=4, n=400, s=50, tol=1e-8, forcing="continuous"),
    "multiscale-k16-disc": lambda: synth.multiscale_burgers(P=4, k0=16, n=400, s=50, tol=1e-8, forcing="discrete"),
}
_F2_REF = {}


def _f2_oracle(name, pb):
    if name not in _F2_REF:   # one oracle run serves both routes
        _F2_REF[name] = oracle.solve_burgers(pb.n, pb.nu, pb.u0, pb.T, pb.P, pb.s, pb.tol, f=pb.f, return_info=True)
    return _F2_REF[name]


@pytest.mark.parametrize("route", ROUTES)
@pytest.mark.parametrize("case", list(F2_CASES))
def test_f2_forced_burgers(case, route):
    """f2: Eq.(burgersEq) with forcing through pexp_solve_burgers_forced:
    equal WR iteration counts and outputs equal to the oracle's to 1e-8; with the discrete forcing
     the result also tracks the manufactured solution itself."""
    pb = F2_CASES[case]()
    out, st = _burgers_forced(pb, route=route)
    ref, info = _f2_oracle(case, pb)
    assert st["wr_iters"] == info["iters"], (st["delta_hist"], info["delta"])
    assert rel(out, ref) < 1e-8, st


def test_f2_discrete_forcing_tracks_exact_solution():
    pb = synth.multiscale_burgers(P=4, k0=4, n=256, s=32, tol=1e-8, forcing="discrete")
    out, st = _burgers_forced(pb)
    x = synth.grid_x(pb.n, "periodic")
    ex = np.stack([synth.multiscale_exact(x, ti, 4) for ti in (np.arange(pb.P) + 1) * pb.T / pb.P])
    assert rel(out, ex) < 1e-6, st


def test_f2_null_forcing_equals_unforced():
    p = synth.config3(n=256, P=4, s=12, T=0.2, nu=0.02)
    out0, _ = _burgers(p)
    c = pexp.Context(p.n, "periodic", p.nu, 0.0, s=p.s)
    out1, _ = c.solve_burgers(t(p.u0), p.nu, p.T, p.P, p.tol, p.max_wr_iters, f=t(np.zeros((p.P, p.s, p.n))))
    # (not bitwise: the scan's converged dimension depends on the checker's timing, at the eta level)
    assert rel(out1.cpu().numpy(), out0) < 1e-9


# ---------------------------------------------------------------- stage parity

def _oracle_linear_stages(p, dense_max=1024):
    """v_j(T_j) (Eq.(linivpSubproblem)) and every homogeneous leg exp((T_i - T_j)A) v_j(T_j)
    (Fig. 2 line 3) from the oracle's primitives, problem 0 of p."""
    from oracle.lowrank import truncated_svd, notaknot_taylor
    from oracle.ebk import ebk_dense, ebk_krylov
    A = ade_matrix(p.n, p.bc, p.nu[0], p.a[0])
    dT = p.T / p.P
    h = dT / (p.s - 1)
    Au0 = A @ p.u0[0]
    dense = p.n <= dense_max
    vend = np.zeros((p.P, p.n))
    for j in range(p.P):
        U, C, _ = truncated_svd(Au0[:, None] + p.src[0, j].T, 0.01 * p.tol)
        if U.shape[1]:
            coef = notaknot_taylor(C, h)
            Y = ebk_dense(A, U, coef, h, p.s - 1) if dense else ebk_krylov(A, U, coef, h, p.s - 1, gamma=dT / 10)
            vend[j] = Y[-1]
    legs = np.zeros((p.P - 1, p.P, p.n))          # legs[j][i] = leg of v_{j+1} at T_{i+1}, i > j
    for j in range(p.P - 1):
        nleg = p.P - 1 - j
        W = (ebk_dense(A, None, None, dT, nleg, y0=vend[j]) if dense
             else ebk_krylov(A, None, None, dT, nleg, gamma=p.T / 10, y0=vend[j]))
        legs[j, j + 1:] = W[1:]
    return vend, legs


@pytest.mark.parametrize("make", [
    lambda: synth.config2(n=1200, P=8, T=0.125, s=64),
    lambda: synth.generic_linear(n=777, bc="periodic", nu=5e-3, a=1.3, P=5, s=12, T=0.5, seed=7),
], ids=["c2-reduced", "generic-periodic"])
def test_stage_vend_and_homogeneous_legs(make):
    """Stage parity: (i) v_j(T_j) from the same u0/src, 1e-9; (ii) the homogeneous
    legs fed the ORACLE's v_j(T_j) (pexp_solve_linear_stages vstart), every leg on its own
    (hom_group = 1) and as group sums (default grouping), 1e-9 relative to the leg's start norm."""
    p = make()
    vend_ref, legs_ref = _oracle_linear_stages(p, dense_max=0)
    c = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=384, hom_group=1)
    out, vend, _, st = c.solve_linear_stages(t(p.u0), t(p.src), p.T, p.P, p.tol)
    vend = vend.cpu().numpy()[0]
    assert rel(vend, vend_ref) < 1e-9, st
    for j in range(p.P):
        assert np.linalg.norm(vend[j] - vend_ref[j]) < 1e-9 * np.linalg.norm(vend_ref), j
    # legs from the oracle's start vectors, one leg per group
    _, _, legs, st = c.solve_linear_stages(t(p.u0), None, p.T, p.P, p.tol, vstart=t(vend_ref[None]))
    legs = legs.cpu().numpy()[0]                  # [P-1][P][n]
    for j in range(p.P - 1):
        assert np.linalg.norm(legs[j] - legs_ref[j]) < 1e-9 * max(np.linalg.norm(vend_ref[j]), 1e-300), j
    # default grouping (8 legs share one block Krylov space): group sums
    c8 = pexp.Context(p.n, p.bc, list(p.nu), list(p.a), s=p.s, k_max=384)
    _, _, legs8, st = c8.solve_linear_stages(t(p.u0), None, p.T, p.P, p.tol, vstart=t(vend_ref[None]))
    legs8 = legs8.cpu().numpy()[0]
    mh = min(8, p.P - 1)
    for g in range(legs8.shape[0]):
        ref = legs_ref[g * mh:(g + 1) * mh].sum(axis=0)
        assert np.linalg.norm(legs8[g] - ref) < 1e-9 * np.linalg.norm(vend_ref), g


@pytest.mark.parametrize("route", ROUTES)
def test_stage_wr_map_on_steep_iterate(route):
    """Stage parity: one WR map F(u_k) (Eq.(ivpSubproblem)/(updateSolution) P:326-335) applied to the
    ORACLE's third iterate of a steepening Burgers run (per-subinterval Jacobians differ, block
    widths > 1), against oracle.wr.wr_map of the same iterate: 1e-8, and the same delta."""
    from oracle.wr import wr_map
    p = synth.config3(n=1024, P=8, s=16, T=0.2, nu=5e-3)
    _, info = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, p.P, p.s, p.tol, return_info=True, fixed_iters=3)
    Uk = info["U"]
    ref = wr_map(Uk, p.u0, p.nu, p.n, p.T, p.P, p.s, p.tol)
    c = pexp.Context(p.n, "periodic", p.nu, 0.0, s=p.s, k_max=512, route=route)
    Unew, out, st = c.wr_map(t(p.u0), t(Uk), p.nu, p.T, p.P, p.tol)
    Unew = Unew.cpu().numpy()
    assert rel(Unew, ref) < 1e-8, st
    assert rel(out.cpu().numpy(), ref[:, -1, :]) < 1e-8
    assert abs(st["wr_last_delta"] - np.max(np.abs(ref - Uk))) < 1e-8
    assert st["max_m"] > 1


# ---------------------------------------------------------------- f3: Chebyshev nodes, higher-order p(t)

@pytest.mark.parametrize("route", ROUTES)
@pytest.mark.parametrize("make", [
    lambda: synth.config1(node_rule=1),
    lambda: synth.generic_linear(n=777, bc="periodic", nu=5e-3, a=1.3, P=5, s=12, T=0.5, seed=7, node_rule=1),
    lambda: synth.generic_linear(n=600, bc="dirichlet", nu=1e-3, a=1.0, P=5, s=20, T=0.5, seed=7, node_rule=1),
], ids=["c1", "generic-periodic", "generic-dirichlet"])
def test_f3_chebyshev_nodes(make, route):
    """f3 (P:451 Chebyshev nodes; higher-order p(t)): pexp_options.node_rule = 1 against the oracle's
    node_rule = 1 (degree-(s-1) interpolant, exact re-expansion) to 1e-8."""
    p = make()
    out, st = _linear(p, route=route, node_rule=1)
    ref = _oracle_linear(p, node_rule=1)
    assert rel(out, ref) < 1e-8, st


def test_f3_pulse_reaches_exact_source_solution():
    """The f1 pulse problem sampled at 32 Chebyshev nodes per subinterval: the CUDA path equals the
    closed-form semi-discrete solution with the EXACT source to 1e-9 (uniform nodes + cubic spline
    stop at the 4e-5 interpolation floor), and the oracle to 1e-8."""
    from tests.closed_forms import pulse_semidiscrete
    p = synth.pulse_ade(P=4, s=32, tol=1e-8, node_rule=1)
    out, st = _linear(p, node_rule=1)
    x = synth.grid_x(p.n, p.bc)
    Ti = (np.arange(p.P) + 1) * p.T / p.P
    ref = np.stack([pulse_semidiscrete(x, ti, p.nu[0], p.a[0], p.n) for ti in Ti])
    assert rel(out[0], ref) < 1e-9, st
    out0, _ = _linear(synth.pulse_ade(P=4, s=32, tol=1e-8), k_max=256)
    assert rel(out0[0], ref) > 1e-6          # the cubic-spline floor the variant removes
    assert rel(out, _oracle_linear(p, node_rule=1)) < 1e-8


def test_f3_sample_times_and_burgers_rejected():
    c = pexp.Context(64, "periodic", 1e-2, 0.0, s=9, node_rule=1)
    np.testing.assert_allclose(c.sample_times(0.9, 3).numpy(), synth.node_times(0.9, 3, 9, node_rule=1), atol=1e-15)
    with pytest.raises(pexp.PexpError):
        c.solve_burgers(t(np.ones(64)), 1e-2, 0.1, 2, 1e-8, 3)


def test_burgers_config5_full_size_late_wr_map_sampled():
    """C5 at its full size (n = 65536, P = 256, s = 64, bench launch configuration) BEYOND the first
    iterate: eight WR maps through pexp_wr_map bring the waveform to the steep regime (block widths
    ~17-25, per-subinterval Jacobians, width buckets, the streaming route, the persistent scan); the
    eighth map u_7 -> u_8 is then checked on sampled subintervals j against the oracle's primitives
    evaluated one subinterval at a time from the SAME inputs (the GPU's u_7 on subinterval j and the
    GPU's scan state u_hat(T_{j-1})): u_8 = u0 + exp((t - T_{j-1}) A_j) u_hat(T_{j-1}) + v_j(t) at all 64
    nodes (Eq.(ivpSubproblem)/(updateSolution) P:326-335), relative 2-norm 1e-8, equal retained rank."""
    from oracle.ebk import ebk_krylov
    from oracle.lowrank import truncated_svd, notaknot_taylor
    from oracle.operators import burgers_J, d1_matrix, d2_matrix
    from oracle.wr import trapezoid_mean, wr_gamma
    p = synth.config5()
    n, s, P = p.n, p.s, p.P
    c = pexp.Context(n, "periodic", p.nu, 0.0, s=s, **C5_BENCH_OPTIONS)
    u0 = t(p.u0)
    Uk = u0.expand(P, s, n).contiguous()
    Un = None
    for k in range(8):
        if Un is not None:
            Uk = Un
        Un, out, st = c.wr_map(u0, Uk, p.nu, p.T, P, p.tol)
    assert st["max_m"] >= 12, st                      # the steep regime
    dT = p.T / P
    h = dT / (s - 1)
    D1, D2 = d1_matrix(n), d2_matrix(n)
    A0 = p.nu * D2
    A0u0 = A0 @ p.u0
    for j in (70, 201):
        Ukj = Uk[j].cpu().numpy()
        ubar = trapezoid_mean(Ukj)
        J = burgers_J(ubar, n)
        Aj = (A0 + J).tocsr()
        gam = wr_gamma(ubar, D1, dT)
        G = np.stack([A0u0 - u * (D1 @ u) - J @ (u - p.u0) for u in Ukj], axis=1)      # [n][s]
        U, C, _ = truncated_svd(G, 0.01 * p.tol)
        V = ebk_krylov(Aj, U, notaknot_taylor(C, h), h, s - 1, gamma=gam, kmax=1600)
        uh_prev = Un[j - 1, -1].cpu().numpy() - p.u0
        Wh = ebk_krylov(Aj, None, None, h, s - 1, gamma=gam, y0=uh_prev, kmax=1600)
        ref = p.u0[None, :] + Wh + V
        got = Un[j].cpu().numpy()
        assert U.shape[1] >= 8, U.shape
        assert rel(got, ref) < 1e-8, (j, U.shape[1])
        assert rel(got - p.u0[None, :], ref - p.u0[None, :]) < 1e-7, j        # the increment itself


@pytest.mark.parametrize("gamma_factor,scan_gamma_factor", [(0.5, 0.7), (2.0, 0.5), (1.0, 2.0)])
def test_shift_parameters_are_route_only(gamma_factor, scan_gamma_factor):
    """pexp_options.gamma_factor / scan_gamma_factor (reading #4: the paper gives no shift) change the
    Krylov spaces, not the result: linear and Burgers solves stay within 1e-8 of the oracle, whose own
    shift is the default dT/10, and the WR iteration count is unchanged."""
    p = synth.generic_linear(n=600, bc="dirichlet", nu=1e-3, a=1.0, P=5, s=12, T=0.5, seed=7)
    out, st = _linear(p, k_max=512, gamma_factor=gamma_factor)
    assert rel(out, _oracle_linear(p)) < 1e-8, st
    q = synth.config3(n=256, P=4, s=12, T=0.2, nu=0.02)
    outb, stb = _burgers(q, gamma_factor=gamma_factor, scan_gamma_factor=scan_gamma_factor)
    ref, info = oracle.solve_burgers(q.n, q.nu, q.u0, q.T, q.P, q.s, q.tol, return_info=True)
    assert stb["wr_iters"] == info["iters"]
    assert rel(outb, ref) < 1e-8, stb
