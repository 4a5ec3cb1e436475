"""Pins of the oracle against what the paper and the mathematics fix (all CPU, -m "not gpu").

Each test names the oracle function it pins and what a plausible mistake would break.
"""
import json
import os

import numpy as np
import pytest
from scipy.interpolate import CubicSpline
from scipy.integrate import solve_ivp

import synth
import oracle
from oracle.operators import ade_matrix, d1_matrix, d2_matrix, burgers_N, burgers_J, grid_dx
from oracle.lowrank import truncated_svd, notaknot_taylor, eval_taylor
from oracle.ebk import ebk_dense, ebk_krylov
from oracle.expm import phi_blocks
from oracle.wr import wr_map, trapezoid_mean
from tests.closed_forms import phi_scalar, periodic_eigs, periodic_forced_solution, periodic_propagate

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- operators

def test_stencil_golden_rows():
    g = json.load(open(os.path.join(GOLD, "stencil_rows.json")))
    c0, c1, c2 = g["cases"]
    A = ade_matrix(c0["n"], "periodic", c0["nu"], c0["a"])
    np.testing.assert_allclose(A @ np.array(c0["x"], float), c0["Ax"], rtol=0, atol=1e-12)
    A = ade_matrix(c1["n"], "periodic", c1["nu"], c1["a"]).toarray()
    np.testing.assert_allclose(A[0], c1["row0"], atol=1e-12)
    A = ade_matrix(c2["n"], "periodic", c2["nu"], c2["a"]).toarray()
    np.testing.assert_allclose(A[c2["row"], c2["cols"]], c2["vals"], atol=1e-12)


@pytest.mark.parametrize("n,nu,a", [(16, 1e-2, 1.0), (64, 1e-3, 2.0), (33, 0.1, -0.5)])
def test_periodic_operator_eigenpairs(n, nu, a):
    """Circulant closed form: A e_k = λ_k e_k; null space = constants."""
    A = ade_matrix(n, "periodic", nu, a)
    lam = periodic_eigs(n, nu, a)
    j = np.arange(n)
    for k in range(n):
        e = np.exp(2j * np.pi * k * j / n)
        np.testing.assert_allclose(A @ e, lam[k] * e, rtol=1e-12, atol=1e-12 * abs(lam).max())
    assert np.max(np.abs(A @ np.ones(n))) < 1e-10 * abs(lam).max()


def test_dirichlet_operator_eigenpairs():
    """D2 with zero Dirichlet values: sin(kπx_i) eigenvectors, λ = -(4/dx²) sin²(kπ/(2(n+1)))."""
    n = 31
    dx = grid_dx(n, "dirichlet")
    D2 = d2_matrix(n, "dirichlet")
    x = (np.arange(n) + 1) * dx
    for k in range(1, n + 1):
        v = np.sin(k * np.pi * x)
        lam = -(4 / dx ** 2) * np.sin(k * np.pi / (2 * (n + 1))) ** 2
        np.testing.assert_allclose(D2 @ v, lam * v, atol=1e-9 * abs(lam))


def test_burgers_jacobian_exact_for_quadratic():
    """g(u) = -u∘D1u is quadratic, so the central difference quotient equals J(u)v exactly
    (up to rounding): pins the signs/indices of burgers_J."""
    n = 40
    r = np.random.default_rng(0)
    u, v = r.standard_normal(n), r.standard_normal(n)
    eps = 1e-3
    fd = (burgers_N(u + eps * v, n) - burgers_N(u - eps * v, n)) / (2 * eps)
    np.testing.assert_allclose(burgers_J(u, n) @ v, fd, rtol=1e-9, atol=1e-9 * np.abs(fd).max())


def test_mass_of_operators():
    """1ᵀA = 0, 1ᵀJ(u) = 0, 1ᵀ(u∘D1u) = 0 on the periodic grid (SURVEY §8(c).4 'Mass')."""
    n = 50
    r = np.random.default_rng(1)
    u, v = r.standard_normal(n), r.standard_normal(n)
    one = np.ones(n)
    assert abs(one @ (ade_matrix(n, "periodic", 0.3, 1.7) @ v)) < 1e-9
    assert abs(one @ (burgers_J(u, n) @ v)) < 1e-9
    assert abs(one @ burgers_N(u, n)) < 1e-9


# ---------------------------------------------------------------- low-rank source

def test_spline_reproduces_cubics():
    """A not-a-knot spline through samples of a cubic IS that cubic."""
    s, h = 9, 0.3
    t = np.arange(s) * h
    c = np.array([[0.7, -1.2, 0.4, 2.5], [1.0, 0.0, 0.0, 0.0], [-2.0, 3.0, -1.0, 0.5]])
    Y = np.stack([ci[0] + ci[1] * t + ci[2] * t ** 2 + ci[3] * t ** 3 for ci in c])
    T = notaknot_taylor(Y, h)
    for i in range(s - 1):
        ti = i * h
        d0 = c[:, 0] + c[:, 1] * ti + c[:, 2] * ti ** 2 + c[:, 3] * ti ** 3
        d1 = c[:, 1] + 2 * c[:, 2] * ti + 3 * c[:, 3] * ti ** 2
        d2 = 2 * c[:, 2] + 6 * c[:, 3] * ti
        d3 = 6 * c[:, 3]
        np.testing.assert_allclose(T[i], np.stack([d0, d1, d2, d3]), rtol=1e-10, atol=1e-10)


@pytest.mark.parametrize("s", [4, 5, 12, 33])
def test_spline_matches_independent_notaknot(s):
    """Against scipy's CubicSpline(bc_type='not-a-knot') — a different implementation."""
    r = np.random.default_rng(s)
    h = 0.01
    t = np.arange(s) * h
    Y = r.standard_normal((3, s))
    T = notaknot_taylor(Y, h)
    for row in range(3):
        cs = CubicSpline(t, Y[row], bc_type="not-a-knot")
        for i in range(s - 1):
            for q in range(4):
                np.testing.assert_allclose(T[i, q, row], cs(t[i], q) if q < 3 else cs(t[i] + h / 2, 3),
                                           rtol=1e-9, atol=1e-9 * np.abs(T[:, q, row]).max())


def test_truncated_svd_known_spectrum():
    """G = Q1 diag(σ) Q2ᵀ with known σ: m counts σ > τσ1, projection = top-m part."""
    r = np.random.default_rng(3)
    n, s = 200, 16
    Q1, _ = np.linalg.qr(r.standard_normal((n, s)))
    Q2, _ = np.linalg.qr(r.standard_normal((s, s)))
    sig = 10.0 ** -np.arange(s, dtype=float)        # 1, 1e-1, ..., 1e-15
    G = (Q1 * sig) @ Q2.T
    U, C, sv = truncated_svd(G, 1e-10)
    assert U.shape[1] == 10                          # σ_1..σ_10 > 1e-10
    np.testing.assert_allclose(sv[:10], sig[:10], rtol=1e-8)
    P_true = (Q1[:, :10] * sig[:10]) @ Q2[:, :10].T
    assert np.linalg.norm(U @ C - P_true) < 1e-13
    Z, Cz, _ = truncated_svd(np.zeros((n, s)), 1e-10)
    assert Z.shape[1] == 0


def test_config1_source_rank_is_four():
    """C1: Ĝ = A u0 + Σ_{r=1}^{3} mode_r sin(2πw_r t) has rank exactly 4."""
    p = synth.config1()
    A = ade_matrix(p.n, p.bc, p.nu[0], p.a[0])
    for j in (0, 3, 7):
        G = (A @ p.u0[0])[:, None] + p.src[0, j].T
        U, C, sv = truncated_svd(G, 0.01 * p.tol)
        assert U.shape[1] == 4 and sv[4] < 1e-13 * sv[0]


def test_theorem1_singular_value_decay():
    """Theorem 1: σ_{j+1} = sqrt(s-j) O(ΔT^j) — fitted log-log slope >= j - 0.3
    for j = 1, 2, 3 under ΔT halving with s fixed."""
    n, s = 400, 12
    x = np.arange(n) / n
    nu = 1e-2

    def g(t):  # smooth travelling Gaussian pulse (infinite rank in space-time)
        d = np.abs(x - 0.5 - t)
        return np.exp(-((np.minimum(d, 1 - d)) / 0.1) ** 2) * (1 + nu * t)

    dts = [0.008, 0.004, 0.002, 0.001]   # asymptotic regime: ΔT << pulse width
    sig = []
    for dT in dts:
        t = np.arange(s) * dT / (s - 1)
        G = np.stack([g(ti) for ti in t], axis=1)
        sig.append(np.linalg.svd(G, compute_uv=False))
    sig = np.array(sig)
    for j in (1, 2, 3):
        slope = np.polyfit(np.log(dts), np.log(sig[:, j]), 1)[0]
        assert slope >= j - 0.3, (j, slope)


# ---------------------------------------------------------------- EBK solve

def test_golden_scalar_examples():
    g = json.load(open(os.path.join(GOLD, "scalar_examples.json")))
    for ex in g["ebk_scalar"]:
        A = np.array([[ex["lambda"]]])
        U = np.array([[1.0]])
        s = 5
        h = ex["t"] / (s - 1)
        coef = np.zeros((s - 1, 4, 1)); coef[:, 0, 0] = ex["c"]
        Y = ebk_dense(A, U, coef, h, s - 1)
        np.testing.assert_allclose(Y[-1, 0], ex["y"], rtol=1e-13)
    from scipy.linalg import expm
    for ex in g["expm"]:
        np.testing.assert_allclose(expm(np.array(ex["M"], float)), ex["expM"], rtol=1e-14, atol=1e-15)


def test_phi_blocks_against_scalar_phi():
    """Augmented-exponential φ blocks vs the scalar φ recurrence on a diagonal X."""
    lam = np.array([-3.0, -0.2, 0.0, 0.7, -40.0])
    h = 0.37
    F0, B = phi_blocks(np.diag(lam), np.eye(5), h)
    np.testing.assert_allclose(np.diag(F0), np.exp(lam * h), rtol=1e-13)
    for q in range(4):
        ref = phi_scalar(q + 1, lam * h).real * h
        np.testing.assert_allclose(np.diag(B[q]), ref, rtol=1e-12, atol=1e-16)
        assert np.max(np.abs(B[q] - np.diag(np.diag(B[q])))) < 1e-15


@pytest.mark.parametrize("route", ["dense", "krylov"])
def test_ebk_periodic_closed_form(route):
    """One EBK evaluation on the periodic ADE vs the per-Fourier-mode exact solution of the
    interpolated-source problem, for non-Fourier (Gaussian-bump) data."""
    p = synth.generic_linear(n=256, P=4, s=16, nu=5e-3, a=1.3, seed=5)
    A = ade_matrix(p.n, p.bc, p.nu[0], p.a[0])
    dT = p.T / p.P
    h = dT / (p.s - 1)
    G = (A @ p.u0[0])[:, None] + p.src[0, 1].T
    U, C, _ = truncated_svd(G, 1e-10)
    coef = notaknot_taylor(C, h)
    if route == "dense":
        Y = ebk_dense(A, U, coef, h, p.s - 1)
    else:
        Y = ebk_krylov(A, U, coef, h, p.s - 1, gamma=dT / 10)
    coef_phys = np.einsum("nm,iqm->iqn", U, coef)
    Yex = periodic_forced_solution(p.n, p.nu[0], p.a[0], coef_phys, h)
    assert np.linalg.norm(Y - Yex) <= 1e-11 * np.linalg.norm(Yex)


def test_ebk_homogeneous_krylov_closed_form():
    n, nu, a = 512, 2e-3, 1.0
    r = np.random.default_rng(4)
    x = np.arange(n) / n
    v = np.exp(-((x - 0.4) / 0.05) ** 2) + 0.1 * r.standard_normal(n)
    A = ade_matrix(n, "periodic", nu, a)
    Y = ebk_krylov(A, None, None, 0.05, 6, gamma=0.03, y0=v)
    for q in range(7):
        ex = periodic_propagate(n, nu, a, v, 0.05 * q)
        assert np.linalg.norm(Y[q] - ex) <= 1e-11 * np.linalg.norm(v)


def test_ebk_dirichlet_vs_bruteforce_implicit_rk():
    """Tiny Dirichlet grid: oracle (dense and Krylov) vs scipy Radau (independent integrator)
    on y' = A y + U p(t) with the spline source evaluated continuously."""
    p = synth.generic_linear(n=24, bc="dirichlet", P=2, s=8, nu=2e-2, a=1.0, T=0.2, seed=9)
    A = ade_matrix(p.n, p.bc, p.nu[0], p.a[0])
    h = p.T / p.P / (p.s - 1)
    G = (A @ p.u0[0])[:, None] + p.src[0, 0].T
    U, C, _ = truncated_svd(G, 1e-10)
    coef = notaknot_taylor(C, h)
    Ad = A.toarray()
    f = lambda t, y: Ad @ y + U @ eval_taylor(coef, h, t)
    tend = (p.s - 1) * h
    sol = solve_ivp(f, (0, tend), np.zeros(p.n), method="Radau", rtol=1e-12, atol=1e-14,
                    t_eval=np.arange(p.s) * h, max_step=h / 4)
    Yd = ebk_dense(A, U, coef, h, p.s - 1)
    Yk = ebk_krylov(A, U, coef, h, p.s - 1, gamma=h)
    ref = sol.y.T
    assert np.linalg.norm(Yd - ref) <= 1e-8 * np.linalg.norm(ref)
    assert np.linalg.norm(Yk - Yd) <= 1e-11 * np.linalg.norm(Yd)


# ---------------------------------------------------------------- Paraexp

def _linear(p, **kw):
    return oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol, **kw)


@pytest.mark.parametrize("dense_max", [10 ** 6, 0])
def test_paraexp_periodic_closed_form(dense_max):
    """Full solve_linear (SVD, spline, nonhomogeneous legs, homogeneous legs, superposition)
    vs the circulant closed form of û' = Aû + S(t) integrated mode by mode across all
    subintervals (sequentially), with S built from the same truncated projection."""
    p = synth.generic_linear(n=200, P=5, s=10, nu=4e-3, a=0.8, T=0.6, seed=21)
    out = _linear(p, dense_max=dense_max)
    A = ade_matrix(p.n, p.bc, p.nu[0], p.a[0])
    dT = p.T / p.P
    h = dT / (p.s - 1)
    uhat = np.zeros(p.n)
    for j in range(p.P):
        G = (A @ p.u0[0])[:, None] + p.src[0, j].T
        U, C, _ = truncated_svd(G, 0.01 * p.tol)
        coef_phys = np.einsum("nm,iqm->iqn", U, notaknot_taylor(C, h))
        uhat = periodic_forced_solution(p.n, p.nu[0], p.a[0], coef_phys, h, z0=uhat)[-1]
        ref = p.u0[0] + uhat
        assert np.linalg.norm(out[0, j] - ref) <= 1e-11 * np.linalg.norm(ref), j


def test_paraexp_unforced_closed_form_and_P_invariance():
    """g = 0: the shifted source A u0 is constant ⇒ rank 1, spline exact, so
    u(T_i) = e^{T_i A} u0 exactly, independent of P; energy non-increasing."""
    n, T = 128, 1.0
    x = np.arange(n) / n
    u0 = np.exp(-((x - 0.5) / 0.08) ** 2)
    for P in (1, 2, 4):
        src = np.zeros((1, P, 6, n))
        out = oracle.solve_linear(n, "periodic", [1e-2], [1.0], u0[None], src, T, P, 6, 1e-8)
        for i in range(P):
            ex = periodic_propagate(n, 1e-2, 1.0, u0, (i + 1) * T / P)
            assert np.linalg.norm(out[0, i] - ex) <= 1e-10 * np.linalg.norm(ex)
        e = [np.linalg.norm(u0)] + [np.linalg.norm(out[0, i]) for i in range(P)]
        assert all(e[i + 1] <= e[i] * (1 + 1e-12) for i in range(P))


def test_paraexp_dirichlet_unforced_energy_decay():
    n = 100
    x = (np.arange(n) + 1) / (n + 1)
    u0 = np.exp(-((x - 0.3) / 0.05) ** 2)
    src = np.zeros((1, 8, 6, n))
    out = oracle.solve_linear(n, "dirichlet", [1e-3], [1.0], u0[None], src, 1.0, 8, 6, 1e-8)
    e = [np.linalg.norm(u0)] + [np.linalg.norm(out[0, i]) for i in range(8)]
    assert all(e[i + 1] < e[i] for i in range(8))


def test_paraexp_mass_conservation_config1():
    """Periodic: 1ᵀu(T_i) = 1ᵀu0 + ∫1ᵀS dt; C1's modes have k >= 1 ⇒ zero-mean source."""
    p = synth.config1()
    out = _linear(p)
    m0 = p.u0[0].sum()
    for i in range(p.P):
        assert abs(out[0, i].sum() - m0) <= 1e-10 * np.abs(out[0, i]).sum()


def test_paraexp_krylov_equals_dense_dirichlet():
    p = synth.generic_linear(n=150, bc="dirichlet", P=3, s=8, nu=1e-3, a=1.0, T=0.3, seed=2)
    o1 = _linear(p)
    o2 = _linear(p, dense_max=0)
    assert np.linalg.norm(o1 - o2) <= 1e-11 * np.linalg.norm(o1)


# ---------------------------------------------------------------- waveform relaxation

@pytest.mark.parametrize("dense_max", [1024, 0])
def test_wr_first_iterate_closed_form(dense_max):
    """u_0 ≡ u0 ⇒ ū_j = u0, one operator B = νD2 + J(u0), constant source c = νD2u0 - u0∘D1u0
    ⇒ u_1(t) = u0 + t φ1(tB) c (SURVEY §8(c).4 'WR iteration 1').  dense_max = 0 forces the
    Krylov branch of wr_map (the one the n > 1024 parity references use) for the nonhomogeneous
    legs and the scan."""
    from scipy.linalg import expm
    p = synth.config3(n=96, P=3, s=7, T=0.15, nu=0.03)
    U0 = np.broadcast_to(p.u0, (p.P, p.s, p.n)).copy()
    U1 = wr_map(U0, p.u0, p.nu, p.n, p.T, p.P, p.s, p.tol, dense_max=dense_max)
    B = (p.nu * d2_matrix(p.n) + burgers_J(p.u0, p.n)).toarray()
    c = p.nu * (d2_matrix(p.n) @ p.u0) - p.u0 * (d1_matrix(p.n) @ p.u0)
    t = synth.node_times(p.T, p.P, p.s)
    M = np.zeros((p.n + 1, p.n + 1)); M[:p.n, :p.n] = B; M[:p.n, p.n] = c
    for j in range(p.P):
        for i in range(p.s):
            ex = p.u0 + expm(t[j, i] * M)[:p.n, p.n]
            assert np.linalg.norm(U1[j, i] - ex) <= 1e-10 * np.linalg.norm(ex), (j, i)


@pytest.mark.parametrize("dense_max", [1024, 0])
def test_wr_mass_conserved_every_iterate(dense_max):
    p = synth.config3(n=128, P=4, s=8, T=0.2, nu=0.02)
    U = np.broadcast_to(p.u0, (p.P, p.s, p.n)).copy()
    m0 = p.u0.sum()
    for _ in range(3):
        U = wr_map(U, p.u0, p.nu, p.n, p.T, p.P, p.s, p.tol, dense_max=dense_max)
        assert np.max(np.abs(U.sum(axis=2) - m0)) <= 1e-9 * np.abs(p.u0).sum()


@pytest.mark.parametrize("dense_max", [1024, 0])
def test_wr_fixed_point_vs_bruteforce_radau(dense_max):
    """Tiny grid: the converged WR iterate vs an independent implicit integrator (Radau) on the
    full semi-discrete Burgers u' = νD2u - u∘D1u; agreement at the level of the
    source-interpolation error.  dense_max = 0: the SaI Krylov branch and the Krylov scan."""
    p = synth.config3(n=32, P=4, s=16, T=0.2, nu=0.05)
    out, info = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, p.P, p.s, p.tol, wr_tol=1e-13,
                                     max_wr_iters=40, return_info=True, dense_max=dense_max)
    D1, D2 = d1_matrix(p.n).toarray(), d2_matrix(p.n).toarray()
    f = lambda t, u: p.nu * D2 @ u - u * (D1 @ u)
    Tj = np.arange(1, p.P + 1) * p.T / p.P
    sol = solve_ivp(f, (0, p.T), p.u0, method="Radau", rtol=1e-12, atol=1e-14, t_eval=Tj)
    err = np.linalg.norm(out - sol.y.T) / np.linalg.norm(sol.y)
    assert info["delta"][-1] < 1e-12
    assert err < 1e-7, err


@pytest.mark.parametrize("dense_max", [1024, 0])
def test_wr_P1_vs_P4_same_solution(dense_max):
    p = synth.config3(n=64, P=1, s=24, T=0.1, nu=0.05)
    o1 = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, 1, 24, p.tol, wr_tol=1e-12, dense_max=dense_max)
    o4 = oracle.solve_burgers(p.n, p.nu, p.u0, p.T, 4, 8, p.tol, wr_tol=1e-12, dense_max=dense_max)
    assert np.linalg.norm(o1[-1] - o4[-1]) <= 1e-7 * np.linalg.norm(o1[-1])


def test_trapezoid_mean_exact_for_linear_in_time():
    s, n = 9, 5
    r = np.random.default_rng(0)
    a, b = r.standard_normal(n), r.standard_normal(n)
    tt = np.linspace(0, 1, s)
    U = a[None] + tt[:, None] * b[None]
    np.testing.assert_allclose(trapezoid_mean(U), a + 0.5 * b, rtol=1e-14)


def test_wr_krylov_branch_equals_dense_branch_steep():
    """The two branches of wr_map on a steep-front case (ν = 2e-3, n = 128, several iterations,
    block widths > 1 and per-subinterval Jacobians that differ): the Krylov branch (SaI block
    Arnoldi + Krylov scan, used by every n > 1024 parity reference) equals the dense-expm
    branch (the definition) to the Krylov stop tolerance."""
    p = synth.config5(n=128, P=4, s=16, T=0.2, nu=2e-3)
    U = np.broadcast_to(p.u0, (p.P, p.s, p.n)).copy()
    for k in range(4):
        info_d, info_k = {}, {}
        Ud = wr_map(U, p.u0, p.nu, p.n, p.T, p.P, p.s, p.tol, info=info_d)
        Uk = wr_map(U, p.u0, p.nu, p.n, p.T, p.P, p.s, p.tol, dense_max=0, info=info_k)
        assert info_d["m"] == info_k["m"]
        assert np.linalg.norm(Ud - Uk) <= 1e-10 * np.linalg.norm(Ud), k
        U = Ud
    assert max(info_d["m"]) > 1
