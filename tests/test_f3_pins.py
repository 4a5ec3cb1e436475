"""Pins of the oracle's f3 variant ("Chebyshev nodes", "other
types of p(t) are possible"): Chebyshev-Lobatto sample nodes and p(t) = the degree-(s-1)
interpolant.  CPU only (-m "not gpu")."""
import numpy as np

import oracle
import synth
from oracle.lowrank import cheb_taylor
from synth.configs import grid_x, node_times
from tests.closed_forms import pulse_semidiscrete


def test_chebyshev_nodes_closed_form():
    """t_{j,i} = j dT + (dT/2)(1 - cos(pi i/(s-1))): endpoints included, symmetric, clustered
    at the ends; the interior nodes are the extrema of T_{s-1} mapped to the subinterval."""
    T, P, s = 0.9, 3, 9
    t = node_times(T, P, s, node_rule=1)
    dT = T / P
    for j in range(P):
        assert t[j, 0] == j * dT and abs(t[j, -1] - (j + 1) * dT) < 1e-15
        loc = (t[j] - j * dT) / dT
        np.testing.assert_allclose(loc + loc[::-1], 1.0, atol=1e-15)
        x = 2 * loc - 1
        # extrema of the Chebyshev polynomial T_{s-1}: |T_{s-1}(x_i)| = 1, alternating sign
        Tn = np.cos((s - 1) * np.arccos(np.clip(x, -1, 1)))
        np.testing.assert_allclose(np.abs(Tn), 1.0, atol=1e-12)
        assert np.all(np.diff(np.sign(Tn)) != 0)
    assert np.diff(t[0])[0] < np.diff(t[0])[s // 2 - 1] / 2    # clustered at the ends


def test_cheb_taylor_reproduces_polynomials_exactly():
    """A polynomial of degree s-1 IS its interpolant: cheb_taylor must return its exact derivatives
    p^{(q)} at every uniform piece start (hand-differentiated monomials, no library call)."""
    s, dT, npieces = 7, 0.3, 5
    r = np.random.default_rng(3)
    a = r.standard_normal((2, s))                       # p_r(tau) = sum_d a[r][d] tau^d
    tau = 0.5 * dT * (1 - np.cos(np.pi * np.arange(s) / (s - 1)))
    Y = np.stack([sum(a[r_, d] * tau ** d for d in range(s)) for r_ in range(2)])
    out = cheb_taylor(Y, dT, npieces)                   # [npieces][s][2]
    for i in range(npieces):
        sg = i * dT / npieces
        for q in range(s):
            for r_ in range(2):
                ref = sum(a[r_, d] * np.prod(np.arange(d, d - q, -1)) * sg ** (d - q) for d in range(q, s))
                assert abs(out[i, q, r_] - ref) <= 1e-9 * (1 + abs(ref)) * max(1.0, (2 / dT) ** q * 1e-3), (i, q)


def _pulse_err(node_rule, s, n=200, P=2):
    p = synth.pulse_ade(P=P, s=s, tol=1e-8, n=n, node_rule=node_rule)
    out = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol, node_rule=node_rule)[0]
    x = grid_x(p.n, p.bc)
    Ti = (np.arange(P) + 1) * p.T / P
    ref = np.stack([pulse_semidiscrete(x, t, p.nu[0], p.a[0], p.n) for t in Ti])
    return np.linalg.norm(out - ref) / np.linalg.norm(ref)


def test_f3_removes_the_interpolation_floor():
    """The f1 pulse problem has a closed-form semi-discrete solution with the EXACT source
    (tests/closed_forms.pulse_semidiscrete, single circulant mode).  With uniform nodes and the cubic
    spline the oracle sits at the spline's interpolation floor (4e-5 at s = 32); with Chebyshev nodes
    and the degree-(s-1) interpolant it reaches the closed form to rounding (spectral convergence:
    s = 16 -> 2e-7, s = 32 -> 1e-13).  A wrong node formula, a dropped Taylor term or a wrong
    derivative scale leaves an error far above these levels."""
    e_uni = _pulse_err(0, 32)
    e16, e32 = _pulse_err(1, 16), _pulse_err(1, 32)
    assert 1e-5 < e_uni < 1e-4, e_uni
    assert 1e-8 < e16 < 1e-6, e16
    assert e32 < 1e-12, e32


def test_f3_krylov_route_equals_dense_route():
    """node_rule 1 through the oracle's SaI block Arnoldi (dense_max = 0) equals the dense route."""
    p = synth.generic_linear(n=200, bc="dirichlet", nu=2e-3, a=1.0, P=3, s=12, T=0.3, seed=4, node_rule=1)
    a = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol, node_rule=1)
    b = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol, node_rule=1, dense_max=0)
    assert np.linalg.norm(a - b) / np.linalg.norm(a) < 1e-10
