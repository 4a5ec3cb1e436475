"""Pins of the oracle on the paper's own workloads (CPU, -m "not gpu").

f1: Eq.(ade)/(manusol), Table 1.  f2: Eq.(burgersEq) with forcing
(P:636-653), Eq.(multiscale_solution), discrete forcing.
"""
import numpy as np

import oracle
import synth
from synth.configs import grid_x
from tests.closed_forms import pulse_semidiscrete


def _pulse(P, s=64, tol=1e-8):
    p = synth.pulse_ade(P=P, s=s, tol=tol)
    out = oracle.solve_linear(p.n, p.bc, p.nu, p.a, p.u0, p.src, p.T, p.P, p.s, p.tol)[0]
    x = grid_x(p.n, p.bc)
    Ti = (np.arange(P) + 1) * p.T / P
    return p, out, x, Ti


def test_f1_pulse_vs_semidiscrete_closed_form():
    """oracle.solve_linear on the f1 workload vs the single-mode circulant closed form of the
    semi-discrete system with the EXACT (not interpolated) source.  The difference is the not-a-knot
    spline error of cos(10π(x - t)) sampled at h = ΔT/(s-1): at least fourth order in h, so s = 32 -> 64
    must shrink it by ≥ (63/31)^4 ≈ 17 (measured ≈ 56: at ωh = 0.5 the s = 32 case is pre-asymptotic);
    a dropped Taylor term or a wrong node spacing breaks it."""
    errs = []
    for s in (32, 64):
        p, out, x, Ti = _pulse(2, s=s)
        ref = np.stack([pulse_semidiscrete(x, t, p.nu[0], p.a[0], p.n) for t in Ti])
        errs.append(np.linalg.norm(out - ref) / np.linalg.norm(ref))
    assert errs[1] < 2e-6, errs
    assert errs[0] / errs[1] > 12, errs


def test_f1_table1_serial_error():
    """Table 1: serial PEBK error 3.05e-4 in the relative l2 norm Eq.(relerr) vs
    the exact PDE solution.  At Δx = 1e-3 this is the semi-discrete model's own error (the phase lag
    of the central difference on the k = 10π pulses saturates once the forcing balances diffusion,
    T ≳ 0.5); the oracle at T = 1 must reproduce the printed value within 2 %."""
    p, out, x, Ti = _pulse(2)
    ue = synth.pulse_exact(x, Ti[-1])
    err = np.linalg.norm(out[-1] - ue) / np.linalg.norm(ue)
    assert abs(err - 3.05e-4) < 0.02 * 3.05e-4, err


def _wr(pb):
    return oracle.solve_burgers(pb.n, pb.nu, pb.u0, pb.T, pb.P, pb.s, pb.tol, f=pb.f, return_info=True)


def test_f2_discrete_forcing_reproduces_exact_solution():
    """With the discrete forcing the semi-discrete Burgers system has the manufactured
    solution Eq.(multiscale_solution) as its exact solution, so the converged WR fixed point equals
    u(x, T_i) up to the source interpolation error (fourth order in h: s = 16 -> 32 shrinks it
    ≳ 8x).  A wrong sign or a dropped forcing term leaves an O(1) error."""
    errs = []
    for s in (16, 32):
        pb = synth.multiscale_burgers(P=2, k0=4, n=64, s=s, tol=1e-8, forcing="discrete")
        out, info = _wr(pb)
        x = grid_x(pb.n, "periodic")
        ex = np.stack([synth.multiscale_exact(x, t, 4) for t in (np.arange(pb.P) + 1) * pb.T / pb.P])
        errs.append(np.linalg.norm(out - ex) / np.linalg.norm(ex))
        assert info["delta"][-1] < 1e-6
    assert errs[0] < 1e-6 and errs[1] < errs[0] / 8, errs


def test_f2_continuous_forcing_second_order_in_dx():
    """Continuous forcing: the WR fixed point carries the O(Δx²) error of the central differences
    (Fig. error_differentdx); halving Δx divides it by ≈ 4."""
    errs = []
    for n in (64, 128):
        pb = synth.multiscale_burgers(P=2, k0=4, n=n, s=16, tol=1e-8, forcing="continuous")
        out, _ = _wr(pb)
        x = grid_x(n, "periodic")
        ex = np.stack([synth.multiscale_exact(x, t, 4) for t in (np.arange(pb.P) + 1) * pb.T / pb.P])
        errs.append(np.linalg.norm(out - ex) / np.linalg.norm(ex))
    assert 3.6 < errs[0] / errs[1] < 4.4, errs


def test_f2_sawtooth_discrete_forcing():
    """Smoothed sawtooth Eq.(modifiedSawtooth) with discrete forcing: WR converges and
    its fixed point tracks the travelling wave to the interpolation level."""
    pb = synth.sawtooth_burgers(P=2, n=128, s=32, tol=1e-8, forcing="discrete")
    out, info = _wr(pb)
    x = grid_x(pb.n, "periodic")
    Ti = (np.arange(pb.P) + 1) * pb.T / pb.P
    ex = np.stack([synth.sawtooth_exact(x, t + 0 * x) for t in Ti])
    assert info["delta"][-1] < 1e-6
    assert np.linalg.norm(out - ex) / np.linalg.norm(ex) < 2e-6
