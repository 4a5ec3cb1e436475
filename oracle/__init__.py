"""ORACLE — plain, slow, CPU, fp64 reference of the Paraexp-EBK hot path (§2).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
from this package.  The product path (``paper_1509_04567_b200``) never imports it,
and this package never imports the product path: the two share no code, no
headers, no constants.  Only ``synth`` (seeded inputs, no method arithmetic)
feeds both.

Layout (each function cites the PAPER.md passage it follows; "P:nnn" = PAPER.md
line nnn, "S:nnn" = SPEC.md line nnn, readings #k = SURVEY.md §8(c).3 / DESIGN.md §3):
  operators.py  A = nu*D2 - a*D1, Burgers N(u), J(u)
  lowrank.py    truncated thin SVD and the not-a-knot cubic p(t)
  expm.py       exact piecewise-cubic integration via the augmented exponential (phi_q)
  krylov.py     shift-and-invert block Arnoldi EBK solve, no restart
  paraexp.py    linear Paraexp superposition (Fig. 2)
  wr.py         waveform relaxation with per-subinterval averaged Jacobians (Fig. 5)

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``): circulant closed form per
Fourier mode, dense expm on tiny grids, brute-force implicit Runge-Kutta on tiny
Burgers, mass conservation, energy decay, P-invariance, WR iteration-1 closed
form, Theorem 1 decay slopes, spline polynomial reproduction.
Parity unpinned: none of the functions above.
"""
from .operators import ade_matrix, d1_matrix, d2_matrix, burgers_N, burgers_J  # noqa: F401
from .lowrank import truncated_svd, notaknot_taylor  # noqa: F401
from .paraexp import solve_linear  # noqa: F401
from .wr import solve_burgers  # noqa: F401
