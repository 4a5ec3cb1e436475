"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the method (no stencil, no SVD, no Krylov,
no expm).  It only draws random numbers with numpy's PCG64 and evaluates the
closed-form initial conditions / sources of SURVEY.md §8(d).2 at grid points
and sample nodes, so that the GPU path and the oracle consume identical bytes.
"""
from .configs import (  # noqa: F401
    LinearProblem,
    BurgersProblem,
    grid_x,
    node_times,
    config1,
    config2,
    config3,
    config4,
    config5,
    generic_linear,
    make_config,
)
from .paper_workloads import (  # noqa: F401,E402
    pulse_ade,
    pulse_exact,
    sawtooth_burgers,
    sawtooth_exact,
    multiscale_burgers,
    multiscale_exact,
)
