"""Seeded synthetic workloads C1..C5 (BASELINE.json `configs`, recipe in SURVEY.md §8(d).2).

Every array is IEEE fp64, little-endian, C-contiguous, last index fastest.
Random draws come from ``numpy.random.Generator(PCG64(...))``; per-problem streams
(C4) are seeded with ``[seed, b]`` so a subset of the batch can be regenerated
bit-identically without materialising the whole 2 GiB source.

Conventions fixed here (they are *inputs*, not method arithmetic):
  * periodic grid  x_i = i/n,        i = 0..n-1          (SURVEY §8(c) reading #15)
  * Dirichlet grid x_i = (i+1)/(n+1), i = 0..n-1, u = 0 at x = 0, 1
  * uniform sample nodes, endpoints included (reading #9):
        dT = T/P,  t_{j,i} = j*dT + i*(dT/(s-1)),  j = 0..P-1, i = 0..s-1
    (0-based; "0 = t_1 < ... < t_s = ΔT" on each subinterval).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

PERIODIC = "periodic"
DIRICHLET = "dirichlet"


def _rng(seed) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def grid_x(n: int, bc: str) -> np.ndarray:
    i = np.arange(n, dtype=np.float64)
    if bc == PERIODIC:
        return i / n
    if bc == DIRICHLET:
        return (i + 1.0) / (n + 1.0)
    raise ValueError(bc)


def node_times(T: float, P: int, s: int, node_rule: int = 0) -> np.ndarray:
    """[P][s] sample times.  node_rule 0 (default): uniform, t_{j,i} = j*dT + i*(dT/(s-1));
    node_rule 1: Chebyshev-Lobatto points of each subinterval ("Chebyshev nodes",
    endpoints included as in P:64), t_{j,i} = j*dT + (dT/2)(1 - cos(pi i/(s-1)))."""
    dT = T / P
    j = np.arange(P, dtype=np.float64)[:, None]
    i = np.arange(s, dtype=np.float64)[None, :]
    if node_rule == 1:
        return j * dT + 0.5 * dT * (1.0 - np.cos(np.pi * i / (s - 1)))
    return j * dT + i * (dT / (s - 1))


@dataclass
class LinearProblem:
    """u' = A u + g(t), A = nu*D2 - a*D1, batch of problems."""
    name: str
    n: int
    bc: str
    nu: np.ndarray          # [batch]
    a: np.ndarray           # [batch]
    T: float
    P: int
    s: int
    tol: float
    u0: np.ndarray          # [batch][n]
    src: np.ndarray         # [batch][P][s][n]  g(x, t_{j,i})
    batch_index: np.ndarray = field(default=None)  # which problems of the full batch these are

    @property
    def batch(self) -> int:
        return int(self.u0.shape[0])


@dataclass
class BurgersProblem:
    """u' = nu*D2 u - u∘(D1 u) + f (f = 0 for C3/C5), periodic."""
    name: str
    n: int
    nu: float
    T: float
    P: int
    s: int
    tol: float
    u0: np.ndarray          # [n]
    max_wr_iters: int = 30
    wr_tol: float = 1e-6
    bc: str = PERIODIC
    f: Optional[np.ndarray] = None   # [P][s][n] forcing f(x, t_{j,i}) of Eq.(burgersEq) P:636 (None: f = 0)


def _fourier(x, k, c, s_):
    return c * np.cos(2 * np.pi * k * x) + s_ * np.sin(2 * np.pi * k * x)


def config1(n=256, P=8, s=32, T=1.0, tol=1e-8, seed=1, node_rule=0) -> LinearProblem:
    """C1: periodic ADE, a=1, nu=1e-2; 4-mode u0 (k distinct in 1..8), rank-3 source."""
    r = _rng(seed)
    x = grid_x(n, PERIODIC)
    k = r.choice(np.arange(1, 9), size=4, replace=False)
    al, be = r.standard_normal(4), r.standard_normal(4)
    u0 = sum(_fourier(x, k[q], al[q], be[q]) for q in range(4))
    kap = r.integers(1, 9, size=3)
    ga, de = r.standard_normal(3), r.standard_normal(3)
    w = r.uniform(1.0, 5.0, size=3)
    t = node_times(T, P, s, node_rule)
    modes = np.stack([_fourier(x, kap[q], ga[q], de[q]) for q in range(3)])   # [3][n]
    temp = np.stack([np.sin(2 * np.pi * w[q] * t) for q in range(3)])        # [3][P][s]
    src = np.einsum("rps,rn->psn", temp, modes)
    return LinearProblem("C1", n, PERIODIC, np.array([1e-2]), np.array([1.0]), T, P, s, tol,
                         u0[None].copy(), src[None].copy(), np.array([0]))


def config2(n=4096, P=64, s=64, T=1.0, tol=1e-8, seed=2, noise=1e-10) -> LinearProblem:
    """C2: Dirichlet ADE, a=1, nu=1e-3; Gaussian bump u0; rank-10 source + 1e-10 noise."""
    r = _rng(seed)
    x = grid_x(n, DIRICHLET)
    u0 = np.exp(-(((x - 0.3) / 0.05) ** 2))
    c = r.standard_normal(10)
    w = r.uniform(1.0, 5.0, size=10)
    ph = r.uniform(0.0, 2 * np.pi, size=10)
    t = node_times(T, P, s)
    modes = np.stack([c[q] * np.sin((q + 1) * np.pi * x) for q in range(10)])
    temp = np.stack([np.sin(2 * np.pi * w[q] * t + ph[q]) for q in range(10)])
    src = np.einsum("rps,rn->psn", temp, modes)
    if noise:
        src += noise * r.standard_normal(src.shape)
    return LinearProblem("C2", n, DIRICHLET, np.array([1e-3]), np.array([1.0]), T, P, s, tol,
                         u0[None].copy(), src[None].copy(), np.array([0]))


def config3(n=2048, P=32, s=32, T=0.5, tol=1e-8, nu=1e-2, seed=3) -> BurgersProblem:
    """C3: periodic viscous Burgers, u0 = sin 2πx + 0.5 sin(4πx + φ)."""
    r = _rng(seed)
    x = grid_x(n, PERIODIC)
    ph = r.uniform(0.0, 2 * np.pi)
    u0 = np.sin(2 * np.pi * x) + 0.5 * np.sin(4 * np.pi * x + ph)
    return BurgersProblem("C3", n, nu, T, P, s, tol, u0)


def config4(n=1024, P=16, s=32, T=1.0, tol=1e-8, batch=512, seed=4,
            indices: Optional[np.ndarray] = None) -> LinearProblem:
    """C4: batch of periodic ADE problems, a~U[0.5,2], log10 nu~U[-4,-2], 8-mode u0, rank-5 source.

    ``indices`` selects problems of the full batch (each is drawn from its own
    PCG64([seed, b]) stream, so the subset is bit-identical to the full batch's rows).
    """
    idx = np.arange(batch) if indices is None else np.asarray(indices)
    x = grid_x(n, PERIODIC)
    t = node_times(T, P, s)
    nus, as_, u0s, srcs = [], [], [], []
    for b in idx:
        r = _rng([seed, int(b)])
        as_.append(r.uniform(0.5, 2.0))
        nus.append(10.0 ** r.uniform(-4.0, -2.0))
        al, be = r.standard_normal(8), r.standard_normal(8)
        u0s.append(sum(_fourier(x, q + 1, al[q], be[q]) for q in range(8)))
        kap = r.integers(1, 17, size=5)
        ga, de = r.standard_normal(5), r.standard_normal(5)
        w = r.uniform(1.0, 5.0, size=5)
        ph = r.uniform(0.0, 2 * np.pi, size=5)
        modes = np.stack([_fourier(x, kap[q], ga[q], de[q]) for q in range(5)])
        temp = np.stack([np.sin(2 * np.pi * w[q] * t + ph[q]) for q in range(5)])
        srcs.append(np.einsum("rps,rn->psn", temp, modes))
    return LinearProblem("C4", n, PERIODIC, np.array(nus), np.array(as_), T, P, s, tol,
                         np.stack(u0s), np.stack(srcs), idx)


def config5(n=65536, P=256, s=64, T=1.0, tol=1e-8, nu=1e-3, seed=5) -> BurgersProblem:
    """C5: periodic Burgers, nu=1e-3, u0 = sin 2πx + 0.1·(16-mode N(0,1) Fourier perturbation)."""
    r = _rng(seed)
    x = grid_x(n, PERIODIC)
    al, be = r.standard_normal(16), r.standard_normal(16)
    u0 = np.sin(2 * np.pi * x) + 0.1 * sum(_fourier(x, k + 1, al[k], be[k]) for k in range(16))
    return BurgersProblem("C5", n, nu, T, P, s, tol, u0)


def _bump(x, c, w):
    d = np.abs(x - c)
    d = np.minimum(d, 1.0 - d)
    return np.exp(-((d / w) ** 2))


def generic_linear(n=256, bc=PERIODIC, nu=1e-2, a=1.0, P=4, s=16, T=0.5, tol=1e-8,
                   rank=3, seed=11, noise=0.0, node_rule=0) -> LinearProblem:
    """Non-Fourier data (periodic Gaussian bumps): the Krylov space is NOT invariant,
    so the block Arnoldi runs deep."""
    r = _rng(seed)
    x = grid_x(n, bc)
    u0 = _bump(x, r.uniform(0.2, 0.8), r.uniform(0.05, 0.1))
    if bc == DIRICHLET:
        u0 = u0 * np.sin(np.pi * x)
    t = node_times(T, P, s, node_rule)
    modes = np.stack([r.standard_normal() * _bump(x, r.uniform(0, 1), r.uniform(0.03, 0.1))
                      for _ in range(rank)])
    w = r.uniform(1.0, 5.0, size=rank)
    ph = r.uniform(0, 2 * np.pi, size=rank)
    temp = np.stack([np.sin(2 * np.pi * w[q] * t + ph[q]) for q in range(rank)])
    src = np.einsum("rps,rn->psn", temp, modes)
    if noise:
        src += noise * r.standard_normal(src.shape)
    return LinearProblem("generic", n, bc, np.array([nu]), np.array([a]), T, P, s, tol,
                         u0[None].copy(), src[None].copy(), np.array([0]))


def make_config(name: str, **kw):
    return {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5,
            "generic": generic_linear}[name](**kw)
