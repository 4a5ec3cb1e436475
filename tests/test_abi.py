"""C-ABI checks that need no GPU: the library loads, exports every symbol include/pexp.h
declares, and its host-only calls validate arguments (no compute calls here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pexp.h")


@pytest.fixture(scope="module")
def P():
    from paper_1509_04567_b200 import build
    build.build()
    from paper_1509_04567_b200 import pexp
    return pexp


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"PEXP_API\s+[\w\s\*]+?\b(pexp_\w+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("pexp_create", "pexp_solve_linear", "pexp_solve_burgers", "pexp_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(P):
    lib = C.CDLL(P.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(P.EXPORTED) == declared_symbols()


def test_no_oracle_or_cpu_fallback_in_product(root):
    """The product package never imports the oracle, and the binding has no fallback path."""
    pkg = os.path.join(root, "paper_1509_04567_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "numpy.linalg" not in txt and "scipy" not in txt, f


def test_create_validation(P):
    with pytest.raises(P.PexpError):
        P.Context(2, "periodic", 1e-2, 1.0)              # n < 3
    with pytest.raises(P.PexpError):
        P.Context(64, "periodic", -1.0, 1.0)             # nu < 0
    with pytest.raises(P.PexpError):
        P.Context(64, "periodic", 1e-2, 1.0, s=3)         # s < 4 (not-a-knot minimum)
    with pytest.raises(P.PexpError):
        P.Context(64, "periodic", 1e-2, 1.0, s=65)        # s > 64
    c = P.Context(64, "dirichlet", [1e-2, 1e-3], [1.0, 0.5])
    assert c.batch == 2


def test_sample_times_match_synth_convention(P):
    c = P.Context(50, "periodic", 1e-2, 1.0, s=7)
    t = c.sample_times(0.9, 5).numpy()
    np.testing.assert_array_equal(t, synth.node_times(0.9, 5, 7))


def test_sample_times_chebyshev_rule(P):
    """node_rule = 1 (row f3): Chebyshev-Lobatto nodes of each subinterval, endpoints included."""
    c = P.Context(50, "periodic", 1e-2, 1.0, s=9, node_rule=1)
    t = c.sample_times(0.9, 5).numpy()
    np.testing.assert_allclose(t, synth.node_times(0.9, 5, 9, node_rule=1), rtol=0, atol=2e-16)
    with pytest.raises(P.PexpError):
        P.Context(50, "periodic", 1e-2, 1.0, s=64, k_max=512, node_rule=1)   # K + 12 s > capacity
    with pytest.raises(P.PexpError):
        P.Context(50, "periodic", 1e-2, 1.0, node_rule=2)


def test_chebyshev_taylor_matrix_host_logic(P):
    """Host logic of node_rule = 1: the library's nodal-values -> Taylor-coefficients map (long double
    Chebyshev recurrences) against (i) exact derivatives of a polynomial of degree s-1, hand-differentiated,
    and (ii) the oracle's numpy.polynomial route on a smooth function (low orders, where that route is
    accurate)."""
    from oracle.lowrank import cheb_taylor
    s, dT = 10, 0.3
    c = P.Context(50, "periodic", 1e-2, 1.0, s=s, node_rule=1)
    D = c.chebyshev_taylor_matrix(dT).numpy()                      # [s-1][12][s]
    tau = 0.5 * dT * (1 - np.cos(np.pi * np.arange(s) / (s - 1)))
    r = np.random.default_rng(1)
    a = r.standard_normal(s)                                       # p(tau) = sum_d a[d] (tau/dT)^d
    y = sum(a[d] * (tau / dT) ** d for d in range(s))
    got = D @ y                                                    # [s-1][12]
    for i in range(s - 1):
        sg = i * dT / (s - 1)
        for q in range(min(12, s)):
            ref = sum(a[d] * np.prod(np.arange(d, d - q, -1)) * (sg / dT) ** (d - q) / dT ** q for d in range(q, s))
            assert abs(got[i, q] - ref) <= 1e-10 * max(1.0, abs(ref), (s * s / dT) ** q * 1e-6), (i, q)
    f = np.sin(7 * tau + 0.3)
    ref = cheb_taylor(f[None, :], dT, s - 1)[:, :4, 0]             # orders 0..3
    np.testing.assert_allclose((D @ f)[:, :4], ref, rtol=1e-9, atol=1e-9 * 7 ** 3)
    assert P.Context(50, "periodic", 1e-2, 1.0, s=s)._h is not None
    with pytest.raises(P.PexpError):
        P.Context(50, "periodic", 1e-2, 1.0, s=s).chebyshev_taylor_matrix(dT)   # node_rule = 0


def test_workspace_query_and_solve_without_workspace(P):
    c = P.Context(128, "periodic", 1e-2, 1.0, s=8)
    assert c.workspace_bytes(4, 0) > 0
    assert c.workspace_bytes(4, 1) > 0
    assert c.workspace_bytes(4, 2) == max(c.workspace_bytes(4, 0), c.workspace_bytes(4, 1))
    assert c.workspace_bytes(0, 0) == 0
    d = P.Context(128, "dirichlet", 1e-2, 1.0, s=8)
    assert d.workspace_bytes(4, 1) == 256          # Burgers plan: none for Dirichlet
    lib = P._lib
    # solve calls fail cleanly (ENOMEM: no workspace bound) before touching the device
    st = lib.pexp_solve_linear(c._h, 1, 1, 1.0, 4, 1e-8, 1, None)
    assert st == P.PEXP_ENOMEM
    assert b"workspace" in lib.pexp_last_error(c._h)
    st = lib.pexp_solve_linear(c._h, 1, 1, 1.0, 4, 1.0, 1, None)   # tol out of range
    assert st == P.PEXP_EINVAL
    st = lib.pexp_solve_burgers(d._h, 1, 1e-2, 1.0, 4, 1e-8, 30, 1, None)
    assert st == P.PEXP_EINVAL and b"periodic" in lib.pexp_last_error(d._h)


def test_struct_layout_matches_header(P, tmp_path):
    """The ctypes mirrors of pexp_options / pexp_stats have the C compiler's layout."""
    import subprocess
    fields_o = [f for f, _ in P.Options._fields_]
    fields_s = [f for f, _ in P.Stats._fields_]
    src = tmp_path / "layout.c"
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pexp.h"', "int main(void) {",
             'printf("%zu %zu\\n", sizeof(pexp_options), sizeof(pexp_stats));']
    lines += [f'printf("%zu\\n", offsetof(pexp_options, {f}));' for f in fields_o]
    lines += [f'printf("%zu\\n", offsetof(pexp_stats, {f}));' for f in fields_s]
    lines += ["return 0; }"]
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert vals[0] == C.sizeof(P.Options) and vals[1] == C.sizeof(P.Stats)
    offs = vals[2:]
    assert offs[:len(fields_o)] == [getattr(P.Options, f).offset for f in fields_o]
    assert offs[len(fields_o):] == [getattr(P.Stats, f).offset for f in fields_s]


def test_option_validation(P):
    for kw in ({"route": 3}, {"route": -1}, {"hom_group": 17}, {"defl_tol": -1.0}, {"piv_tol": -1.0}):
        with pytest.raises(P.PexpError):
            P.Context(64, "periodic", 1e-2, 1.0, **kw)
    P.Context(64, "periodic", 1e-2, 1.0, route=1, hom_group=16, defl_tol=1e-9, piv_tol=1e-13)


def test_no_environment_knobs_in_library(root):
    """Numerics and routing come from pexp_options only (SURVEY §5 'no env-var magic'); the one
    environment read left is the PEXP_SYNC fault-localisation switch (no numerical effect)."""
    csrc = os.path.join(root, "paper_1509_04567_b200", "csrc")
    reads = []
    for f in os.listdir(csrc):
        if f.endswith((".cu", ".cuh", ".h")):
            reads += re.findall(r'getenv\("(\w+)"\)', open(os.path.join(csrc, f)).read())
    assert reads == ["PEXP_SYNC"], reads
