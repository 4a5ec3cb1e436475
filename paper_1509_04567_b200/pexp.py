"""Thin ctypes binding of libpexp.so (include/pexp.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  torch supplies device
memory (tensors, the workspace) and the stream.  There is NO fallback: if the library
is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpexp.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built — run `python -m paper_1509_04567_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

PEXP_OK, PEXP_EINVAL, PEXP_ENOMEM, PEXP_ECUDA, PEXP_ENOCONV, PEXP_EDIVERGED, PEXP_EPIVOT = range(7)
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENOCONV", 5: "EDIVERGED", 6: "EPIVOT"}
BC = {"periodic": 0, "dirichlet": 1}

EXPORTED = ["pexp_create", "pexp_create_batched", "pexp_destroy", "pexp_last_error", "pexp_sample_times",
            "pexp_workspace_bytes", "pexp_set_workspace", "pexp_solve_linear", "pexp_solve_burgers",
            "pexp_solve_burgers_forced", "pexp_solve_linear_stages", "pexp_wr_map",
            "pexp_chebyshev_taylor_matrix",
            "pexp_sai_solve", "pexp_source_svd", "pexp_expm_batched", "pexp_profile_enable", "pexp_profile_read"]
PROFILE_CLASSES = ["sai_solve", "xty", "combine", "small_problem", "small_dense", "stencil", "factor",
                   "arnoldi_step", "hom_scan", "small_hom", "stream_proj", "stream_update",
                   "scan_output"]


class Options(C.Structure):
    _fields_ = [("s", C.c_int32), ("node_rule", C.c_int32), ("svd_tau_factor", C.c_double),
                ("stop_factor", C.c_double), ("restart_blocks", C.c_int32), ("k_max", C.c_int32),
                ("stream", C.c_void_p), ("stop_rule", C.c_int32), ("basis_cols", C.c_int32),
                ("eval_chunk", C.c_int32), ("route", C.c_int32), ("defl_tol", C.c_double),
                ("piv_tol", C.c_double), ("hom_group", C.c_int32), ("width_buckets", C.c_int32),
                ("scan_gamma_factor", C.c_double), ("gamma_factor", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("wr_iters", C.c_int32), ("wr_last_delta", C.c_double), ("max_m", C.c_int32),
                ("max_k", C.c_int32), ("restarts", C.c_int32), ("best_residual", C.c_double),
                ("ms_total", C.c_float), ("evals", C.c_int32), ("kernel_launches", C.c_int32),
                ("host_syncs", C.c_int32), ("delta_hist", C.c_double * 64),
                ("m_j", C.POINTER(C.c_int32)), ("k_j", C.POINTER(C.c_int32)), ("gamma_j", C.POINTER(C.c_double)),
                ("kscan_j", C.POINTER(C.c_int32)), ("ms_nonhom", C.c_float), ("ms_hom", C.c_float),
                ("scan_steps", C.c_double), ("scan_checks", C.c_double), ("scan_check_cycles", C.c_double)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("delta_hist", "m_j", "k_j", "gamma_j", "kscan_j")}
        d["delta_hist"] = list(self.delta_hist[:min(max(self.wr_iters, 0), 64)])
        return d


def _records(nrec: int):
    """Caller-owned host arrays for the per-evaluation records of pexp_stats."""
    m = (C.c_int32 * nrec)()
    k = (C.c_int32 * nrec)()
    g = (C.c_double * nrec)()
    return m, k, g


_P = C.c_void_p
_lib.pexp_create.argtypes = [C.POINTER(_P), C.c_int64, C.c_int, C.c_double, C.c_double, C.POINTER(Options)]
_lib.pexp_create_batched.argtypes = [C.POINTER(_P), C.c_int64, C.c_int, C.c_int32, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(Options)]
_lib.pexp_destroy.argtypes = [_P]
_lib.pexp_destroy.restype = None
_lib.pexp_last_error.argtypes = [_P]
_lib.pexp_last_error.restype = C.c_char_p
_lib.pexp_sample_times.argtypes = [_P, C.c_double, C.c_int32, C.POINTER(C.c_double)]
_lib.pexp_workspace_bytes.argtypes = [_P, C.c_int32, C.c_int32]
_lib.pexp_workspace_bytes.restype = C.c_size_t
_lib.pexp_set_workspace.argtypes = [_P, _P, C.c_size_t]
_lib.pexp_solve_linear.argtypes = [_P, _P, _P, C.c_double, C.c_int32, C.c_double, _P, C.POINTER(Stats)]
_lib.pexp_solve_burgers.argtypes = [_P, _P, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_int32, _P,
                                    C.POINTER(Stats)]
_lib.pexp_solve_burgers_forced.argtypes = [_P, _P, _P, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_int32, _P,
                                           C.POINTER(Stats)]
_lib.pexp_solve_linear_stages.argtypes = [_P, _P, _P, _P, C.c_double, C.c_int32, C.c_double, _P, _P, _P,
                                          C.POINTER(Stats)]
_lib.pexp_wr_map.argtypes = [_P, _P, _P, _P, C.c_double, C.c_double, C.c_int32, C.c_double, _P, _P, C.POINTER(Stats)]
_lib.pexp_chebyshev_taylor_matrix.argtypes = [_P, C.c_double, C.POINTER(C.c_double)]
_lib.pexp_chebyshev_taylor_matrix.restype = C.c_int32
_lib.pexp_sai_solve.argtypes = [_P, C.c_int32, C.c_double, _P, C.c_int32, _P]
_lib.pexp_source_svd.argtypes = [_P, _P, C.c_int32, C.c_double, C.POINTER(C.c_int32), _P, _P]
_lib.pexp_expm_batched.argtypes = [_P, _P, C.c_int32, C.c_int32, _P]
_lib.pexp_profile_enable.argtypes = [C.c_int32]
_lib.pexp_profile_enable.restype = None
_lib.pexp_profile_read.argtypes = [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_int32)]
_lib.pexp_profile_read.restype = C.c_int32
for _f in EXPORTED:
    if _f not in ("pexp_destroy", "pexp_last_error", "pexp_workspace_bytes", "pexp_profile_enable",
                  "pexp_profile_read", "pexp_chebyshev_taylor_matrix"):
        getattr(_lib, _f).restype = C.c_int


class PexpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"pexp status {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _dev(t: torch.Tensor, name: str) -> int:
    if not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
    return t.data_ptr()


class Context:
    """One pexp context (an operator A = nu*D2 - a*D1 on n points, or a batch of them)."""

    def __init__(self, n: int, bc: str = "periodic", nu=1e-2, a=0.0, *, s: int = 32, k_max: int = 256,
                 svd_tau_factor: float = 0.01, stop_factor: float = 0.1, restart_blocks: int = 20,
                 stream: Optional[torch.cuda.Stream] = None, stop_rule: int = 0, basis_cols: int = 0,
                 eval_chunk: int = 0, route: int = 0, defl_tol: float = 0.0, piv_tol: float = 0.0,
                 hom_group: int = 0, width_buckets: int = 0, node_rule: int = 0, scan_gamma_factor: float = 0.0,
                 gamma_factor: float = 0.0):
        self.n, self.bc, self.s = int(n), bc, int(s)
        self._stream = stream
        nu = [float(v) for v in (nu if hasattr(nu, "__len__") else [nu])]
        a = [float(v) for v in (a if hasattr(a, "__len__") else [a])]
        if len(a) == 1 and len(nu) > 1:
            a = a * len(nu)
        self.batch = len(nu)
        handle = stream.cuda_stream if stream is not None else None  # None = legacy default stream
        self.opt = Options(self.s, int(node_rule), svd_tau_factor, stop_factor, restart_blocks, k_max, handle, stop_rule,
                           basis_cols, eval_chunk, route, defl_tol, piv_tol, hom_group, width_buckets,
                           scan_gamma_factor, gamma_factor)
        self._h = _P()
        arr = C.c_double * self.batch
        st = _lib.pexp_create_batched(C.byref(self._h), self.n, BC[bc], self.batch, arr(*nu), arr(*a),
                                      C.byref(self.opt))
        if st != 0:
            raise PexpError(st, "pexp_create_batched rejected the arguments")
        self._ws = None
        self._ws_P = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.pexp_destroy(h)
            self._h = _P()

    def _check(self, st):
        if st != 0:
            raise PexpError(st, _lib.pexp_last_error(self._h).decode())

    def workspace_bytes(self, P: int, kind: int = 0) -> int:
        return int(_lib.pexp_workspace_bytes(self._h, int(P), int(kind)))

    def ensure_workspace(self, P: int, device="cuda", kind: int = 0):
        need = self.workspace_bytes(P, kind)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need + 256, dtype=torch.uint8, device=device)
            ptr = (self._ws.data_ptr() + 255) & ~255
            self._check(_lib.pexp_set_workspace(self._h, ptr, need))
        return need

    def sample_times(self, T: float, P: int) -> torch.Tensor:
        t = torch.empty(P * self.s, dtype=torch.float64)
        self._check(_lib.pexp_sample_times(self._h, float(T), int(P), C.cast(t.data_ptr(), C.POINTER(C.c_double))))
        return t.view(P, self.s)

    def chebyshev_taylor_matrix(self, dT: float) -> torch.Tensor:
        """pexp_chebyshev_taylor_matrix (node_rule = 1, host-only): tensor [s-1][12][s]."""
        D = torch.empty((self.s - 1) * 12 * self.s, dtype=torch.float64)
        nq = _lib.pexp_chebyshev_taylor_matrix(self._h, float(dT), C.cast(D.data_ptr(), C.POINTER(C.c_double)))
        if nq != 12:
            raise PexpError(PEXP_EINVAL, "pexp_chebyshev_taylor_matrix: needs a node_rule = 1 context")
        return D.view(self.s - 1, 12, self.s)

    def solve_linear(self, u0: torch.Tensor, src: torch.Tensor, T: float, P: int, tol: float,
                     out: Optional[torch.Tensor] = None, records: bool = False):
        self.ensure_workspace(P, u0.device)
        if out is None:
            out = torch.empty((self.batch, P, self.n), dtype=torch.float64, device=u0.device)
        st = Stats()
        if records:
            rm, rk, rg = _records(self.batch * P)
            st.m_j, st.k_j, st.gamma_j = (C.cast(rm, C.POINTER(C.c_int32)), C.cast(rk, C.POINTER(C.c_int32)),
                                           C.cast(rg, C.POINTER(C.c_double)))
        self._check(_lib.pexp_solve_linear(self._h, _dev(u0, "u0"), _dev(src, "src"), float(T), int(P), float(tol),
                                           _dev(out, "out"), C.byref(st)))
        d = st.as_dict()
        if records:
            d["m_j"], d["k_j"], d["gamma_j"] = list(rm), list(rk), list(rg)
        return out, d

    def solve_burgers(self, u0: torch.Tensor, nu: float, T: float, P: int, tol: float, max_wr_iters: int = 30,
                      out: Optional[torch.Tensor] = None, records: bool = False,
                      f: Optional[torch.Tensor] = None):
        """f: forcing samples [P][s][n] at the sample nodes (pexp_solve_burgers_forced), None = unforced."""
        self.ensure_workspace(P, u0.device, kind=1)
        if f is not None and tuple(f.shape) != (P, self.s, self.n):
            raise ValueError("f must have shape [P][s][n]")
        if out is None:
            out = torch.empty((P, self.n), dtype=torch.float64, device=u0.device)
        st = Stats()
        if records:
            rm, rk, rg = _records(int(max_wr_iters) * P)
            rs = (C.c_int32 * (int(max_wr_iters) * P))()
            st.m_j, st.k_j, st.gamma_j = (C.cast(rm, C.POINTER(C.c_int32)), C.cast(rk, C.POINTER(C.c_int32)),
                                           C.cast(rg, C.POINTER(C.c_double)))
            st.kscan_j = C.cast(rs, C.POINTER(C.c_int32))
        if f is None:
            self._check(_lib.pexp_solve_burgers(self._h, _dev(u0, "u0"), float(nu), float(T), int(P), float(tol),
                                                int(max_wr_iters), _dev(out, "out"), C.byref(st)))
        else:
            self._check(_lib.pexp_solve_burgers_forced(self._h, _dev(u0, "u0"), _dev(f, "f"), float(nu), float(T),
                                                       int(P), float(tol), int(max_wr_iters), _dev(out, "out"),
                                                       C.byref(st)))
        d = st.as_dict()
        if records:
            K = d["wr_iters"]
            d["m_j"] = [list(rm[k * P:(k + 1) * P]) for k in range(K)]
            d["k_j"] = [list(rk[k * P:(k + 1) * P]) for k in range(K)]
            d["gamma_j"] = [list(rg[k * P:(k + 1) * P]) for k in range(K)]
            d["kscan_j"] = [list(rs[k * P:(k + 1) * P]) for k in range(K)]
        return out, d

    def solve_linear_stages(self, u0, src, T, P, tol, vstart=None, hom_group=None):
        """pexp_solve_linear_stages: returns (out, vend [batch][P][n], legs [batch][G][P][n], stats)."""
        self.ensure_workspace(P, u0.device)
        hg = self.opt.hom_group if self.opt.hom_group > 0 else 8
        G = max(1, -(-(P - 1) // max(1, min(hg, P - 1)))) if P > 1 else 1
        out = torch.empty((self.batch, P, self.n), dtype=torch.float64, device=u0.device)
        vend = torch.empty_like(out)
        legs = torch.zeros((self.batch, G, P, self.n), dtype=torch.float64, device=u0.device)
        st = Stats()
        self._check(_lib.pexp_solve_linear_stages(
            self._h, _dev(u0, "u0"), None if src is None else _dev(src, "src"),
            None if vstart is None else _dev(vstart, "vstart"), float(T), int(P), float(tol), _dev(out, "out"),
            _dev(vend, "vend"), _dev(legs, "legs"), C.byref(st)))
        return out, vend, legs, st.as_dict()

    def wr_map(self, u0, Uk, nu, T, P, tol, f=None):
        """pexp_wr_map: one WR map u_k -> u_{k+1}; returns (Unew [P][s][n], out [P][n], stats)."""
        self.ensure_workspace(P, u0.device, kind=1)
        Unew = torch.empty_like(Uk)
        out = torch.empty((P, self.n), dtype=torch.float64, device=u0.device)
        st = Stats()
        self._check(_lib.pexp_wr_map(self._h, _dev(u0, "u0"), None if f is None else _dev(f, "f"), _dev(Uk, "Uk"),
                                     float(nu), float(T), int(P), float(tol), _dev(Unew, "Unew"), _dev(out, "out"),
                                     C.byref(st)))
        return Unew, out, st.as_dict()

    def sai_solve(self, b: int, gamma: float, rhs: torch.Tensor) -> torch.Tensor:
        self.ensure_workspace(1, rhs.device)
        rhs = rhs.reshape(-1, self.n).contiguous()
        x = torch.empty_like(rhs)
        self._check(_lib.pexp_sai_solve(self._h, int(b), float(gamma), _dev(rhs, "rhs"), rhs.shape[0], _dev(x, "x")))
        return x

    def source_svd(self, G: torch.Tensor, tol: float):
        E = G.shape[0]
        P = -(-E // self.batch)
        self.ensure_workspace(P, G.device)
        m = (C.c_int32 * E)()
        sig = torch.empty((E, self.s), dtype=torch.float64, device=G.device)
        proj = torch.empty_like(G)
        self._check(_lib.pexp_source_svd(self._h, _dev(G, "G"), E, float(tol), m, _dev(sig, "sigma"),
                                         _dev(proj, "proj")))
        return list(m), sig, proj

    def expm_batched(self, A: torch.Tensor) -> torch.Tensor:
        E, N, _ = A.shape
        need = min(E, 148) * (7 * N * N * 8 + N * 4) + 1024 + 4096
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need + 256, dtype=torch.uint8, device=A.device)
            ptr = (self._ws.data_ptr() + 255) & ~255
            self._check(_lib.pexp_set_workspace(self._h, ptr, need))
        At = A.transpose(1, 2).contiguous()  # column-major per matrix
        X = torch.empty_like(At)
        self._check(_lib.pexp_expm_batched(self._h, _dev(At, "A"), E, N, _dev(X, "X")))
        return X.transpose(1, 2).contiguous()


def profile_enable(on: bool = True) -> None:
    _lib.pexp_profile_enable(1 if on else 0)


def profile_read() -> dict:
    k = len(PROFILE_CLASSES)
    ms, by, fl = (C.c_double * k)(), (C.c_double * k)(), (C.c_double * k)()
    nl = (C.c_int32 * k)()
    if _lib.pexp_profile_read(k, ms, by, fl, nl) < 0:
        raise PexpError(PEXP_ECUDA, "profile read failed")
    return {name: {"ms": ms[i], "bytes": by[i], "flops": fl[i], "launches": nl[i]}
            for i, name in enumerate(PROFILE_CLASSES)}
