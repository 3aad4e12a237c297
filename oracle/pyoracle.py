"""ctypes binding of the CPU oracle (oracle/build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs, always as the checker
or the CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

DIRICHLET, NEUMANN, ABSORBING = 0, 1, 2
LEFT, RIGHT, BOTTOM, TOP = 0, 1, 2, 3


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class _Spec(C.Structure):
    _fields_ = [("order", C.c_int), ("wavelengths", C.c_double), ("ppw", C.c_double),
                ("side", C.c_int * 4), ("layer_mask", C.c_uint),
                ("layer_width_dofs", C.c_double), ("damping_D", C.c_double), ("element_kind", C.c_int)]


class _Desc(C.Structure):
    _fields_ = [("order", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("h", C.c_double),
                ("k_cells", C.POINTER(C.c_double)), ("eps_cells", C.POINTER(C.c_double)),
                ("side", C.c_int * 4), ("element_kind", C.c_int)]


class _Cfg(C.Structure):
    _fields_ = [("alpha_s", C.c_double), ("alpha_c", C.c_double), ("n_s", C.c_int),
                ("n_dd", C.c_int), ("omega_c", C.c_double), ("l_dd", C.c_int),
                ("coarsening", C.c_int), ("smoother", C.c_int), ("outer", C.c_int),
                ("tol", C.c_double), ("max_iters", C.c_int)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_symbol.restype = C.c_double
        _lib.orc_symbol.argtypes = [C.c_double] * 3
        _lib.orc_stencil.argtypes = [C.c_double, C.c_void_p]
        _lib.orc_evaluate.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_double, C.c_double, C.c_void_p]
        for name in ("orc_session_from_spec", "orc_session_from_desc"):
            getattr(_lib, name).argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        _lib.orc_session_free.argtypes = [C.c_void_p]
        _lib.orc_session_free.restype = None
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def cvec(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


@dataclass
class SolverConfig:
    """proj/core/include/helmtg/twogrid.hpp:18-30 (same names and defaults)."""
    alpha_s: float = 0.2
    alpha_c: float = 0.0
    n_s: int = 1
    n_dd: int = 1
    omega_c: float = 1.0
    l_dd: int = 4
    coarsening: int = 0  # 0 OptimizedFD, 1 GalerkinP, 2 None
    smoother: int = 0  # 0 CSDD, 1 ExactShifted
    outer: int = 0  # 0 Richardson, 1 KrylovAccelerated (GMRES)
    stop_rel_residual: float = 1e-6
    max_iters: int = 200

    def _c(self) -> _Cfg:
        return _Cfg(self.alpha_s, self.alpha_c, self.n_s, self.n_dd, self.omega_c, self.l_dd,
                    self.coarsening, self.smoother, self.outer, self.stop_rel_residual, self.max_iters)


@dataclass
class ProblemSpec:
    """proj/core/include/helmtg/problem.hpp:16-29 (square elements)."""
    order: int = 4
    wavelengths: float = 20.0
    ppw: float = 10.0
    side_tags: tuple = (ABSORBING, ABSORBING, ABSORBING, ABSORBING)  # L, R, B, T
    layer_sides: tuple = ()
    layer_width_dofs: float = 40.0
    damping_D: float = 0.0
    element_kind: int = 0  # 0 squares, 1 triangles (the reference's ElementKind; the restated oracle: squares)


class Session:
    """A problem plus (optionally) its two-grid operators inside the oracle."""

    def __init__(self, spec: ProblemSpec | None = None, config: SolverConfig | None = None, *,
                 desc: dict | None = None):
        L = lib()
        h = C.c_void_p()
        cfg = config._c() if config is not None else None
        cfgp = C.byref(cfg) if cfg is not None else None
        if desc is None:
            spec = spec or ProblemSpec()
            if spec.element_kind != 0:
                raise ValueError("the restated oracle covers square elements; use oracle.pyref for triangles")
            mask = 0
            for s in spec.layer_sides:
                mask |= 1 << s
            cs = _Spec(spec.order, spec.wavelengths, spec.ppw, (C.c_int * 4)(*spec.side_tags), mask,
                       spec.layer_width_dofs, spec.damping_D, 0)
            _check(L.orc_session_from_spec(C.byref(cs), cfgp, C.byref(h)))
        else:
            nx, ny = desc["nx"], desc["ny"]
            self._k = np.ascontiguousarray(np.broadcast_to(np.asarray(desc["k"], float), (ny, nx)))
            self._e = np.ascontiguousarray(np.broadcast_to(np.asarray(desc.get("eps", 0.0), float), (ny, nx)))
            d = _Desc(desc["order"], nx, ny, desc["h"], self._k.ctypes.data_as(C.POINTER(C.c_double)),
                      self._e.ctypes.data_as(C.POINTER(C.c_double)), (C.c_int * 4)(*desc["side_tags"]), 0)
            if desc.get("element_kind", 0) != 0:
                raise ValueError("the restated oracle covers square elements; use oracle.pyref for triangles")
            _check(L.orc_session_from_desc(C.byref(d), cfgp, C.byref(h)))
        self._h = h
        self.config = config
        info = np.zeros(9, dtype=np.int64)
        _check(L.orc_info(h, _p(info)))
        (self.ndof, self.coarse_ndof, self.nx, self.ny, self.n_subdomains, self.n_factors,
         self.nnz_A, self.nnz_Ac, self.nnz_IP) = (int(v) for v in info)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib().orc_session_free(self._h)
            self._h = None

    # -- data
    def rhs(self) -> np.ndarray:
        out = np.zeros(self.ndof, np.complex128)
        _check(lib().orc_rhs(self._h, _p(out)))
        return out

    def coeffs(self):
        k = np.zeros(self.nx * self.ny)
        e = np.zeros(self.nx * self.ny)
        _check(lib().orc_coeffs(self._h, _p(k), _p(e)))
        return k.reshape(self.ny, self.nx), e.reshape(self.ny, self.nx)

    # -- operators: which = 0 A, 1 A_s, 2 A_c, 3 IP, 4 IP^H
    def apply(self, which: int, x) -> np.ndarray:
        x = cvec(x)
        m = {0: self.ndof, 1: self.ndof, 2: self.coarse_ndof, 3: self.ndof, 4: self.coarse_ndof}[which]
        y = np.zeros(m, np.complex128)
        _check(lib().orc_apply(self._h, which, _p(x), _p(y)))
        return y

    def residual(self, f, u, shifted: bool = False) -> np.ndarray:
        f, u = cvec(f), cvec(u)
        r = np.zeros(self.ndof, np.complex128)
        _check(lib().orc_residual(self._h, int(shifted), _p(f), _p(u), _p(r)))
        return r

    def csr(self, which: int):
        import scipy.sparse as sp
        nnz = lib().orc_nnz(self._h, which)
        if nnz < 0:
            _check(1)
        rows = self.ndof if which in (0, 1, 3) else self.coarse_ndof
        cols = self.coarse_ndof if which in (2, 3) else self.ndof
        rp = np.zeros(rows + 1, np.int32)
        ci = np.zeros(nnz, np.int32)
        v = np.zeros(nnz, np.complex128)
        _check(lib().orc_export_csr(self._h, which, _p(rp), _p(ci), _p(v)))
        return sp.csr_matrix((v, ci, rp), shape=(rows, cols))

    def build_matrix(self, kind: int, alpha: float = 0.0, weight: complex = 1.0):
        """kind 0 Helmholtz(alpha), 1 weighted mass, 2 boundary mass, 3 QSFEM (p=1 space)."""
        _check(lib().orc_build_matrix(self._h, kind, C.c_double(alpha), C.c_double(weight.real),
                                      C.c_double(complex(weight).imag)))
        import scipy.sparse as sp
        nnz = lib().orc_nnz(self._h, 0)
        rp = np.zeros(self.ndof + 1, np.int32)
        ci = np.zeros(nnz, np.int32)
        v = np.zeros(nnz, np.complex128)
        _check(lib().orc_export_csr(self._h, 0, _p(rp), _p(ci), _p(v)))
        return sp.csr_matrix((v, ci, rp), shape=(self.ndof, self.ndof))

    def dd_step(self, u, f) -> np.ndarray:
        u, f = cvec(u), cvec(f)
        out = np.zeros(self.ndof, np.complex128)
        _check(lib().orc_dd_step(self._h, _p(u), _p(f), _p(out)))
        return out

    def csdd_smoother(self, u, f) -> np.ndarray:
        u = cvec(u).copy()
        f = cvec(f)
        _check(lib().orc_csdd(self._h, _p(u), _p(f)))
        return u

    def coarse_solve(self, rc) -> np.ndarray:
        rc = cvec(rc)
        uc = np.zeros(self.coarse_ndof, np.complex128)
        _check(lib().orc_coarse_solve(self._h, _p(rc), _p(uc)))
        return uc

    def two_grid_step(self, u, f) -> np.ndarray:
        u = cvec(u).copy()
        f = cvec(f)
        _check(lib().orc_two_grid_step(self._h, _p(u), _p(f)))
        return u

    def solve(self, f):
        f = cvec(f)
        u = np.zeros(self.ndof, np.complex128)
        cap = (self.config.max_iters if self.config else 200) + 1
        hist = np.zeros(cap)
        it, conv = C.c_int(), C.c_int()
        _check(lib().orc_solve(self._h, _p(f), _p(u), _p(hist), cap, C.byref(it), C.byref(conv)))
        return SolveResult(u, it.value, list(hist[: it.value]), bool(conv.value))

    # -- structure
    def partition_info(self) -> np.ndarray:
        out = np.zeros((self.n_subdomains, 11), np.int32)
        _check(lib().orc_partition_info(self._h, _p(out)))
        return out

    def subdomain_maps(self, i: int):
        info = self.partition_info()[i]
        g = np.zeros(info[8], np.int32)
        u = np.zeros(info[9], np.int32)
        _check(lib().orc_subdomain_maps(self._h, i, _p(g), _p(u)))
        return g, u

    def multiplicity(self) -> np.ndarray:
        out = np.zeros(self.ndof)
        _check(lib().orc_multiplicity(self._h, _p(out)))
        return out

    def dirichlet_dofs(self, coarse: bool = False) -> np.ndarray:
        cap = max(self.ndof, 1)
        out = np.zeros(cap, np.int32)
        n = lib().orc_dirichlet(self._h, int(coarse), _p(out), cap)
        if n < 0:
            _check(1)
        return out[:n].copy()

    def find_dof(self, kind: str, x: int, y: int, off: int = 0, coarse: bool = False) -> int:
        return lib().orc_find_dof(self._h, int(coarse), ord(kind), int(x), int(y), int(off))

    def dof_keys(self, coarse: bool = False) -> np.ndarray:
        n = self.coarse_ndof if coarse else self.ndof
        out = np.zeros((n, 4), np.int32)
        _check(lib().orc_dof_keys(self._h, int(coarse), _p(out)))
        return out

    def evaluate(self, u, x: float, y: float, coarse: bool = False) -> complex:
        u = cvec(u)
        out = np.zeros(2)
        _check(lib().orc_evaluate(self._h, int(coarse), _p(u), x, y, _p(out)))
        return complex(out[0], out[1])


@dataclass
class SolveResult:
    u: np.ndarray
    iterations: int
    residual_history: list = field(default_factory=list)
    converged: bool = True


def element_matrices(p: int):
    n = (p + 1) ** 2
    K = np.zeros((n, n))
    M = np.zeros((n, n))
    _check(lib().orc_element(p, _p(K), _p(M)))
    return K, M


def edge_mass(p: int) -> np.ndarray:
    out = np.zeros((p + 1, p + 1))
    _check(lib().orc_edge_mass(p, _p(out)))
    return out


def stencil(eta: float) -> dict:
    out = np.zeros(5)
    _check(lib().orc_stencil(eta, _p(out)))
    return dict(eta=out[0], P0=out[1], P1=out[2], P2=out[3], N=out[4])


def stencil_symbol(eta: float, t1: float, t2: float) -> float:
    return lib().orc_symbol(eta, t1, t2)


def stage_interp(p: int, q: int):
    n = (p + 1) ** 2
    npts = 4 + 4 * (q - 1) + (q - 1) ** 2
    E = np.zeros((n, npts))
    pts = np.zeros((npts, 2))
    _check(lib().orc_stage_interp(p, q, _p(E), _p(pts)))
    return E, pts


def random_vector(n: int, seed: int) -> np.ndarray:
    out = np.zeros(n, np.complex128)
    _check(lib().orc_random_vector(n, seed, _p(out)))
    return out


def lu_solve_csr(A, b) -> np.ndarray:
    A = A.tocsr()
    n = A.shape[0]
    rp = np.ascontiguousarray(A.indptr, np.int32)
    ci = np.ascontiguousarray(A.indices, np.int32)
    v = cvec(A.data)
    b = cvec(b)
    x = np.zeros(n, np.complex128)
    _check(lib().orc_lu_solve_csr(n, _p(rp), _p(ci), _p(v), _p(b), _p(x)))
    return x


def set_threads(n: int):
    lib().orc_set_threads(n)
