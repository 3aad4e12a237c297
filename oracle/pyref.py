"""ctypes binding of the reference itself (oracle/_ref/libhelmtg_ref.so).

The library is the reference's own hot-path sources
(/root/reference/proj/core/src/{basis,fespace,mesh,qsfem,twogrid,linalg,parallel}.cpp),
compiled unmodified against the Eigen-subset shim in oracle/eigen_shim by
oracle/Makefile.ref, plus the driver oracle/ref_capi.cpp.

TEST INFRASTRUCTURE ONLY: it pins the restated oracle (tests/test_ref_pins.py),
generates tests/golden/ref_*.npz (tools/make_ref_golden.py) and is the CPU
baseline of bench.py. It is never the product path.

The API mirrors ``oracle.pyoracle.Session`` so a test can run the same calls
against both.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .pyoracle import ProblemSpec, SolveResult, SolverConfig, _Cfg, _Desc, _Spec, cvec

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libhelmtg_ref.so")
REF_ROOT = "/root/reference/proj/core"
_lib = None


def available() -> bool:
    """True when the reference library exists or can be built here."""
    return os.path.exists(LIB_PATH) or os.path.isdir(REF_ROOT)


def build() -> str:
    """Compile the reference sources (only where /root/reference is present)."""
    if os.path.isdir(REF_ROOT):
        subprocess.run(["make", "-s", "-j8", "-f", "Makefile.ref", "-C", _HERE], check=True)
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} missing and {REF_ROOT} absent: cannot build the reference")
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        for name in ("ref_session_from_spec", "ref_session_from_desc"):
            getattr(_lib, name).argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        _lib.ref_session_free.argtypes = [C.c_void_p]
        _lib.ref_session_free.restype = None
        for name in ("ref_info", "ref_rhs", "ref_multiplicity", "ref_partition_sizes"):
            getattr(_lib, name).argtypes = [C.c_void_p, C.c_void_p]
        _lib.ref_coeffs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.ref_apply.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        _lib.ref_residual.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.ref_nnz.argtypes = [C.c_void_p, C.c_int]
        _lib.ref_export_csc.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        for name in ("ref_dd_step",):
            getattr(_lib, name).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        for name in ("ref_csdd", "ref_coarse_solve", "ref_two_grid_step", "ref_exact_smooth"):
            getattr(_lib, name).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.ref_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                   C.POINTER(C.c_int), C.POINTER(C.c_int)]
        _lib.ref_dirichlet.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        for name in ("ref_bench_csdd", "ref_bench_two_grid"):
            getattr(_lib, name).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_double)]
        _lib.ref_add_coarse_parts.argtypes = [C.c_void_p]
        _lib.ref_set_threads.argtypes = [C.c_int]
        _lib.ref_set_threads.restype = None
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def set_threads(n: int):
    lib().ref_set_threads(int(n))


class RefSession:
    """build_problem (+ setup_two_grid when a config is given) inside the reference."""

    def __init__(self, spec: ProblemSpec | None = None, config: SolverConfig | None = None, *,
                 desc: dict | None = None):
        L = lib()
        h = C.c_void_p()
        cfg = config._c() if config is not None else None
        cfgp = C.byref(cfg) if cfg is not None else None
        if desc is None:
            spec = spec or ProblemSpec()
            mask = 0
            for s in spec.layer_sides:
                mask |= 1 << s
            cs = _Spec(spec.order, spec.wavelengths, spec.ppw, (C.c_int * 4)(*spec.side_tags), mask,
                       spec.layer_width_dofs, spec.damping_D, spec.element_kind)
            _check(L.ref_session_from_spec(C.byref(cs), cfgp, C.byref(h)))
        else:
            nx, ny = desc["nx"], desc["ny"]
            self._k = np.ascontiguousarray(np.broadcast_to(np.asarray(desc["k"], float), (ny, nx)))
            self._e = np.ascontiguousarray(np.broadcast_to(np.asarray(desc.get("eps", 0.0), float), (ny, nx)))
            d = _Desc(desc["order"], nx, ny, desc["h"], self._k.ctypes.data_as(C.POINTER(C.c_double)),
                      self._e.ctypes.data_as(C.POINTER(C.c_double)), (C.c_int * 4)(*desc["side_tags"]),
                      int(desc.get("element_kind", 0)))
            _check(L.ref_session_from_desc(C.byref(d), cfgp, C.byref(h)))
        self._h = h
        self.config = config
        info = np.zeros(9, dtype=np.int64)
        _check(L.ref_info(h, _p(info)))
        (self.ndof, self.coarse_ndof, self.nx, self.ny, self.n_subdomains, self.n_factors,
         self.nnz_A, self.nnz_Ac, self.nnz_IP) = (int(v) for v in info)

    def add_coarse_parts(self):
        """A_c, IP, IP^H of the OptimizedFD level on a CoarseKind::None session (no coarse factor)."""
        _check(lib().ref_add_coarse_parts(self._h))
        info = np.zeros(9, dtype=np.int64)
        _check(lib().ref_info(self._h, _p(info)))
        self.coarse_ndof, self.nnz_Ac, self.nnz_IP = int(info[1]), int(info[7]), int(info[8])

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_session_free(self._h)
            self._h = None

    def rhs(self) -> np.ndarray:
        out = np.zeros(self.ndof, np.complex128)
        _check(lib().ref_rhs(self._h, _p(out)))
        return out

    def coeffs(self):
        k = np.zeros(self.nx * self.ny)
        e = np.zeros(self.nx * self.ny)
        _check(lib().ref_coeffs(self._h, _p(k), _p(e)))
        return k.reshape(self.ny, self.nx), e.reshape(self.ny, self.nx)

    # which = 0 A, 1 A_s, 2 A_c, 3 IP, 4 IP^H
    def apply(self, which: int, x) -> np.ndarray:
        x = cvec(x)
        m = {0: self.ndof, 1: self.ndof, 2: self.coarse_ndof, 3: self.ndof, 4: self.coarse_ndof}[which]
        y = np.zeros(m, np.complex128)
        _check(lib().ref_apply(self._h, which, _p(x), _p(y)))
        return y

    def residual(self, f, u, shifted: bool = False) -> np.ndarray:
        f, u = cvec(f), cvec(u)
        r = np.zeros(self.ndof, np.complex128)
        _check(lib().ref_residual(self._h, int(shifted), _p(f), _p(u), _p(r)))
        return r

    def csr(self, which: int):
        import scipy.sparse as sp
        nnz = lib().ref_nnz(self._h, which)
        if nnz < 0:
            _check(1)
        rows = self.ndof if which in (0, 1, 3) else self.coarse_ndof
        cols = self.coarse_ndof if which in (2, 3) else self.ndof
        cp = np.zeros(cols + 1, np.int32)
        ri = np.zeros(nnz, np.int32)
        v = np.zeros(nnz, np.complex128)
        _check(lib().ref_export_csc(self._h, which, _p(cp), _p(ri), _p(v)))
        return sp.csc_matrix((v, ri, cp), shape=(rows, cols)).tocsr()

    def dd_step(self, u, f) -> np.ndarray:
        u, f = cvec(u), cvec(f)
        out = np.zeros(self.ndof, np.complex128)
        _check(lib().ref_dd_step(self._h, _p(u), _p(f), _p(out)))
        return out

    def csdd_smoother(self, u, f) -> np.ndarray:
        u = cvec(u).copy()
        _check(lib().ref_csdd(self._h, _p(u), _p(cvec(f))))
        return u

    def exact_smooth(self, u, f) -> np.ndarray:
        u = cvec(u).copy()
        _check(lib().ref_exact_smooth(self._h, _p(u), _p(cvec(f))))
        return u

    def coarse_solve(self, rc) -> np.ndarray:
        rc = cvec(rc)
        uc = np.zeros(self.coarse_ndof, np.complex128)
        _check(lib().ref_coarse_solve(self._h, _p(rc), _p(uc)))
        return uc

    def two_grid_step(self, u, f) -> np.ndarray:
        u = cvec(u).copy()
        _check(lib().ref_two_grid_step(self._h, _p(u), _p(cvec(f))))
        return u

    def solve(self, f) -> SolveResult:
        f = cvec(f)
        u = np.zeros(self.ndof, np.complex128)
        cap = (self.config.max_iters if self.config else 200) + 1
        hist = np.zeros(cap)
        it, conv = C.c_int(), C.c_int()
        _check(lib().ref_solve(self._h, _p(f), _p(u), _p(hist), cap, C.byref(it), C.byref(conv)))
        return SolveResult(u, it.value, list(hist[: it.value]), bool(conv.value))

    def bench_csdd(self, u: np.ndarray, f, steps: int) -> float:
        """`steps` reference csdd_smoother sweeps in place on u; returns the loop's wall seconds."""
        assert u.dtype == np.complex128 and u.flags.c_contiguous and u.size == self.ndof
        t = C.c_double()
        _check(lib().ref_bench_csdd(self._h, _p(u), _p(cvec(f)), int(steps), C.byref(t)))
        return t.value

    def bench_two_grid(self, u: np.ndarray, f, steps: int) -> float:
        assert u.dtype == np.complex128 and u.flags.c_contiguous and u.size == self.ndof
        t = C.c_double()
        _check(lib().ref_bench_two_grid(self._h, _p(u), _p(cvec(f)), int(steps), C.byref(t)))
        return t.value

    def multiplicity(self) -> np.ndarray:
        out = np.zeros(self.ndof)
        _check(lib().ref_multiplicity(self._h, _p(out)))
        return out

    def partition_sizes(self) -> np.ndarray:
        out = np.zeros((self.n_subdomains, 2), np.int32)
        _check(lib().ref_partition_sizes(self._h, _p(out)))
        return out

    def dirichlet_dofs(self, coarse: bool = False) -> np.ndarray:
        cap = max(self.ndof, 1)
        out = np.zeros(cap, np.int32)
        n = lib().ref_dirichlet(self._h, int(coarse), _p(out), cap)
        if n < 0:
            _check(1)
        return out[:n].copy()
