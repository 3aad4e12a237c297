"""Host-side mirror of the reference two-grid API over the C-ABI.

Names, argument meaning and error behaviour follow
proj/core/include/helmtg/twogrid.hpp and proj/core/include/helmtg/problem.hpp:
``build_problem`` (commands.cpp:14-39), ``SolverConfig`` (twogrid.hpp:18-30),
``setup_two_grid`` (twogrid.hpp:107-108) returning ``TwoGridOperators`` with
``two_grid_step`` / ``solve`` / ``csdd_smoother`` / ``dd_step`` and the
operator, transfer and coarse entry points of the hot path.

Device vectors are ``torch.complex128`` CUDA tensors in the reference dof
order; host vectors are ``numpy.complex128`` arrays. PyTorch is only used for
device memory and streams; every operation runs in libhelmtg_b200.so.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import HtgError, check, lib

DIRICHLET, NEUMANN, ABSORBING = 0, 1, 2
LEFT, RIGHT, BOTTOM, TOP = 0, 1, 2, 3
OPTIMIZED_FD, GALERKIN_P, NONE = 0, 1, 2
SQUARE, TRIANGLE = 0, 1  # element kinds (proj/core/include/helmtg/mesh.hpp ElementKind)
CSDD, EXACT_SHIFTED = 0, 1
RICHARDSON, KRYLOV = 0, 1


@dataclass
class SolverConfig:
    alpha_s: float = 0.2
    alpha_c: float = 0.0
    n_s: int = 1
    n_dd: int = 1
    omega_c: float = 1.0
    l_dd: int = 4
    coarsening: int = OPTIMIZED_FD
    smoother: int = CSDD
    outer: int = RICHARDSON
    stop_rel_residual: float = 1e-6
    max_iters: int = 200

    def _c(self) -> _lib.Config:
        return _lib.Config(self.alpha_s, self.alpha_c, self.n_s, self.n_dd, self.omega_c, self.l_dd,
                           self.coarsening, self.smoother, self.outer, self.stop_rel_residual, self.max_iters)


@dataclass
class ProblemSpec:
    """proj/core/include/helmtg/problem.hpp:16-29 (square elements)."""
    order: int = 4
    wavelengths: float = 20.0
    ppw: float = 10.0
    side_tags: tuple = (ABSORBING, ABSORBING, ABSORBING, ABSORBING)  # left, right, bottom, top
    layer_sides: tuple = ()
    layer_width_dofs: float = 40.0
    damping_D: float = 0.0
    element_kind: int = 0  # SQUARE (0) or TRIANGLE (1)


@dataclass
class Problem:
    """Unit-square problem: mesh size, per-cell k and eps, tags, point-load RHS."""
    order: int
    n_cells: int
    h: float
    k: float
    k_cells: np.ndarray
    eps_cells: np.ndarray
    side_tags: tuple
    rhs: np.ndarray = field(repr=False)
    ny: int | None = None  # cells in y (None: n_cells, the unit square of build_problem)
    element_kind: int = 0  # SQUARE, or TRIANGLE: cells split along the (0,0)-(1,1) diagonal

    @property
    def ndof(self) -> int:
        ny = self.ny or self.n_cells
        return (self.n_cells * self.order + 1) * (ny * self.order + 1)


def dof_index(nx: int, ny: int, p: int, gx, gy):
    """Reference dof number of the tensor pair (gx, gy) (proj/core/src/fespace.cpp:37-54)."""
    gx = np.asarray(gx)
    gy = np.asarray(gy)
    x, jx = gx // p, gx % p
    y, jy = gy // p, gy % p
    row = nx * p * p + p
    base = y * row + np.where(y < ny, x * p * p, x * p)
    return np.where((jx == 0) & (jy == 0), base,
                    np.where(jy == 0, base + jx,
                             np.where(jx == 0, base + np.where(x < nx, p, 1) + jy - 1,
                                      base + 2 * p - 1 + (jx - 1) * (p - 1) + (jy - 1))))


def layer_epsilon(k: float, depth, width: float):
    """sin^2 ramp up to 2 k^2 / pi (proj/core/src/mesh.cpp:225-230)."""
    d = np.clip(depth, 0.0, width)
    s = np.sin(np.pi / 2.0 * d / width)
    return np.where(d > 0.0, 2.0 * k * k / np.pi * s * s, 0.0)


def build_problem(spec: ProblemSpec) -> Problem:
    """proj/core/src/commands.cpp:14-39: k = 2 pi W, n = round(W ppw / p), point load at (n/2, n/2)."""
    p = spec.order
    if p < 2 or p > 8 or p % 2:
        raise HtgError(_lib.HTG_ERR_INVALID, "build_space: order must be even, 2 <= p <= 8")
    k = 2.0 * math.pi * spec.wavelengths
    n = int(math.floor(spec.wavelengths * spec.ppw / p + 0.5))  # lround (positive values)
    if n < 2:
        raise HtgError(_lib.HTG_ERR_INVALID, "build_problem: domain under-resolved")
    h = 1.0 / n
    eps_vol = k * k * spec.damping_D / math.pi
    kc = np.full((n, n), k)
    if not spec.layer_sides:
        ec = np.full((n, n), eps_vol)
    else:
        cells = int(math.ceil(spec.layer_width_dofs / p - 1e-12))
        width = cells * h
        if width > n * h:
            raise HtgError(_lib.HTG_ERR_INVALID, "absorbing_layer: layer wider than domain")
        yy, xx = np.mgrid[0:n, 0:n]
        d = np.zeros((n, n))
        for s in spec.layer_sides:
            dist = {LEFT: (xx + 0.5) * h, RIGHT: (n - 1 - xx + 0.5) * h,
                    BOTTOM: (yy + 0.5) * h, TOP: (n - 1 - yy + 0.5) * h}[s]
            d = np.maximum(d, width - dist)
        ec = layer_epsilon(k, d, width)
        if eps_vol > 0.0:
            ec = ec + eps_vol
    ndof = (n * p + 1) ** 2
    rhs = np.zeros(ndof, np.complex128)
    rhs[int(dof_index(n, n, p, (n // 2) * p, (n // 2) * p))] = 1.0
    tags = tuple(spec.side_tags)
    if DIRICHLET in tags:
        rhs[dirichlet_mask(n, n, p, tags)] = 0.0
    return Problem(p, n, h, k, kc, ec, tags, rhs, element_kind=spec.element_kind)


def dirichlet_mask(nx: int, ny: int, p: int, side_tags) -> np.ndarray:
    """Dofs in the closure of Dirichlet sides (proj/core/src/fespace.cpp:146-153)."""
    gx = np.arange(nx * p + 1)
    gy = np.arange(ny * p + 1)
    X, Y = np.meshgrid(gx, gy)
    m = np.zeros_like(X, dtype=bool)
    if side_tags[LEFT] == DIRICHLET:
        m |= X == 0
    if side_tags[RIGHT] == DIRICHLET:
        m |= X == nx * p
    if side_tags[BOTTOM] == DIRICHLET:
        m |= Y == 0
    if side_tags[TOP] == DIRICHLET:
        m |= Y == ny * p
    out = np.zeros((nx * p + 1) * (ny * p + 1), bool)
    out[dof_index(nx, ny, p, X[m], Y[m])] = True
    return out


def _dptr(t, n: int | None = None, device: int | None = None) -> C.c_void_p:
    """Device pointer of a contiguous complex128 CUDA tensor of exactly n entries on the
    handle's device (the C-ABI reads/writes n entries: a short tensor would be overrun)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.complex128 and t.is_contiguous()):
        raise HtgError(_lib.HTG_ERR_INVALID, "device vectors must be contiguous complex128 CUDA tensors")
    if n is not None and t.numel() != n:
        raise HtgError(_lib.HTG_ERR_INVALID, f"device vector has {t.numel()} entries, expected {n}")
    if device is not None and t.device.index != device:
        raise HtgError(_lib.HTG_ERR_INVALID, f"device vector on cuda:{t.device.index}, handle on cuda:{device}")
    return C.c_void_p(t.data_ptr())


def _hptr(a: np.ndarray, n: int | None = None) -> C.c_void_p:
    if not (isinstance(a, np.ndarray) and a.dtype == np.complex128 and a.flags.c_contiguous):
        raise HtgError(_lib.HTG_ERR_INVALID, "host vectors must be contiguous complex128 arrays")
    if n is not None and a.size != n:
        raise HtgError(_lib.HTG_ERR_INVALID, f"host vector has {a.size} entries, expected {n}")
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class SolveResult:
    u: object
    iterations: int
    residual_history: list
    converged: bool


class TwoGridOperators:
    """GPU-resident operators of one problem (one handle of the C-ABI)."""

    def __init__(self, problem: Problem, config: SolverConfig, stream=None):
        L = lib()
        self.problem = problem
        self.config = config
        self._k = np.ascontiguousarray(problem.k_cells, dtype=np.float64)
        self._e = np.ascontiguousarray(problem.eps_cells, dtype=np.float64)
        n = problem.n_cells
        cp = _lib.Problem(problem.order, n, problem.ny or n, problem.h, problem.k, 0.0,
                          self._k.ctypes.data_as(C.POINTER(C.c_double)),
                          self._e.ctypes.data_as(C.POINTER(C.c_double)),
                          (C.c_int * 4)(*problem.side_tags), None, None, None, None, int(problem.element_kind))
        cfg = config._c()
        h = C.c_void_p()
        import torch
        self.device = torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream()  # order the handle with torch's work
        st = C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        check(L.htg_create(C.byref(cp), C.byref(cfg), st, C.byref(h)))
        self._h = h
        info = (C.c_longlong * 20)()
        check(L.htg_info(h, info))
        (self.ndof, self.coarse_ndof, self.n_subdomains, self.n_classes, self.device_bytes,
         self.coarse_factor_bytes) = (int(v) for v in info[:6])
        self.dd_flops = int(info[9])
        self.coarse_levels = int(info[10])
        self.dd_flops_dense = int(info[11])
        self.fdm_subdomains = int(info[12])
        self.sum_u, self.sum_omega, self.coarse_read_bytes = int(info[14]), int(info[15]), int(info[16])
        self.band_subdomains, self.band_factor_bytes = int(info[17]), int(info[18])
        self.device_inverse_classes = int(info[19])

    def _f(self, t):  # fine-space device vector
        return _dptr(t, self.ndof, self.device)

    def _c(self, t):  # coarse-space device vector
        return _dptr(t, self.coarse_ndof, self.device)

    @property
    def cached_graphs(self) -> int:
        info = (C.c_longlong * 20)()
        check(lib().htg_info(self._h, info))
        return int(info[13])

    def close(self):
        if getattr(self, "_h", None):
            lib().htg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream):
        check(lib().htg_set_stream(self._h, C.c_void_p(stream.cuda_stream)))

    # ---------------------------------------------------------------- device API
    def residual(self, f, u, r, shifted: bool = False):
        check(lib().htg_residual(self._h, self._f(f), self._f(u), self._f(r), int(shifted)))
        return r

    def residual_norm(self, f, u) -> float:
        out = C.c_double()
        check(lib().htg_residual_norm(self._h, self._f(f), self._f(u), C.byref(out)))
        return out.value

    def dd_step(self, u, f, out):
        check(lib().htg_dd_step(self._h, self._f(u), self._f(f), self._f(out)))
        return out

    def csdd_smoother(self, u, f):
        check(lib().htg_csdd_smoother(self._h, self._f(u), self._f(f)))
        return u

    def restrict(self, r, rc):
        check(lib().htg_restrict(self._h, self._f(r), self._c(rc)))
        return rc

    def residual_restrict(self, f, u, rc):
        check(lib().htg_residual_restrict(self._h, self._f(f), self._f(u), self._c(rc)))
        return rc

    def prolong_add(self, u, uc, omega: float):
        check(lib().htg_prolong_add(self._h, self._f(u), self._c(uc), float(omega)))
        return u

    def coarse_apply(self, x, y):
        check(lib().htg_coarse_apply(self._h, self._c(x), self._c(y)))
        return y

    def coarse_solve(self, rc, uc):
        check(lib().htg_coarse_solve(self._h, self._c(rc), self._c(uc)))
        return uc

    def two_grid_step(self, u, f):
        check(lib().htg_two_grid_step(self._h, self._f(u), self._f(f)))
        return u

    def solve(self, f, u=None) -> SolveResult:
        import torch
        if u is None:
            u = torch.zeros_like(f)
        cap = self.config.max_iters + 1
        hist = np.zeros(cap)
        it, conv = C.c_int(), C.c_int()
        check(lib().htg_solve(self._h, self._f(f), self._f(u), hist.ctypes.data_as(C.c_void_p), cap, C.byref(it),
                              C.byref(conv)), allow_not_converged=True)
        return SolveResult(u, it.value, list(hist[: it.value]), bool(conv.value))

    def profile(self, u, f, reps: int = 10) -> dict:
        """Mean device time (ms) of each hot-path phase (CUDA events, handle stream)."""
        ms = (C.c_double * 13)()
        check(lib().htg_profile(self._h, self._f(u), self._f(f), int(reps), ms))
        keys = ("residual", "dd_gemm", "dd_combine", "residual_restrict", "coarse_solve", "prolong",
                "residual_norm", "smoother_sweep", "two_grid_step", "coarse_apply", "smoother_sweep_graph",
                "two_grid_step_graph", "coarse_solve_graph")
        return dict(zip(keys, list(ms)))

    # ---------------------------------------------------------------- host API
    def solve_host(self, f: np.ndarray) -> SolveResult:
        f = np.ascontiguousarray(f, dtype=np.complex128)
        u = np.zeros_like(f)
        cap = self.config.max_iters + 1
        hist = np.zeros(cap)
        it, conv = C.c_int(), C.c_int()
        check(lib().htg_solve_host(self._h, _hptr(f, self.ndof), _hptr(u, self.ndof), hist.ctypes.data_as(C.c_void_p), cap, C.byref(it),
                                   C.byref(conv)), allow_not_converged=True)
        return SolveResult(u, it.value, list(hist[: it.value]), bool(conv.value))

    def two_grid_step_host(self, u: np.ndarray, f: np.ndarray) -> np.ndarray:
        check(lib().htg_two_grid_step_host(self._h, _hptr(u, self.ndof), _hptr(f, self.ndof)))
        return u

    def csdd_smoother_host(self, u: np.ndarray, f: np.ndarray) -> np.ndarray:
        check(lib().htg_csdd_smoother_host(self._h, _hptr(u, self.ndof), _hptr(f, self.ndof)))
        return u


def setup_two_grid(problem: Problem, config: SolverConfig | None = None, stream=None) -> TwoGridOperators:
    return TwoGridOperators(problem, config or SolverConfig(), stream)


def launch_count() -> int:
    return int(lib().htg_launch_count())


def reset_launch_count() -> None:
    lib().htg_reset_launch_count()


def fp64_tensor_peak_tflops() -> float:
    out = C.c_double()
    check(lib().htg_measure_fp64_tensor_peak(C.byref(out)))
    return out.value
