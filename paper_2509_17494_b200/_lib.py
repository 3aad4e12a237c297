"""Loader for the in-tree CUDA library libhelmtg_b200.so (C-ABI: include/helmtg_b200.h).

There is no CPU fallback: if the library is missing or no GPU is present, the
product path raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
# HTG_LIB selects another build of the same library (kernel variants under exp/)
LIB_PATH = os.environ.get("HTG_LIB") or os.path.join(HERE, "libhelmtg_b200.so")
CSRC = os.path.join(HERE, "csrc")

HTG_OK, HTG_ERR_RUNTIME, HTG_ERR_INVALID, HTG_NOT_CONVERGED = 0, 1, 2, 3

# every symbol include/helmtg_b200.h declares
EXPORTS = (
    "htg_config_default", "htg_last_error", "htg_create", "htg_destroy", "htg_info", "htg_set_stream",
    "htg_residual", "htg_residual_norm", "htg_dd_step", "htg_csdd_smoother", "htg_restrict",
    "htg_residual_restrict", "htg_prolong_add", "htg_coarse_apply", "htg_coarse_solve", "htg_two_grid_step",
    "htg_solve", "htg_solve_host", "htg_two_grid_step_host", "htg_csdd_smoother_host",
    "htg_measure_fp64_tensor_peak", "htg_profile", "htg_launch_count", "htg_reset_launch_count",
)


class Problem(C.Structure):
    _fields_ = [("order", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("h", C.c_double),
                ("k_const", C.c_double), ("eps_const", C.c_double),
                ("k_cells", C.POINTER(C.c_double)), ("eps_cells", C.POINTER(C.c_double)),
                ("side_tags", C.c_int * 4),
                ("tags_bottom", C.POINTER(C.c_int)), ("tags_right", C.POINTER(C.c_int)),
                ("tags_top", C.POINTER(C.c_int)), ("tags_left", C.POINTER(C.c_int)),
                ("element_kind", C.c_int)]


HTG_ELEM_SQUARE, HTG_ELEM_TRIANGLE = 0, 1


class Config(C.Structure):
    _fields_ = [("alpha_s", C.c_double), ("alpha_c", C.c_double), ("n_s", C.c_int), ("n_dd", C.c_int),
                ("omega_c", C.c_double), ("l_dd", C.c_int), ("coarsening", C.c_int), ("smoother", C.c_int),
                ("outer", C.c_int), ("stop_rel_residual", C.c_double), ("max_iters", C.c_int)]


def build(verbose: bool = False) -> str:
    """Compile the CUDA library for sm_100a (nvcc cross-compiles without a GPU)."""
    out = subprocess.run(["make", "-s", "-j8", "-C", CSRC], capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError("building libhelmtg_b200.so failed:\n" + (out.stdout or "") + (out.stderr or ""))
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, dp, ip = C.c_void_p, C.c_void_p, C.POINTER(C.c_int)
    L.htg_last_error.restype = C.c_char_p
    L.htg_create.argtypes = [C.POINTER(Problem), C.POINTER(Config), vp, C.POINTER(vp)]
    L.htg_destroy.argtypes = [vp]
    L.htg_info.argtypes = [vp, C.POINTER(C.c_longlong)]
    L.htg_set_stream.argtypes = [vp, vp]
    L.htg_residual.argtypes = [vp, dp, dp, dp, C.c_int]
    L.htg_residual_norm.argtypes = [vp, dp, dp, C.POINTER(C.c_double)]
    L.htg_dd_step.argtypes = [vp, dp, dp, dp]
    L.htg_csdd_smoother.argtypes = [vp, dp, dp]
    L.htg_restrict.argtypes = [vp, dp, dp]
    L.htg_residual_restrict.argtypes = [vp, dp, dp, dp]
    L.htg_prolong_add.argtypes = [vp, dp, dp, C.c_double]
    L.htg_coarse_apply.argtypes = [vp, dp, dp]
    L.htg_coarse_solve.argtypes = [vp, dp, dp]
    L.htg_two_grid_step.argtypes = [vp, dp, dp]
    L.htg_solve.argtypes = [vp, dp, dp, dp, C.c_int, ip, ip]
    L.htg_solve_host.argtypes = [vp, dp, dp, dp, C.c_int, ip, ip]
    L.htg_two_grid_step_host.argtypes = [vp, dp, dp]
    L.htg_csdd_smoother_host.argtypes = [vp, dp, dp]
    L.htg_measure_fp64_tensor_peak.argtypes = [C.POINTER(C.c_double)]
    L.htg_profile.argtypes = [vp, dp, dp, C.c_int, C.POINTER(C.c_double)]
    L.htg_launch_count.restype = C.c_longlong
    L.htg_config_default.argtypes = [C.POINTER(Config)]
    _lib = L
    return L


class HtgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"helmtg_b200 error {code}: {msg}")
        self.code = code


def check(rc: int, allow_not_converged: bool = False) -> int:
    if rc == HTG_OK or (allow_not_converged and rc == HTG_NOT_CONVERGED):
        return rc
    raise HtgError(rc, lib().htg_last_error().decode())
