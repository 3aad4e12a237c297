"""B200-native two-grid Helmholtz hot path (arXiv 2509.17494, reference helmtg).

The compute runs in the in-tree CUDA library ``libhelmtg_b200.so`` behind the
C-ABI of ``include/helmtg_b200.h``; this package is the host-side mirror of
the reference's two-grid interface.
"""
from ._lib import HtgError, build  # noqa: F401
from .twogrid import (  # noqa: F401
    ABSORBING, BOTTOM, CSDD, DIRICHLET, EXACT_SHIFTED, GALERKIN_P, KRYLOV, LEFT, NEUMANN, NONE, OPTIMIZED_FD,
    RICHARDSON, RIGHT, TOP,
    Problem, ProblemSpec, SolveResult, SolverConfig, TwoGridOperators, build_problem, dirichlet_mask,
    dof_index, fp64_tensor_peak_tflops, launch_count, reset_launch_count, setup_two_grid,
)
