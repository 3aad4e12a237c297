"""Generate tests/golden/*.npz: seeded inputs and the oracle's outputs for the hot-path
entry points on small problems (run from the repo root: python tools/make_golden.py).

The reference (C++, needs Eigen3) cannot be built here and ships no golden vectors
(SURVEY 8c), so these fixtures are outputs of the pinned CPU oracle (oracle/, itself
checked against the reference's known-answer tests). They freeze the oracle's
results: tests/test_golden.py re-derives them on the CPU (oracle drift) and
tests/test_gpu_golden.py checks the CUDA path against them without the oracle.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

A_, N_, D_ = po.ABSORBING, po.NEUMANN, po.DIRICHLET
CASES = {
    "p4_abs": (dict(order=4, wavelengths=3, ppw=10), dict()),
    "p2_dir_neu": (dict(order=2, wavelengths=3, ppw=8, side_tags=(D_, A_, N_, A_)), dict(n_s=2)),
    "p4_layer": (dict(order=4, wavelengths=4, ppw=10, side_tags=(N_, A_, N_, A_), layer_sides=(po.LEFT, po.BOTTOM),
                      layer_width_dofs=12), dict()),
    "p4_galerkin": (dict(order=4, wavelengths=3, ppw=10, side_tags=(D_, A_, A_, A_)),
                    dict(coarsening=1, alpha_s=0.02, alpha_c=0.02)),
    "p4_exact": (dict(order=4, wavelengths=3, ppw=10), dict(smoother=1, outer=1)),
}


def make(name):
    spec, cfg = CASES[name]
    ses = po.Session(po.ProblemSpec(**spec), po.SolverConfig(**cfg))
    n, nc = ses.ndof, ses.coarse_ndof
    f, u = po.random_vector(n, 11), po.random_vector(n, 12)
    rc = po.random_vector(nc, 13)
    out = dict(f=f, u=u, rc=rc, rhs=ses.rhs(),
               residual=ses.residual(f, u), residual_shifted=ses.residual(f, u, shifted=True),
               restrict=ses.apply(4, f), prolong=ses.apply(3, rc), coarse_apply=ses.apply(2, rc),
               coarse_solve=ses.coarse_solve(rc), two_grid_step=ses.two_grid_step(u, f))
    if cfg.get("smoother", 0) == 0:
        out["dd_step"] = ses.dd_step(u, f)
        out["csdd_smoother"] = ses.csdd_smoother(u, f)
    res = ses.solve(ses.rhs())
    out["solve_u"] = res.u
    out["solve_iterations"] = np.array(res.iterations)
    out["spec"] = np.array(repr(spec))
    out["config"] = np.array(repr(cfg))
    return out


if __name__ == "__main__":
    po.build()
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    for name in CASES:
        np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"{name}.npz"), **make(name))
        print("wrote", name)
