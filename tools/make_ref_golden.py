"""Generate tests/golden/ref_*.npz: seeded inputs and the REFERENCE's outputs for
every hot-path entry point (run from the repo root: python tools/make_ref_golden.py).

The outputs come from the reference's own code: /root/reference/proj/core/src/
{basis,fespace,mesh,qsfem,twogrid,linalg,parallel}.cpp compiled unmodified
against the Eigen-subset shim (oracle/Makefile.ref -> oracle/_ref/libhelmtg_ref.so,
driven through oracle/pyref.py). The reference tree does not exist on the GPU box,
so the vectors are committed; tests/test_ref_golden_cpu.py checks the restated
oracle against them and tests/test_gpu_ref_golden.py checks the CUDA path.

Families cover p = 2, 4, 6, 8; absorbing / Dirichlet / Neumann sides and the sin^2
layer; n_s = 2, n_dd = 2, l_dd = 3; GalerkinP and ExactShifted; Richardson and
GMRES outer loops; a p = 6, 8 ppw solve; and rectangles
with per-cell random k and eps.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402
from oracle import pyref  # noqa: E402

A_, N_, D_ = po.ABSORBING, po.NEUMANN, po.DIRICHLET
L_, R_, B_, T_ = po.LEFT, po.RIGHT, po.BOTTOM, po.TOP

# name -> (spec dict | desc dict, config dict)
SPEC_CASES = {
    "ref_p2_abs_ns2": (dict(order=2, wavelengths=3, ppw=8), dict(n_s=2)),
    "ref_p4_abs": (dict(order=4, wavelengths=5, ppw=10), dict()),
    "ref_p4_dir_neu": (dict(order=4, wavelengths=4, ppw=10, side_tags=(D_, A_, N_, A_)), dict()),
    "ref_p4_layer": (dict(order=4, wavelengths=4, ppw=10, side_tags=(N_, A_, N_, A_), layer_sides=(L_, B_),
                          layer_width_dofs=12), dict()),
    "ref_p4_ndd2_ldd3": (dict(order=4, wavelengths=4, ppw=10), dict(n_dd=2, l_dd=3)),
    "ref_p4_krylov_dir": (dict(order=4, wavelengths=4, ppw=10, side_tags=(A_, D_, A_, N_)), dict(outer=1)),
    "ref_p4_galerkin": (dict(order=4, wavelengths=3, ppw=10, side_tags=(D_, A_, A_, A_)),
                        dict(coarsening=1, alpha_s=0.02, alpha_c=0.02)),
    "ref_p4_exact_krylov": (dict(order=4, wavelengths=3, ppw=10), dict(smoother=1, outer=1)),
    "ref_p6_abs": (dict(order=6, wavelengths=5, ppw=8), dict()),
    "ref_p6_ppw8_solve": (dict(order=6, wavelengths=8, ppw=8), dict()),
    "ref_p8_abs": (dict(order=8, wavelengths=4, ppw=12), dict()),
    "ref_p8_dir_krylov": (dict(order=8, wavelengths=3, ppw=16, side_tags=(D_, A_, N_, D_)), dict(outer=1)),
}
DESC_CASES = {
    "ref_rect_p4_hetero": (dict(order=4, nx=13, ny=7, h=0.05, side_tags=(A_, D_, N_, A_), kr=(8.0, 12.0), er=0.5,
                                seed=3), dict()),
    "ref_rect_p2_hetero_galerkin": (dict(order=2, nx=9, ny=16, h=1.0 / 16, side_tags=(D_, A_, A_, N_), kr=(5.0, 9.0),
                                         er=0.2, seed=4), dict(coarsening=1, alpha_c=0.05)),
    "ref_rect_p6_hetero_exact": (dict(order=6, nx=5, ny=4, h=0.1, side_tags=(N_, A_, A_, A_), kr=(6.0, 9.0), er=1.0,
                                      seed=5), dict(smoother=1, outer=1)),
}
# triangle meshes (ElementKind::Triangle): the restated oracle covers squares only,
# so these pin the product's host assembly (tests/test_tri_cpu.py) and its CUDA path
# (tests/test_gpu_ref_golden.py) to the reference's outputs
TRI_SPEC_CASES = {
    "reftri_p2_abs_ns2": (dict(order=2, wavelengths=3, ppw=8, element_kind=1), dict(n_s=2)),
    "reftri_p4_dir_neu": (dict(order=4, wavelengths=4, ppw=10, side_tags=(D_, A_, N_, A_), element_kind=1), dict()),
    "reftri_p4_galerkin_exact": (dict(order=4, wavelengths=3, ppw=10, side_tags=(A_, A_, D_, A_), element_kind=1),
                                 dict(coarsening=1, alpha_c=0.05, smoother=1, outer=1)),
    "reftri_p6_layer_krylov": (dict(order=6, wavelengths=3, ppw=8, side_tags=(N_, A_, A_, A_), layer_sides=(L_,),
                                    layer_width_dofs=8, element_kind=1), dict(outer=1)),
    "reftri_p8_abs": (dict(order=8, wavelengths=2, ppw=8, element_kind=1), dict()),
}
SPEC_CASES.update(TRI_SPEC_CASES)
DESC_CASES["reftri_rect_p4_hetero"] = (dict(order=4, nx=11, ny=7, h=0.07, side_tags=(A_, D_, N_, A_), kr=(8.0, 12.0),
                                            er=0.5, seed=6, element_kind=1), dict())


def desc_arrays(d):
    g = np.random.default_rng(d["seed"])
    k = g.uniform(*d["kr"], size=(d["ny"], d["nx"]))
    eps = d["er"] * g.random((d["ny"], d["nx"]))
    return k, eps


def make(name):
    if name in SPEC_CASES:
        spec, cfg = SPEC_CASES[name]
        ses = pyref.RefSession(po.ProblemSpec(**spec), po.SolverConfig(**cfg))
        extra = dict(spec=np.array(repr(spec)))
    else:
        d, cfg = DESC_CASES[name]
        k, eps = desc_arrays(d)
        ses = pyref.RefSession(desc=dict(order=d["order"], nx=d["nx"], ny=d["ny"], h=d["h"], k=k, eps=eps,
                                         side_tags=d["side_tags"], element_kind=d.get("element_kind", 0)),
                               config=po.SolverConfig(**cfg))
        extra = dict(desc=np.array(repr(d)), k_cells=k, eps_cells=eps)
    n, nc = ses.ndof, ses.coarse_ndof
    f, u = po.random_vector(n, 11), po.random_vector(n, 12)
    rc = po.random_vector(nc, 13)
    out = dict(f=f, u=u, rc=rc, rhs=ses.rhs(),
               residual=ses.residual(f, u), residual_shifted=ses.residual(f, u, shifted=True),
               restrict=ses.apply(4, f), prolong=ses.apply(3, rc), coarse_apply=ses.apply(2, rc),
               coarse_solve=ses.coarse_solve(rc), two_grid_step=ses.two_grid_step(u, f),
               dirichlet=ses.dirichlet_dofs(), nnz_A=np.array(ses.nnz_A))
    if cfg.get("smoother", 0) == 0:
        out["dd_step"] = ses.dd_step(u, f)
        out["csdd_smoother"] = ses.csdd_smoother(u, f)
        out["multiplicity"] = ses.multiplicity()
    else:
        out["exact_smooth"] = ses.exact_smooth(u, f)
    # the reference RHS for build_problem families, the seeded f for rectangles
    fs = out["rhs"] if name in SPEC_CASES else f
    res = ses.solve(fs)
    out["solve_f"] = fs
    out["solve_u"] = res.u
    out["solve_iterations"] = np.array(res.iterations)
    out["solve_history"] = np.array(res.residual_history)
    out["solve_converged"] = np.array(res.converged)
    out["config"] = np.array(repr(cfg))
    out.update(extra)
    return out


ALL = list(SPEC_CASES) + list(DESC_CASES)

if __name__ == "__main__":
    po.build()
    pyref.build()
    names = sys.argv[1:] or ALL
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    for name in names:
        o = make(name)
        np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"{name}.npz"), **o)
        print(f"wrote {name}: ndof {o['f'].size}, coarse {o['rc'].size}, iterations {int(o['solve_iterations'])}")
