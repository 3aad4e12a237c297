"""Triangle meshes (ElementKind::Triangle: every cell split along its (0,0)-(1,1)
diagonal, hierarchical P_p elements, proj/core/src/basis.cpp:147-252,
fespace.cpp:85-108) through the CUDA path, against the REFERENCE's own code
(oracle/_ref: proj/core/src/*.cpp compiled unmodified). The restated oracle covers
squares only, so every check here is against the reference itself.
North-star tolerances: relative l2 <= 1e-10 per operation, iteration counts within +-1."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
A_, N_, D_ = po.ABSORBING, po.NEUMANN, po.DIRICHLET
TOL = 1e-10
CASES = {
    "p2_abs": (dict(order=2, wavelengths=3, ppw=8), dict()),
    "p4_abs": (dict(order=4, wavelengths=4, ppw=10), dict()),
    "p4_dir_neu": (dict(order=4, wavelengths=4, ppw=10, side_tags=(D_, A_, N_, A_)), dict()),
    "p4_layer_ns2": (dict(order=4, wavelengths=4, ppw=10, side_tags=(N_, A_, N_, A_), layer_sides=(po.LEFT, po.BOTTOM),
                          layer_width_dofs=12), dict(n_s=2)),
    "p4_ldd3_ndd2": (dict(order=4, wavelengths=4, ppw=10), dict(l_dd=3, n_dd=2)),
    "p6_abs_krylov": (dict(order=6, wavelengths=3, ppw=8), dict(outer=1)),
    "p8_dir": (dict(order=8, wavelengths=2, ppw=8, side_tags=(A_, D_, A_, D_)), dict()),
    "p4_exact_krylov": (dict(order=4, wavelengths=3, ppw=10), dict(smoother=1, outer=1)),
    "p4_galerkin_dir": (dict(order=4, wavelengths=3, ppw=10, side_tags=(D_, A_, A_, A_)),
                        dict(coarsening=1, alpha_s=0.02, alpha_c=0.02)),
    "p6_galerkin_exact": (dict(order=6, wavelengths=2, ppw=8), dict(coarsening=1, alpha_c=0.05, smoother=1, outer=1)),
    "p8_galerkin": (dict(order=8, wavelengths=2, ppw=8, side_tags=(A_, N_, D_, A_)), dict(coarsening=1, alpha_c=0.1)),
}


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def ref_lib():
    from oracle import pyref
    if not os.path.exists(pyref.LIB_PATH):
        pytest.skip("oracle/_ref/libhelmtg_ref.so not built")
    pyref.set_threads(os.cpu_count() or 1)
    return pyref


@pytest.mark.parametrize("name", list(CASES))
def test_triangles_match_reference(name, ref_lib):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_17494_b200 as hb
    spec, cfg = CASES[name]
    spec = dict(spec, element_kind=1)
    ref = ref_lib.RefSession(po.ProblemSpec(**spec), po.SolverConfig(**cfg))
    prob = hb.build_problem(hb.ProblemSpec(**spec))
    assert np.array_equal(prob.rhs, ref.rhs())
    ops = hb.setup_two_grid(prob, hb.SolverConfig(**cfg))
    assert (ops.ndof, ops.coarse_ndof) == (ref.ndof, ref.coarse_ndof)
    n = ops.ndof
    f, u = po.random_vector(n, 51), po.random_vector(n, 52)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    r = torch.zeros_like(d(f))
    for shifted in (False, True):
        err = rel(ops.residual(d(f), d(u), r, shifted=shifted).cpu().numpy(), ref.residual(f, u, shifted=shifted))
        assert err <= TOL, ("residual", shifted, err)
    uc = po.random_vector(ops.coarse_ndof, 53)
    rc = torch.zeros_like(d(uc))
    assert rel(ops.restrict(d(f), rc).cpu().numpy(), ref.apply(4, f)) <= TOL
    assert rel(ops.prolong_add(d(u), d(uc), 1.0).cpu().numpy(), u + ref.apply(3, uc)) <= TOL
    y = torch.zeros_like(d(uc))
    assert rel(ops.coarse_apply(d(uc), y).cpu().numpy(), ref.apply(2, uc)) <= TOL
    if cfg.get("smoother", 0) == 0:
        out = torch.zeros_like(d(u))
        err = rel(ops.dd_step(d(u), d(f), out).cpu().numpy(), ref.dd_step(u, f))
        assert err <= TOL, ("dd_step", err)
        ud = d(u)
        ops.csdd_smoother(ud, d(f))
        assert rel(ud.cpu().numpy(), ref.csdd_smoother(u, f)) <= TOL
    ud = d(u)
    ops.two_grid_step(ud, d(f))
    err = rel(ud.cpu().numpy(), ref.two_grid_step(u, f))
    print(f"{name}: ndof {n}, two_grid_step rel err {err:.2e}")
    assert err <= TOL
    fr = prob.rhs
    res, want = ops.solve(d(fr)), ref.solve(fr)
    print(f"  solve: GPU {res.iterations} iterations, reference {want.iterations}")
    assert res.converged == want.converged and abs(res.iterations - want.iterations) <= 1
    k = min(len(res.residual_history), len(want.residual_history))
    assert np.allclose(res.residual_history[:k], want.residual_history[:k], rtol=1e-6)
    ops.close()


def test_triangles_rectangle_heterogeneous(ref_lib):
    """A rectangle with per-cell random k and eps and mixed tags on triangles: every
    subdomain class distinct (dense restricted inverses), against the reference."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_17494_b200 as hb
    g = np.random.default_rng(54)
    nx, ny, h = 11, 7, 0.07
    k = g.uniform(8.0, 12.0, size=(ny, nx))
    eps = 0.5 * g.random((ny, nx))
    tags = (A_, D_, N_, A_)
    ref = ref_lib.RefSession(desc=dict(order=4, nx=nx, ny=ny, h=h, k=k, eps=eps, side_tags=tags, element_kind=1),
                             config=po.SolverConfig())
    n = ref.ndof
    f, u = po.random_vector(n, 55), po.random_vector(n, 56)
    prob = hb.twogrid.Problem(order=4, n_cells=nx, h=h, k=float(k.mean()), k_cells=np.ascontiguousarray(k.ravel()),
                              eps_cells=np.ascontiguousarray(eps.ravel()), side_tags=tags, rhs=f, ny=ny,
                              element_kind=1)
    ops = hb.setup_two_grid(prob, hb.SolverConfig())
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    ud = d(u)
    ops.csdd_smoother(ud, d(f))
    assert rel(ud.cpu().numpy(), ref.csdd_smoother(u, f)) <= TOL
    ud = d(u)
    ops.two_grid_step(ud, d(f))
    assert rel(ud.cpu().numpy(), ref.two_grid_step(u, f)) <= TOL
    ops.close()
