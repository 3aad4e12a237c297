"""Triangle elements on the host (CPU, no GPU): the product's restated P_p triangle
reference elements and staged interpolation (csrc/tri.cpp) and its assembled
Helmholtz matrices A, A_s on triangle meshes (coarse_nd.cpp fe_lattice) against
the reference's own code (oracle/_ref, where it is built: this container)."""
import ast
import ctypes as C
import glob
import os
import sys

import numpy as np
import pytest

from oracle import pyoracle as po

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def _ref():
    from oracle import pyref
    if not (os.path.exists(pyref.LIB_PATH) or os.path.isdir(pyref.REF_ROOT)):
        pytest.skip("the reference library is not available")
    return pyref


@pytest.mark.parametrize("p", [2, 4, 6, 8])
@pytest.mark.parametrize("sub", [0, 1], ids=["lower", "upper"])
def test_triangle_element_matches_reference(p, sub):
    pyref = _ref()
    import ndcheck
    ref = pyref.lib()
    ref.ref_element.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.POINTER(C.c_int), C.POINTER(C.c_int)]
    nd = ndcheck._lib()
    nd.nd_tri_element.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.POINTER(C.c_int), C.POINTER(C.c_int)]
    N = 64
    K1, M1, E1 = np.zeros(N * N), np.zeros(N * N), np.zeros(N * N)
    K2, M2, E2, pl = np.zeros(N * N), np.zeros(N * N), np.zeros(N * N), np.zeros(4 * N, np.int32)
    n1, q1, n2, q2 = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    assert ref.ref_element(p, 1 + sub, p // 2, K1.ctypes.data, M1.ctypes.data, E1.ctypes.data,
                           C.byref(n1), C.byref(q1)) == 0
    assert nd.nd_tri_element(p, sub, K2.ctypes.data, M2.ctypes.data, E2.ctypes.data, pl.ctypes.data,
                             C.byref(n2), C.byref(q2)) == 0
    n, m = n1.value, q1.value
    assert (n, m) == (n2.value, q2.value) == ((p + 1) * (p + 2) // 2, (p // 2 + 1) * (p // 2 + 2) // 2)
    assert np.abs(K1[:n * n] - K2[:n * n]).max() <= 1e-13
    assert np.abs(M1[:n * n] - M2[:n * n]).max() <= 1e-14
    assert np.abs(E1[:n * m] - E2[:n * m]).max() <= 1e-13
    # every unit-cell slot of the element's cell holds one dof (placement is injective)
    slots = {tuple(pl[4 * i:4 * i + 4]) for i in range(n)}
    assert len(slots) == n


@pytest.mark.parametrize("p", [2, 4, 6])
@pytest.mark.parametrize("tags", [(2, 2, 2, 2), (0, 2, 1, 2)], ids=["absorbing", "dir_neu"])
def test_triangle_assembly_matches_reference(p, tags):
    pyref = _ref()
    import ndcheck
    import paper_2509_17494_b200 as hb
    spec = dict(order=p, wavelengths=2, ppw=8, side_tags=tags, element_kind=1)
    prob = hb.build_problem(hb.ProblemSpec(**spec))
    ref = pyref.RefSession(po.ProblemSpec(**spec), po.SolverConfig(coarsening=2))
    assert np.array_equal(prob.rhs, ref.rhs())
    g = np.random.default_rng(p)
    x = g.standard_normal(ref.ndof) + 1j * g.standard_normal(ref.ndof)
    for alpha, which in ((0.0, 0), (0.2, 1)):
        y = ndcheck.fe_apply(prob, p, alpha, x)
        yr = ref.apply(which, x)
        assert np.linalg.norm(y - yr) / np.linalg.norm(yr) <= 1e-13


TRI_GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "reftri_*.npz")))


def _golden_problem(hb, g):
    if "spec" in g:
        prob = hb.build_problem(hb.ProblemSpec(**ast.literal_eval(str(g["spec"]))))
        assert np.array_equal(prob.rhs, g["rhs"])
        return prob, prob.order
    d = ast.literal_eval(str(g["desc"]))
    return hb.twogrid.Problem(order=d["order"], n_cells=d["nx"], h=d["h"], k=float(g["k_cells"].mean()),
                              k_cells=np.ascontiguousarray(g["k_cells"].ravel()),
                              eps_cells=np.ascontiguousarray(g["eps_cells"].ravel()), side_tags=d["side_tags"],
                              rhs=g["f"], ny=d["ny"], element_kind=1), d["order"]


def test_triangle_fixtures_present():
    assert len(TRI_GOLDEN) >= 6
    orders = {ast.literal_eval(str(np.load(p)["spec"] if "spec" in np.load(p) else np.load(p)["desc"]))["order"]
              for p in TRI_GOLDEN}
    assert orders == {2, 4, 6, 8}


@pytest.mark.parametrize("path", TRI_GOLDEN, ids=[os.path.basename(p)[:-4] for p in TRI_GOLDEN])
def test_triangle_host_assembly_matches_reference_fixture(path):
    """No reference at run time: the product's triangle matrices (csrc/tri.cpp +
    coarse_nd.cpp fe_lattice) reproduce the reference's residual f - A u on every
    free dof of the committed fixture (Dirichlet rows are the solver's, not A's)."""
    import ndcheck
    import paper_2509_17494_b200 as hb
    g = np.load(path)
    prob, p = _golden_problem(hb, g)
    f, u = g["f"], g["u"]
    free = np.ones(f.size, bool)
    free[g["dirichlet"]] = False
    for alpha, key in ((0.0, "residual"), (None, "residual_shifted")):
        if alpha is None:
            alpha = po.SolverConfig(**ast.literal_eval(str(g["config"]))).alpha_s
        r = f - ndcheck.fe_apply(prob, p, alpha, u)
        want = g[key]
        assert np.linalg.norm((r - want)[free]) / np.linalg.norm(want[free]) <= 1e-13, key


@pytest.mark.skipif(not os.path.isdir("/root/reference"), reason="/root/reference absent: fixtures are committed")
@pytest.mark.parametrize("name", ["reftri_p4_dir_neu", "reftri_rect_p4_hetero"])
def test_reference_regenerates_triangle_fixture(name):
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tools"))
    import make_ref_golden as mk
    from oracle import pyref
    pyref.build()
    new = mk.make(name)
    g = np.load(os.path.join(HERE, "golden", f"{name}.npz"))
    for key in ("residual", "restrict", "prolong", "coarse_apply", "coarse_solve", "two_grid_step", "solve_u"):
        assert np.linalg.norm(new[key] - g[key]) <= 1e-14 * np.linalg.norm(g[key]), key
