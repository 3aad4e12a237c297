"""Pin the CPU oracle against the reference's own known-answer and property tests.

Each test names the reference test it restates (proj/tests/*.cpp). These run on
CPU only; they are what makes the oracle trustworthy as the parity checker.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import pyoracle as po

A_, N_, D_ = po.ABSORBING, po.NEUMANN, po.DIRICHLET


def desc(n, p, k=1.0, eps=0.0, sides=(A_,) * 4, ny=None, h=None):
    ny = ny or n
    return dict(order=p, nx=n, ny=ny, h=h or 1.0 / n, k=k, eps=eps, side_tags=sides)


# ------------------------------------------------------------------ test_fespace.cpp
def test_dof_counts():  # proj/tests/test_fespace.cpp:31-55
    assert po.Session(desc=desc(1, 2)).ndof == 9
    assert po.Session(desc=desc(2, 4)).ndof == 81
    for n in (1, 3):
        for p in (2, 4, 6, 8):
            assert po.Session(desc=desc(n, p)).ndof == (n * p + 1) ** 2
    assert po.Session(desc=desc(1, 1)).ndof == 4
    assert po.Session(desc=desc(1, 3)).ndof == 16
    with pytest.raises(po.OracleError) as e:  # odd p rejected by the public builder
        po.Session(po.ProblemSpec(order=3, wavelengths=5, ppw=10))
    assert e.value.code == 2


def _vertex_stencil(A, s, cx, cy):
    row = s.find_dof("v", cx, cy)
    return np.array([[A[row, s.find_dof("v", cx + dx, cy + dy)] for dx in (-1, 0, 1)] for dy in (-1, 0, 1)])


def test_p1_stencils():  # proj/tests/test_fespace.cpp:67-88, acceptance.cpp:409-431
    s = po.Session(desc=desc(4, 1, k=1e-30, sides=(N_,) * 4))
    K = s.build_matrix(0, 0.0).toarray()
    st = _vertex_stencil(K, s, 2, 2)
    want = np.full((3, 3), -1 / 3)
    want[1, 1] = 8 / 3
    assert np.abs(st - want).max() < 1e-14
    M = s.build_matrix(1, weight=1.0).toarray()
    h2 = (1 / 4) ** 2
    mw = np.array([[1 / 36, 1 / 9, 1 / 36], [1 / 9, 4 / 9, 1 / 9], [1 / 36, 1 / 9, 1 / 36]])
    assert np.abs(_vertex_stencil(M, s, 2, 2) - h2 * mw).max() < 1e-14 * h2


@pytest.mark.parametrize("p", [2, 4, 6, 8])
def test_patch_test(p):  # proj/tests/test_fespace.cpp:90-113
    s = po.Session(desc=desc(3, p, k=1e-30, sides=(N_,) * 4))
    A = s.build_matrix(0, 0.0).toarray()
    keys = s.dof_keys()
    ones = np.where(keys[:, 0] == ord("v"), 1.0, 0.0)
    assert np.linalg.norm(A @ ones) < 1e-12 * np.linalg.norm(A)
    assert np.abs(A.imag).max() < 1e-14
    assert np.abs(A - A.T).max() < 1e-12
    assert np.linalg.eigvalsh(A.real).min() > -1e-10


def test_assembled_structure():  # proj/tests/test_fespace.cpp:115-152
    s = po.Session(desc=desc(2, 4, k=3.0, eps=0.7, sides=(N_,) * 4))
    A = s.build_matrix(0, 0.0).toarray()
    assert np.abs(A - A.T).max() < 1e-12
    s0 = po.Session(desc=desc(2, 4, k=3.0, eps=0.0, sides=(N_,) * 4))
    assert np.abs(s0.build_matrix(0, 0.0).toarray().imag).max() == 0.0
    alpha = 0.25
    As = s.build_matrix(0, alpha).toarray()
    M = s.build_matrix(1, weight=9.0).toarray()  # k^2 = 9
    assert np.abs(As - (A - 1j * alpha * M)).max() < 1e-12
    sd = po.Session(desc=desc(2, 4, k=3.0, eps=0.7, sides=(D_, A_, A_, A_)), config=None)
    Ad = sd.build_matrix(0, 0.0).toarray()
    dofs = sd.dirichlet_dofs()
    assert len(dofs) == 9
    for d in dofs:
        assert abs(np.abs(Ad[d]).sum() - 1.0) < 1e-14
        assert abs(np.abs(Ad[:, d]).sum() - 1.0) < 1e-14
        assert Ad[d, d] == 1.0


def test_boundary_mass():  # proj/tests/test_fespace.cpp:167-200 (per-side tags)
    s = po.Session(desc=desc(2, 1, k=2.5, sides=(N_,) * 4))
    assert s.build_matrix(2).nnz == 0
    s = po.Session(desc=desc(2, 1, k=2.5, sides=(N_, N_, A_, N_)))
    B = s.build_matrix(2).toarray()
    kh = 2.5 * 0.5
    v0, v1 = s.find_dof("v", 0, 0), s.find_dof("v", 1, 0)
    assert abs(B[v0, v0] - 1j * kh / 3) < 1e-14
    assert abs(B[v0, v1] - 1j * kh / 6) < 1e-14
    assert abs(B[v1, v1] - 2j * kh / 3) < 1e-14  # two absorbing edges meet at (1,0)


def test_translation_invariance():  # proj/tests/test_fespace.cpp:257-278
    s = po.Session(desc=desc(6, 4, k=7.0, eps=0.3, sides=(N_,) * 4))
    A = s.build_matrix(0, 0.1).toarray()

    def cell(cx, cy):
        out = [s.find_dof("v", cx, cy)]
        out += [s.find_dof("h", cx, cy, o) for o in range(3)]
        out += [s.find_dof("e", cx, cy, o) for o in range(3)]
        out += [s.find_dof("c", cx, cy, o) for o in range(9)]
        return out

    c1, c2 = cell(2, 2), cell(3, 3)
    for bx in (-1, 0, 1):
        for by in (-1, 0, 1):
            d1, d2 = cell(2 + bx, 2 + by), cell(3 + bx, 3 + by)
            assert np.abs(A[np.ix_(c1, d1)] - A[np.ix_(c2, d2)]).max() < 1e-12


def test_dof_numbering():  # proj/tests/test_fespace.cpp:280-289
    s = po.Session(desc=desc(3, 4))
    assert s.find_dof("v", 0, 0) == 0
    assert s.find_dof("v", 1, 0) > s.find_dof("v", 0, 0)
    assert s.find_dof("v", 0, 1) > s.find_dof("v", 3, 0)


def test_element_tensor_structure():  # K_e = S1 (x) M1 + M1 (x) S1
    for p in (2, 4):
        K, M = po.element_matrices(p)
        m1 = po.edge_mass(p)
        assert abs(m1[0, 0] - 1 / 3) < 1e-15 and abs(m1[0, 1] - 1 / 6) < 1e-15
        assert np.abs(K - K.T).max() < 1e-14 and np.abs(M - M.T).max() < 1e-15


# ------------------------------------------------------------------ test_qsfem.cpp
def test_stencil_coefficients():  # proj/tests/test_qsfem.cpp:11-57
    for eta in (0.3, 0.9, 1.7, 2.6):
        assert po.stencil(eta)["P0"] == 4.0
    for bad in (0.0, -0.5, math.pi, 3.5):
        with pytest.raises(po.OracleError):
            po.stencil(bad)
    for eta in (0.3, 0.7854, 1.2566, 2.0, 2.9):
        k = 5.0
        hc = eta / k
        s = po.stencil(eta)
        sym = s["N"] / hc ** 2 * po.stencil_symbol(eta, 0.0, 0.0)
        assert abs(sym + k * k) <= 1e-12 * k * k
    for ppw in (4.0, 6.0, 8.0):
        eta = 2 * math.pi / ppw
        for t in (math.pi / 16, 3 * math.pi / 16):
            assert abs(po.stencil_symbol(eta, eta * math.cos(t), eta * math.sin(t))) < 1e-10
    a, b = 0.4, 0.9
    assert po.stencil_symbol(1.3, a, b) == pytest.approx(po.stencil_symbol(1.3, b, a))
    assert po.stencil_symbol(1.3, a, b) == pytest.approx(po.stencil_symbol(1.3, -a, b))


def test_qsfem_assembly():  # proj/tests/test_qsfem.cpp:100-168
    k = 2 * math.pi
    n = 8
    hc = 1 / n
    s = po.stencil(k * hc)
    ses = po.Session(desc=desc(n, 1, k=k, sides=(N_,) * 4))
    A = ses.build_matrix(3).toarray()
    row = ses.find_dof("v", 4, 4)
    v = lambda x, y: ses.find_dof("v", x, y)  # noqa: E731
    assert A[row, row] == s["N"] * s["P0"]
    assert A[row, v(5, 4)] == s["N"] * s["P1"]
    assert A[row, v(4, 3)] == s["N"] * s["P1"]
    assert A[row, v(3, 3)] == s["N"] * s["P2"]
    assert A[row, v(5, 5)] == s["N"] * s["P2"]
    assert np.abs(A - A.T).max() < 1e-14
    assert A[v(0, 0), v(0, 0)] == s["N"] * s["P0"] / 4
    eps = np.zeros((n, n))
    eps[5, 3] = 0.8  # cell (3,5)
    A1 = po.Session(desc=desc(n, 1, k=k, eps=eps, sides=(N_,) * 4)).build_matrix(3).toarray()
    Mcell = po.Session(desc=desc(n, 1, k=k, eps=eps, sides=(N_,) * 4)).build_matrix(1, weight=1.0).toarray()
    # the single-cell mass = (weight-1 mass restricted to cell (3,5)): compare A0 - A1 on that cell's dofs
    cd = [v(3, 5), v(4, 5), v(3, 6), v(4, 6)]
    D = A - A1
    assert np.abs(np.delete(np.delete(D, cd, 0), cd, 1)).max() < 1e-14
    Kloc = po.element_matrices(1)[1] * hc ** 2
    assert np.abs(D[np.ix_(cd, cd)] - 1j * 0.8 * Kloc).max() < 1e-14
    del Mcell
    Aa = po.Session(desc=desc(n, 1, k=k, sides=(A_,) * 4)).build_matrix(3).toarray()
    B = po.Session(desc=desc(n, 1, k=k, sides=(A_,) * 4)).build_matrix(2).toarray()
    assert np.abs(Aa - (A - B)).max() < 1e-14
    sd = po.Session(desc=desc(n, 1, k=k, sides=(D_, A_, A_, A_)))
    Ad = sd.build_matrix(3).toarray()
    d = sd.find_dof("v", 0, 4)
    assert abs(np.abs(Ad[d]).sum() - 1.0) < 1e-14 and Ad[d, d] == 1.0


# ------------------------------------------------------------------ test_linalg.cpp
def test_sparse_lu():  # proj/tests/test_linalg.cpp:10-56
    I = sp.identity(5, dtype=complex, format="csr")
    b = np.random.default_rng(0).standard_normal(5) + 0j
    assert np.linalg.norm(po.lu_solve_csr(I, b) - b) < 1e-14
    rng = np.random.default_rng(42)
    n = 50
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i), cols.append(i), vals.append(6 + rng.uniform(-1, 1) + 1j * rng.uniform(-1, 1))
        for _ in range(4):
            j = int(rng.integers(n))
            if j != i:
                rows.append(i), cols.append(j), vals.append(0.5 * (rng.uniform(-1, 1) + 1j * rng.uniform(-1, 1)))
    A = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    b = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    x = po.lu_solve_csr(A, b)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12
    S = sp.csr_matrix(([1.0 + 0j, 1.0], ([0, 1], [0, 1])), shape=(3, 3))
    with pytest.raises(po.OracleError) as e:
        po.lu_solve_csr(S, np.ones(3, complex))
    assert e.value.code == 1


# ------------------------------------------------------------------ test_twogrid.cpp
def _cfg(**kw):
    return po.SolverConfig(**kw)


def test_partition_layout():  # proj/tests/test_twogrid.cpp:25-72
    s = po.Session(desc=desc(8, 2), config=_cfg(l_dd=4))
    info = s.partition_info()
    assert len(info) == 4 and all(r[2] * r[3] == 16 for r in info)
    s = po.Session(desc=desc(10, 2), config=_cfg(l_dd=4))
    sizes = sorted(int(r[2] * r[3]) for r in s.partition_info())
    assert sizes.count(16) == 4 and sizes.count(8) == 4 and sizes.count(4) == 1
    s = po.Session(desc=desc(12, 2), config=_cfg(l_dd=4))
    inner = [r for r in s.partition_info() if r[0] == 4 and r[1] == 4]
    assert len(inner) == 1 and inner[0][6] * inner[0][7] == 36
    s = po.Session(desc=desc(7, 4), config=_cfg(l_dd=3))
    m = s.multiplicity()
    assert m.min() >= 1.0 and m.max() >= 2.0
    with pytest.raises(po.OracleError):
        po.Session(desc=desc(4, 2), config=_cfg(l_dd=1))


def test_dd_step_consistency():  # proj/tests/test_twogrid.cpp:74-107
    s = po.Session(po.ProblemSpec(order=2, wavelengths=3, ppw=8), _cfg(l_dd=4))
    As = s.csr(1)
    f = po.random_vector(s.ndof, 11)
    u = po.lu_solve_csr(As, f)
    u2 = s.dd_step(u, f)
    assert np.linalg.norm(u2 - u) < 1e-10 * np.linalg.norm(u)
    z = np.zeros(s.ndof, complex)
    assert np.linalg.norm(s.dd_step(z, z)) == 0.0
    one = po.Session(po.ProblemSpec(order=2, wavelengths=3, ppw=8), _cfg(l_dd=1000))
    assert one.n_subdomains == 1
    f = po.random_vector(one.ndof, 12)
    u = one.dd_step(np.zeros(one.ndof, complex), f)
    assert np.linalg.norm(As @ u - f) < 1e-9 * np.linalg.norm(f)


def test_pou_averaging():  # proj/tests/test_twogrid.cpp:109-122
    s = po.Session(po.ProblemSpec(order=4, wavelengths=2, ppw=8), _cfg(l_dd=3))
    u = po.random_vector(s.ndof, 21)
    u2 = s.dd_step(u, s.apply(1, u))
    assert np.linalg.norm(u2 - u) < 1e-10 * np.linalg.norm(u)


def test_subdomain_boundary_inheritance():  # proj/tests/test_twogrid.cpp:124-140
    s = po.Session(po.ProblemSpec(order=2, wavelengths=4, ppw=8, side_tags=(D_, A_, A_, A_)), _cfg(outer=1))
    r = s.solve(s.rhs())
    assert r.converged
    assert all(r.u[d] == 0 for d in s.dirichlet_dofs())


def test_coarse_mesh_counts():  # proj/tests/test_twogrid.cpp:157-176
    s = po.Session(desc=desc(10, 4), config=_cfg())
    assert s.coarse_ndof == 21 * 21
    assert s.ndof / s.coarse_ndof == pytest.approx(4.0, rel=0.05)
    s = po.Session(desc=desc(10, 2), config=_cfg())
    assert s.coarse_ndof == 11 * 11


@pytest.mark.parametrize("p", [2, 4, 6])
def test_prolongation(p):  # proj/tests/test_twogrid.cpp:178-213
    s = po.Session(desc=desc(3, p), config=_cfg())
    ones = np.ones(s.coarse_ndof, complex)
    u1 = s.apply(3, ones)
    keys = s.dof_keys()
    isv = keys[:, 0] == ord("v")
    assert np.abs(u1[isv] - 1).max() < 1e-12 and np.abs(u1[~isv]).max() < 1e-12
    m = p // 2
    hc = 1 / 3 / m
    f = lambda x, y: (0.8 * x - 0.45 * y + 0.3) ** m  # noqa: E731
    ck = s.dof_keys(coarse=True)
    uc = np.array([f(kx * hc, ky * hc) for _, kx, ky, _ in ck], complex)
    uf = s.apply(3, uc)
    for x, y in ((0.11, 0.93), (0.47, 0.52), (0.98, 0.017)):
        assert abs(s.evaluate(uf, x, y) - f(x, y)) < 1e-10


def test_p2_prolongation_injection():  # proj/tests/test_twogrid.cpp:215-234
    s = po.Session(desc=desc(4, 2), config=_cfg())
    IP = s.csr(3)
    keys = s.dof_keys()
    nnz = np.diff(IP.indptr)
    for d, (kind, x, y, _) in enumerate(keys):
        if kind == ord("v"):
            assert nnz[d] == 1 and IP[d, s.find_dof("v", x, y, coarse=True)] == 1.0
        else:
            assert nnz[d] == 0


def test_galerkin_p_coarsening():  # proj/tests/test_twogrid.cpp:236-264
    d = desc(3, 4, k=10.0)
    s = po.Session(desc=d, config=_cfg(coarsening=1, alpha_c=0.0))
    assert s.coarse_ndof == 49  # (3*2+1)^2
    IP = s.csr(3).toarray()
    assert np.abs(IP.conj().T @ IP - np.eye(49)).max() < 1e-14  # 0/1 inclusion of an index subset
    direct = po.Session(desc=desc(3, 2, k=10.0), config=_cfg(coarsening=2)).csr(0).toarray()
    assert np.abs(s.csr(2).toarray() - direct).max() < 1e-14  # alpha_c = 0: plain order-2 matrix
    uc = po.random_vector(49, 7)
    uf = IP @ uc
    for x, y in ((0.21, 0.67), (0.83, 0.12)):  # the included functions are the same functions
        assert abs(s.evaluate(uf, x, y) - s.evaluate(uc, x, y, coarse=True)) < 1e-13


@pytest.mark.parametrize("coarsening", [0, 1])
def test_two_grid_properties(coarsening):  # proj/tests/test_twogrid.cpp:266-299 (OptimizedFD, GalerkinP)
    s = po.Session(po.ProblemSpec(order=4, wavelengths=3, ppw=10), _cfg(l_dd=4, coarsening=coarsening))
    n = s.ndof
    f = po.random_vector(n, 31)
    u = po.lu_solve_csr(s.csr(0), f)
    u2 = s.two_grid_step(u, f)
    assert np.linalg.norm(u2 - u) <= 1e-11 * np.linalg.norm(u)
    e1, e2 = po.random_vector(n, 32), po.random_vector(n, 33)
    z = np.zeros(n, complex)
    lhs = s.two_grid_step(e1 + e2, z)
    rhs = s.two_grid_step(e1, z) + s.two_grid_step(e2, z)
    assert np.linalg.norm(lhs - rhs) < 1e-11 * np.linalg.norm(rhs)


def test_omega_c_zero():  # proj/tests/test_twogrid.cpp:301-317
    s = po.Session(po.ProblemSpec(order=2, wavelengths=2, ppw=8), _cfg(omega_c=0.0))
    f = po.random_vector(s.ndof, 41)
    z = np.zeros(s.ndof, complex)
    u1 = s.two_grid_step(z, f)
    u2 = s.csdd_smoother(s.csdd_smoother(z, f), f)
    assert np.linalg.norm(u1 - u2) < 1e-13 * np.linalg.norm(u2)


def test_smoother_hf_reduction():  # proj/tests/test_twogrid.cpp:319-342
    k = 2 * math.pi * 2
    s = po.Session(desc=desc(16, 2, k=k), config=_cfg(l_dd=4))
    keys = s.dof_keys()
    u = np.exp(1j * math.pi * (keys[:, 1] + keys[:, 2]) * 0.96)
    f = np.zeros(s.ndof, complex)
    r0 = np.linalg.norm(s.residual(f, u))
    u1 = s.csdd_smoother(u, f)
    r1 = np.linalg.norm(s.residual(f, u1))
    assert r1 / r0 < 0.5


def test_solve():  # proj/tests/test_twogrid.cpp:344-383
    spec = po.ProblemSpec(order=4, wavelengths=4, ppw=10)
    s = po.Session(spec, _cfg())
    r = s.solve(np.zeros(s.ndof, complex))
    assert r.iterations == 0 and np.linalg.norm(r.u) == 0 and r.converged
    r1 = s.solve(s.rhs())
    k = po.Session(spec, _cfg(outer=1))
    r2 = k.solve(k.rhs())
    assert r1.converged and r2.converged
    assert np.linalg.norm(r1.u - r2.u) < 2e-6 * np.linalg.norm(r1.u)
    assert r2.iterations <= r1.iterations
    assert r1.residual_history[-1] <= 1e-6
    bad = po.Session(spec, _cfg(max_iters=2))
    rb = bad.solve(bad.rhs())
    assert not rb.converged and rb.iterations == 2


def test_exact_shift_smoother():  # proj/tests/test_twogrid.cpp:385-396
    s = po.Session(po.ProblemSpec(order=4, wavelengths=3, ppw=10), _cfg(smoother=1))
    r = s.solve(s.rhs())
    assert r.converged and r.iterations < 20


# ------------------------------------------------------------------ acceptance / README
def test_readme_iters_7():  # proj/README.md:89-102: dofs=40401 iters=7; acceptance C07 band [4,10]
    s = po.Session(po.ProblemSpec(order=4, wavelengths=20, ppw=10), _cfg(outer=1))
    assert s.ndof == 40401
    r = s.solve(s.rhs())
    assert r.converged and r.iterations == 7


def test_c08_c09_galerkin_p():  # proj/tests/acceptance.cpp:228-282 at the oracle-sized W = 10, 20
    kw = dict(alpha_s=0.02, alpha_c=0.02, l_dd=10, coarsening=1, outer=1)

    def its(W, sides=(A_,) * 4):
        s = po.Session(po.ProblemSpec(order=4, wavelengths=W, ppw=10, side_tags=sides), _cfg(**kw))
        r = s.solve(s.rhs())
        assert r.converged
        return r.iterations

    a10, a20, d20 = its(10), its(20), its(20, (D_, A_, D_, A_))
    assert a10 < a20  # C08: increasing with size
    assert 1.4 <= d20 / a20 <= 2.6  # C09: Dirichlet sides cost 1.4x-2.6x


def test_c11_structural():  # proj/tests/acceptance.cpp:314-360
    s = po.Session(po.ProblemSpec(order=4, wavelengths=3, ppw=10), _cfg())
    rng = np.random.default_rng(5)
    u = rng.standard_normal(s.ndof) + 1j * rng.standard_normal(s.ndof)
    f = s.apply(0, u)
    u2 = s.two_grid_step(u, f)
    assert np.linalg.norm(u2 - u) / np.linalg.norm(u) <= 1e-12
    e1 = rng.standard_normal(s.ndof) + 1j * rng.standard_normal(s.ndof)
    e2 = rng.standard_normal(s.ndof) + 1j * rng.standard_normal(s.ndof)
    z = np.zeros(s.ndof, complex)
    p1, p2 = s.two_grid_step(e1, z), s.two_grid_step(e2, z)
    lin = np.linalg.norm(s.two_grid_step(e1 + e2, z) - p1 - p2) / (np.linalg.norm(p1) + np.linalg.norm(p2))
    assert lin <= 1e-12


def test_problem_construction():  # proj/tests/test_cli.cpp:185-192
    s = po.Session(po.ProblemSpec(order=4, wavelengths=5, ppw=10))
    assert s.nx == 13
    assert np.abs(s.rhs()).sum() == 1.0
    sl = po.Session(po.ProblemSpec(order=4, wavelengths=5, ppw=10, layer_sides=(po.LEFT,),
                                   side_tags=(N_, A_, A_, A_), layer_width_dofs=12))
    k, eps = sl.coeffs()
    assert eps[:, 0].min() > 0 and eps[:, -1].max() == 0.0
    assert np.all(np.diff(eps[0, :3]) < 0)  # sin^2 ramp decreasing away from the left side
