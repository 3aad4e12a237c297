"""Edge cases and error behaviour through the C-ABI, mirroring the reference:
zero RHS (proj/core/src/twogrid.cpp:281-282: converged in 0 iterations),
max_iters reached (SolveResult::converged = false, CLI exit code 3),
invalid configurations (std::invalid_argument -> status 2), calls that need a
component the handle was not built with, and one-cell-wide / minimal meshes."""
import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu


def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_zero_rhs_converges_in_zero_iterations():
    torch = _torch()
    import paper_2509_17494_b200 as hb
    prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=3, ppw=10))
    for cfg in (hb.SolverConfig(), hb.SolverConfig(outer=1)):
        ops = hb.setup_two_grid(prob, cfg)
        res = ops.solve(torch.zeros(ops.ndof, dtype=torch.complex128, device="cuda"))
        assert res.converged and res.iterations == 0
        assert float(torch.linalg.norm(res.u)) == 0.0
        ops.close()


def test_max_iters_not_converged_matches_oracle():
    torch = _torch()
    import paper_2509_17494_b200 as hb
    spec = dict(order=4, wavelengths=6, ppw=10)
    prob = hb.build_problem(hb.ProblemSpec(**spec))
    ops = hb.setup_two_grid(prob, hb.SolverConfig(max_iters=2))
    res = ops.solve(torch.from_numpy(prob.rhs).cuda())
    ref = po.Session(po.ProblemSpec(**spec), po.SolverConfig(max_iters=2)).solve(prob.rhs)
    assert not res.converged and not ref.converged
    assert res.iterations == ref.iterations == 2
    assert np.allclose(res.residual_history, ref.residual_history, rtol=1e-8)
    # status code 3 at the C-ABI (the CLI's "did not converge" exit code)
    from paper_2509_17494_b200 import _lib
    import ctypes as C
    hist = np.zeros(3)
    it, conv = C.c_int(), C.c_int()
    u = torch.zeros(ops.ndof, dtype=torch.complex128, device="cuda")
    f = torch.from_numpy(prob.rhs).cuda()
    rc = _lib.lib().htg_solve(ops._h, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()),
                              hist.ctypes.data_as(C.c_void_p), 3, C.byref(it), C.byref(conv))
    assert rc == _lib.HTG_NOT_CONVERGED and conv.value == 0 and it.value == 2
    ops.close()


@pytest.mark.parametrize("cfg,why", [
    (dict(l_dd=1), "partition"),                       # twogrid.cpp:18 (l_dd >= 2)
    (dict(n_dd=0), "iteration"),
    (dict(coarsening=7), "coarsening"),
    (dict(smoother=5), "smoother"),
])
def test_invalid_config_is_status_2(cfg, why):
    _torch()
    import paper_2509_17494_b200 as hb
    prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=3, ppw=10))
    with pytest.raises(hb.HtgError) as e:
        hb.setup_two_grid(prob, hb.SolverConfig(**cfg))
    assert e.value.code == 2 and why in str(e.value).lower()


def test_qsfem_resolution_limit_is_status_2():
    """eta = k h_c must stay below pi (qsfem.cpp:8-39): too few points per wavelength."""
    _torch()
    import paper_2509_17494_b200 as hb
    prob = hb.build_problem(hb.ProblemSpec(order=2, wavelengths=8, ppw=1.5))
    with pytest.raises(hb.HtgError) as e:
        hb.setup_two_grid(prob, hb.SolverConfig())
    assert e.value.code == 2 and "eta" in str(e.value)


def test_missing_component_calls_are_status_2():
    torch = _torch()
    import paper_2509_17494_b200 as hb
    prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=3, ppw=10))
    ops = hb.setup_two_grid(prob, hb.SolverConfig(smoother=1, coarsening=2))  # ExactShifted, no coarse level
    n = ops.ndof
    u = torch.zeros(n, dtype=torch.complex128, device="cuda")
    with pytest.raises(hb.HtgError) as e:
        ops.dd_step(u, u, u)
    assert e.value.code == 2
    with pytest.raises(hb.HtgError) as e:
        ops.coarse_solve(u[:1], u[:1])
    assert e.value.code == 2
    # the two-grid step still works: two exact-shifted smoothing steps
    f = torch.from_numpy(po.random_vector(n, 3)).cuda()
    ses = po.Session(po.ProblemSpec(order=4, wavelengths=3, ppw=10), po.SolverConfig(smoother=1, coarsening=2))
    ops.two_grid_step(u, f)
    want = ses.two_grid_step(np.zeros(n, complex), f.cpu().numpy())
    assert np.linalg.norm(u.cpu().numpy() - want) <= 1e-10 * np.linalg.norm(want)
    ops.close()


@pytest.mark.parametrize("nx,ny,p", [(1, 1, 4), (1, 5, 2), (7, 1, 4), (2, 2, 2)])
def test_minimal_meshes(nx, ny, p):
    """One-cell and one-row meshes: a single subdomain, coarse lattices of 3 x 3 nodes."""
    torch = _torch()
    import paper_2509_17494_b200 as hb
    k = np.full((ny, nx), 3.0)
    ses = po.Session(desc=dict(order=p, nx=nx, ny=ny, h=0.1, k=k, eps=0.0, side_tags=(2, 2, 2, 2)),
                     config=po.SolverConfig())
    f = po.random_vector(ses.ndof, 5)
    prob = hb.twogrid.Problem(order=p, n_cells=nx, h=0.1, k=3.0, k_cells=np.ascontiguousarray(k.ravel()),
                              eps_cells=np.zeros(nx * ny), side_tags=(2, 2, 2, 2), rhs=f, ny=ny)
    ops = hb.setup_two_grid(prob, hb.SolverConfig())
    assert ops.ndof == ses.ndof
    u = torch.zeros(ops.ndof, dtype=torch.complex128, device="cuda")
    ops.two_grid_step(u, torch.from_numpy(f).cuda())
    want = ses.two_grid_step(np.zeros(ses.ndof, complex), f)
    assert np.linalg.norm(u.cpu().numpy() - want) <= 1e-10 * np.linalg.norm(want)
    ops.close()


def test_vector_lengths_and_devices_are_checked():
    """A short vector would be overrun by the C-ABI (it reads/writes ndof entries):
    rejected with HTG_ERR_INVALID before any launch, device and host paths alike."""
    torch = _torch()
    import paper_2509_17494_b200 as hb
    prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=3, ppw=10))
    ops = hb.setup_two_grid(prob)
    z = lambda n: torch.zeros(n, dtype=torch.complex128, device="cuda")  # noqa: E731
    with pytest.raises(hb.HtgError):
        ops.residual(z(ops.ndof), z(ops.ndof - 1), z(ops.ndof))
    with pytest.raises(hb.HtgError):
        ops.coarse_solve(z(ops.coarse_ndof), z(ops.ndof))
    with pytest.raises(hb.HtgError):
        ops.prolong_add(z(ops.ndof), z(ops.coarse_ndof + 1), 1.0)
    with pytest.raises(hb.HtgError):
        ops.two_grid_step_host(np.zeros(ops.ndof - 3, np.complex128), np.zeros(ops.ndof, np.complex128))
    with pytest.raises(hb.HtgError):
        ops.residual(z(ops.ndof).cpu(), z(ops.ndof), z(ops.ndof))
    ops.close()


def test_graph_cache_is_bounded():
    """solve() with a fresh u every call must not grow the per-handle graph cache."""
    torch = _torch()
    import paper_2509_17494_b200 as hb
    prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=3, ppw=10))
    ops = hb.setup_two_grid(prob)
    f = torch.from_numpy(prob.rhs).cuda()
    first = ops.solve(f)
    for _ in range(24):
        res = ops.solve(f)
        assert res.iterations == first.iterations
    assert 1 <= ops.cached_graphs <= 16
    assert torch.equal(res.u, first.u)
    ops.close()
