"""GPU: GalerkinP coarse level and ExactShifted smoother against the reference's
acceptance properties (proj/tests/acceptance.cpp:228-312, C08-C10) and the oracle."""
import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
A_, D_ = po.ABSORBING, po.DIRICHLET
ALL_ABS = (A_, A_, A_, A_)
DIR2 = (D_, A_, D_, A_)  # Left and Bottom Dirichlet


def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def gal_run(W, sides, oracle=True):
    """run_bench(4, 10, W, GalerkinP, alpha_s = 0.02, alpha_c = 0.02, l_dd = 10, krylov)."""
    import paper_2509_17494_b200 as hb
    torch = _torch()
    kw = dict(alpha_s=0.02, alpha_c=0.02, l_dd=10, coarsening=1, outer=1)
    prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=W, ppw=10, side_tags=sides))
    ops = hb.setup_two_grid(prob, hb.SolverConfig(**kw))
    res = ops.solve(torch.from_numpy(prob.rhs).cuda())
    ops.close()
    ref = None
    if oracle:
        ses = po.Session(po.ProblemSpec(order=4, wavelengths=W, ppw=10, side_tags=sides), po.SolverConfig(**kw))
        ref = ses.solve(prob.rhs)
    return res, ref


def test_c08_galerkin_iterations_increase_with_size():
    """C08: GalerkinP iteration counts increase with the wavelength count (10, 20, 40)."""
    its = []
    for W in (10, 20, 40):
        res, ref = gal_run(W, ALL_ABS, oracle=W <= 20)
        assert res.converged
        if ref is not None:
            assert abs(res.iterations - ref.iterations) <= 1, (W, res.iterations, ref.iterations)
        its.append(res.iterations)
    assert its[0] < its[1] < its[2], its


def test_c09_galerkin_dirichlet_ratio():
    """C09: two Dirichlet sides cost GalerkinP 1.4x-2.6x the all-absorbing iterations."""
    a, ra = gal_run(20, ALL_ABS)
    d, rd = gal_run(20, DIR2)
    assert abs(a.iterations - ra.iterations) <= 1 and abs(d.iterations - rd.iterations) <= 1
    ratio = d.iterations / a.iterations
    assert 1.4 <= ratio <= 2.6, (a.iterations, d.iterations)


def test_c10_exact_shifted_contraction_rate():
    """C10 setup: ExactShifted smoother, Q4, 20 wavelengths, damping_D = 0.01; the
    contraction rate of 20 normalised error steps e <- TG(e, 0) matches the oracle."""
    import paper_2509_17494_b200 as hb
    torch = _torch()
    spec = dict(order=4, wavelengths=20, ppw=10, damping_D=0.01)
    prob = hb.build_problem(hb.ProblemSpec(**spec))
    ops = hb.setup_two_grid(prob, hb.SolverConfig(smoother=1))
    ses = po.Session(po.ProblemSpec(**spec), po.SolverConfig(smoother=1))
    n = ops.ndof
    e = po.random_vector(n, 99)
    e /= np.linalg.norm(e)
    eg = torch.from_numpy(e.copy()).cuda()
    zero = torch.zeros_like(eg)
    eo = e.copy()
    zo = np.zeros(n, np.complex128)
    for _ in range(20):
        ops.two_grid_step(eg, zero)
        rg = float(torch.linalg.norm(eg))
        eg /= rg
        eo = ses.two_grid_step(eo, zo)
        ro = np.linalg.norm(eo)
        eo /= ro
        assert abs(rg - ro) <= 1e-8 * ro
    assert rg < 1.0  # a contraction
    assert np.linalg.norm(eg.cpu().numpy() - eo) <= 1e-8
    ops.close()
