"""Host-side checks of the coarse nested-dissection factorization (csrc/coarse_nd.cpp)
through tests/native/libndcheck.so: the same explicit factor blocks the GPU level
kernels apply, evaluated on the CPU. No GPU needed."""
import numpy as np
import pytest

import paper_2509_17494_b200 as hb
from oracle import pyoracle as po

from ndcheck import coarse_check, fe_apply, fe_solve

N_, A_ = hb.NEUMANN, hb.ABSORBING


def _rhs(nv, seed, nrhs=2):
    g = np.random.default_rng(seed)
    return g.standard_normal((nrhs, nv)) + 1j * g.standard_normal((nrhs, nv))


@pytest.mark.parametrize("kw", [dict(order=4, wavelengths=4, ppw=10),
                                dict(order=4, wavelengths=6, ppw=12, side_tags=(N_, A_, N_, A_), layer_sides=(0, 2)),
                                dict(order=2, wavelengths=5, ppw=8)])
def test_nd_matches_oracle_coarse_solve(kw):
    """ND solve == the oracle's banded LU (proj/core/src/twogrid.cpp:244,273) on the same A_c."""
    prob = hb.build_problem(hb.ProblemSpec(**kw))
    ses = po.Session(po.ProblemSpec(**kw), po.SolverConfig())
    rc = _rhs(ses.coarse_ndof, 1)
    x, be, st = coarse_check(prob, rc)
    assert be < 1e-13
    for r in range(rc.shape[0]):
        ref = ses.coarse_solve(rc[r])
        assert np.linalg.norm(x[r] - ref) / np.linalg.norm(ref) < 1e-12


def test_nd_delayed_pivots_near_resonance():
    """cfg2 substitute (40 wavelengths, layer): boxes of the dissection sit close to
    Dirichlet resonances. Pivoting restricted to a front leaves a backward error of
    ~1e-10; threshold pivoting with delayed pivots brings it to rounding level."""
    kw = dict(order=4, wavelengths=40, ppw=12, side_tags=(N_, A_, N_, A_), layer_sides=(0, 2))
    prob = hb.build_problem(hb.ProblemSpec(**kw))
    nv = (prob.n_cells * 2 + 1) ** 2
    rc = _rhs(nv, 2, 1)
    _, be0, st0 = coarse_check(prob, rc, pivtol=0.0)
    _, be, st = coarse_check(prob, rc, pivtol=0.3)
    assert st0["delayed"] == 0 and be0 > 1e-12  # the failure mode exists on this case
    assert st["delayed"] > 0 and be < 1e-12
    assert st["max_front"] <= st0["max_front"] + 8  # delays stay local


D_ = hb.DIRICHLET
FE_CASES = [dict(order=4, wavelengths=3, ppw=10),
            dict(order=4, wavelengths=3, ppw=8, side_tags=(D_, A_, N_, A_)),
            dict(order=2, wavelengths=3, ppw=8, side_tags=(A_, D_, A_, N_), layer_sides=(0,), layer_width_dofs=6),
            dict(order=6, wavelengths=2, ppw=12)]


@pytest.mark.parametrize("kw", FE_CASES)
def test_fe_lattice_matches_oracle_assembly(kw):
    """fe_lattice(q = p, alpha_s) == the oracle's A_s, and fe_lattice(q = p/2, alpha_c) == the
    GalerkinP coarse matrix (proj/core/src/fespace.cpp:181-210, twogrid.cpp:189-219), applied to
    seeded vectors."""
    prob = hb.build_problem(hb.ProblemSpec(**kw))
    cfg = po.SolverConfig(coarsening=1, alpha_c=0.05)
    ses = po.Session(po.ProblemSpec(**kw), cfg)
    g = np.random.default_rng(5)
    x = g.standard_normal(ses.ndof) + 1j * g.standard_normal(ses.ndof)
    want = ses.apply(1, x)
    got = fe_apply(prob, kw["order"], cfg.alpha_s, x)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-13
    xc = g.standard_normal(ses.coarse_ndof) + 1j * g.standard_normal(ses.coarse_ndof)
    want = ses.apply(2, xc)
    got = fe_apply(prob, kw["order"] // 2, cfg.alpha_c, xc)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-13


@pytest.mark.parametrize("kw", FE_CASES[:3])
def test_fe_nd_solve(kw):
    """ND factors of the FE lattice matrices (separators on element-boundary lines) solve
    A_s x = b and A_c x = b to rounding level."""
    prob = hb.build_problem(hb.ProblemSpec(**kw))
    p = kw["order"]
    for q, alpha in ((p, 0.2), (p // 2, 0.05)):
        n = (prob.n_cells * q + 1) ** 2
        g = np.random.default_rng(q)
        b = g.standard_normal((2, n)) + 1j * g.standard_normal((2, n))
        x, st = fe_solve(prob, q, alpha, b)
        for r in range(2):
            res = fe_apply(prob, q, alpha, x[r]) - b[r]
            assert np.linalg.norm(res) / np.linalg.norm(b[r]) < 1e-12, (q, st)


def test_nd_shared_fronts_equal_unshared(monkeypatch):
    """Fronts with bit-identical assembled matrices share one set of factor blocks
    (uniform medium: most of the tree). The shared factorization must give the same
    solution, bit for bit, as factoring every front (HTG_ND_SHARE=0), and still match the
    oracle's coarse solve; a medium with a different k in every cell finds nothing to share
    beyond chance and stays correct."""
    kw = dict(order=4, wavelengths=16, ppw=10)  # 40 x 40 cells: 81 x 81 coarse vertices
    prob = hb.build_problem(hb.ProblemSpec(**kw))
    ses = po.Session(po.ProblemSpec(**kw), po.SolverConfig())
    rc = _rhs(ses.coarse_ndof, 3, 1)
    x1, be1, st1 = coarse_check(prob, rc)
    monkeypatch.setenv("HTG_ND_SHARE", "0")
    x0, be0, st0 = coarse_check(prob, rc)
    monkeypatch.delenv("HTG_ND_SHARE")
    assert st0["shared"] == 0 and st1["shared"] > st1["nodes"] // 2
    assert np.array_equal(x0, x1)
    assert be1 < 1e-13
    ref = ses.coarse_solve(rc[0])
    assert np.linalg.norm(x1[0] - ref) / np.linalg.norm(ref) < 1e-12
    # heterogeneous medium
    g = np.random.default_rng(11)
    prob_h = hb.build_problem(hb.ProblemSpec(**kw))
    prob_h.k_cells = prob_h.k_cells * g.uniform(0.9, 1.1, size=prob_h.k_cells.shape)
    xh, beh, sth = coarse_check(prob_h, rc)
    assert beh < 1e-12 and sth["shared"] < sth["nodes"] // 10
