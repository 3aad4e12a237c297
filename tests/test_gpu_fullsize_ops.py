"""Each hot-path operation at the full-size configs 3 (80 wavelengths, 641,601 dofs)
and 4 (160 wavelengths, 2,563,201 dofs), one at a time, against the REFERENCE's own
code (oracle/_ref/libhelmtg_ref.so: proj/core/src/*.cpp compiled unmodified against
oracle/eigen_shim; prebuilt, it travels with the repo, /root/reference is not read):

  residual f - A u and f - A_s u         (twogrid.cpp:116, :94)
  dd_step                                (twogrid.cpp:92-112)
  one csdd_smoother sweep                (twogrid.cpp:114-120)
  restriction IP^H r, and IP^H (f - A u) (twogrid.cpp:272)
  prolongation u + omega IP u_c          (twogrid.cpp:273)
  QSFEM A_c x                            (qsfem.cpp:118-149)

The reference's coarse level is built by its own coarse_mesh_for / coarsen_* /
qsfem::assemble / build_prolongation (ref_add_coarse_parts) without its coarse
SparseLU, which takes hours at these sizes; the GPU coarse solve is checked by its
backward error against the reference's A_c instead.
North-star tolerance: relative l2 <= 1e-10 per application."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module", params=[80, 160], ids=["cfg3", "cfg4"])
def fullsize(request):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import pyref
    if not os.path.exists(pyref.LIB_PATH):
        pytest.skip("oracle/_ref/libhelmtg_ref.so not built")
    import paper_2509_17494_b200 as hb
    W = request.param
    spec = dict(order=4, wavelengths=W, ppw=10)
    pyref.set_threads(os.cpu_count() or 1)
    ref = pyref.RefSession(po.ProblemSpec(**spec), po.SolverConfig(coarsening=2))
    ref.add_coarse_parts()
    prob = hb.build_problem(hb.ProblemSpec(**spec))
    ops = hb.setup_two_grid(prob, hb.SolverConfig())
    assert (ops.ndof, ops.coarse_ndof) == (ref.ndof, ref.coarse_ndof)
    g = np.random.default_rng(2000 + W)
    cv = lambda n: g.standard_normal(n) + 1j * g.standard_normal(n)  # noqa: E731
    data = dict(u=cv(ops.ndof), f=cv(ops.ndof), uc=cv(ops.coarse_ndof))
    yield ref, ops, data, torch
    ops.close()


def test_residual(fullsize):
    ref, ops, d, torch = fullsize
    u, f = torch.from_numpy(d["u"]).cuda(), torch.from_numpy(d["f"]).cuda()
    r = torch.empty_like(u)
    for shifted in (False, True):
        got = ops.residual(f, u, r, shifted=shifted).cpu().numpy()
        err = rel(got, ref.residual(d["f"], d["u"], shifted=shifted))
        print(f"ndof={ops.ndof} residual shifted={shifted}: {err:.2e}")
        assert err <= TOL


def test_dd_step_and_sweep(fullsize):
    ref, ops, d, torch = fullsize
    u, f = torch.from_numpy(d["u"]).cuda(), torch.from_numpy(d["f"]).cuda()
    out = torch.empty_like(u)
    err = rel(ops.dd_step(u, f, out).cpu().numpy(), ref.dd_step(d["u"], d["f"]))
    print(f"ndof={ops.ndof} dd_step: {err:.2e}")
    assert err <= TOL
    us = u.clone()
    err = rel(ops.csdd_smoother(us, f).cpu().numpy(), ref.csdd_smoother(d["u"], d["f"]))
    print(f"ndof={ops.ndof} csdd_smoother sweep: {err:.2e}")
    assert err <= TOL


def test_transfers_and_coarse_apply(fullsize):
    ref, ops, d, torch = fullsize
    u, f = torch.from_numpy(d["u"]).cuda(), torch.from_numpy(d["f"]).cuda()
    uc = torch.from_numpy(d["uc"]).cuda()
    rc = torch.empty_like(uc)
    # restriction of a given fine vector, and fused with the residual
    err = rel(ops.restrict(f, rc).cpu().numpy(), ref.apply(4, d["f"]))
    print(f"ndof={ops.ndof} restrict IP^H r: {err:.2e}")
    assert err <= TOL
    err = rel(ops.residual_restrict(f, u, rc).cpu().numpy(), ref.apply(4, ref.residual(d["f"], d["u"])))
    print(f"ndof={ops.ndof} IP^H (f - A u): {err:.2e}")
    assert err <= TOL
    # prolongation u + omega IP u_c (omega_c = 1 and a non-trivial weight)
    for om in (1.0, 0.7):
        got = ops.prolong_add(u.clone(), uc, om).cpu().numpy()
        err = rel(got, d["u"] + om * ref.apply(3, d["uc"]))
        print(f"ndof={ops.ndof} u + {om} IP u_c: {err:.2e}")
        assert err <= TOL
    # K4: QSFEM A_c x
    y = torch.empty_like(uc)
    err = rel(ops.coarse_apply(uc, y).cpu().numpy(), ref.apply(2, d["uc"]))
    print(f"ndof={ops.ndof} A_c x: {err:.2e}")
    assert err <= TOL


def test_coarse_solve_backward_error(fullsize):
    """The GPU nested-dissection solve against the reference's own A_c: ||A_c u_c - r_c|| / ||r_c||."""
    ref, ops, d, torch = fullsize
    rc = torch.from_numpy(d["uc"]).cuda()
    uc = torch.empty_like(rc)
    got = ops.coarse_solve(rc, uc).cpu().numpy()
    err = rel(ref.apply(2, got), d["uc"])
    print(f"coarse ndof={ops.coarse_ndof} backward error of A_c^-1 r_c: {err:.2e}")
    assert err <= TOL
