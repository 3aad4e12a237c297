"""GPU parity on rectangles (nx != ny) with per-cell heterogeneous k and eps and
mixed boundary tags: the coefficient-class tables, non-separable subdomain
classes (dense path), remainder blocks of the partition and the non-square
coarse lattice, against the oracle built from the same description."""
import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
A_, N_, D_ = po.ABSORBING, po.NEUMANN, po.DIRICHLET
TOL = 1e-10
CASES = {
    "p4_13x7_hetero": dict(order=4, nx=13, ny=7, h=0.05, sides=(A_, D_, N_, A_), kr=(8.0, 12.0), er=0.5, seed=3),
    "p2_9x16_hetero": dict(order=2, nx=9, ny=16, h=1.0 / 16, sides=(D_, A_, A_, N_), kr=(5.0, 9.0), er=0.0, seed=4),
    "p4_11x5_layer_like": dict(order=4, nx=11, ny=5, h=0.1, sides=(N_, A_, A_, A_), kr=(4.0, 4.0), er=3.0, seed=5),
}


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("cfg", [dict(), dict(coarsening=1, alpha_c=0.05), dict(smoother=1, outer=1)],
                         ids=["csdd_qsfem", "csdd_galerkin", "exact_krylov"])
def test_rect_heterogeneous(name, cfg):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_17494_b200 as hb
    c = CASES[name]
    g = np.random.default_rng(c["seed"])
    k = g.uniform(*c["kr"], size=(c["ny"], c["nx"]))
    eps = c["er"] * g.random((c["ny"], c["nx"]))
    ses = po.Session(desc=dict(order=c["order"], nx=c["nx"], ny=c["ny"], h=c["h"], k=k, eps=eps,
                               side_tags=c["sides"]), config=po.SolverConfig(**cfg))
    n = ses.ndof
    f, u = po.random_vector(n, 21), po.random_vector(n, 22)
    prob = hb.twogrid.Problem(order=c["order"], n_cells=c["nx"], h=c["h"], k=float(k.mean()),
                              k_cells=np.ascontiguousarray(k.ravel()), eps_cells=np.ascontiguousarray(eps.ravel()),
                              side_tags=c["sides"], rhs=f, ny=c["ny"])
    ops = hb.setup_two_grid(prob, hb.SolverConfig(**cfg))
    assert ops.ndof == n and ops.coarse_ndof == ses.coarse_ndof
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    r = torch.zeros_like(d(f))
    ops.residual(d(f), d(u), r)
    assert rel(r.cpu().numpy(), ses.residual(f, u)) <= TOL
    if cfg.get("smoother", 0) == 0:
        ud = d(u)
        ops.csdd_smoother(ud, d(f))
        assert rel(ud.cpu().numpy(), ses.csdd_smoother(u, f)) <= TOL
    ud = d(u)
    ops.two_grid_step(ud, d(f))
    assert rel(ud.cpu().numpy(), ses.two_grid_step(u, f)) <= TOL
    rc = po.random_vector(ses.coarse_ndof, 23)
    y = torch.zeros_like(d(rc))
    ops.coarse_solve(d(rc), y)
    assert rel(y.cpu().numpy(), ses.coarse_solve(rc)) <= TOL
    res, ref = ops.solve(d(f)), ses.solve(f)
    assert res.converged == ref.converged and abs(res.iterations - ref.iterations) <= 1
    ops.close()
