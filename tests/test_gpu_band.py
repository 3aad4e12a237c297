"""Subdomains that share no factor (a heterogeneous medium makes every subdomain
operator unique): the device-factored per-subdomain solver (csrc/k_band.cu:
static condensation + banded L D L^T, assembled and factored on the GPU) against
the restated oracle and against the REFERENCE's own code, which factors every
subdomain with its own SparseLU (proj/core/src/twogrid.cpp:76-90, 92-112).
Tolerance: relative l2 <= 1e-10 per dd_step / smoother sweep (north star)."""
import os
import time

import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
A_, N_, D_ = po.ABSORBING, po.NEUMANN, po.DIRICHLET
TOL = 1e-10
CASES = {
    "p4_14x11_mixed": dict(order=4, nx=14, ny=11, h=0.05, sides=(A_, D_, N_, A_), kr=(8.0, 12.0), er=0.5, seed=31,
                           l_dd=4),
    "p2_13x9_dir": dict(order=2, nx=13, ny=9, h=1.0 / 13, sides=(D_, A_, D_, N_), kr=(5.0, 9.0), er=0.2, seed=32,
                        l_dd=4),
    "p6_9x10_abs": dict(order=6, nx=9, ny=10, h=0.1, sides=(A_, A_, A_, A_), kr=(6.0, 8.0), er=0.0, seed=33, l_dd=4),
    "p8_7x8_mixed": dict(order=8, nx=7, ny=8, h=0.125, sides=(N_, A_, D_, A_), kr=(6.0, 9.0), er=1.0, seed=34,
                         l_dd=3),
    "p4_10x10_ldd3_dir": dict(order=4, nx=10, ny=10, h=0.1, sides=(D_, D_, D_, D_), kr=(4.0, 6.0), er=0.3, seed=35,
                              l_dd=3),
}


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def hetero(c):
    g = np.random.default_rng(c["seed"])
    k = g.uniform(*c["kr"], size=(c["ny"], c["nx"]))
    eps = c["er"] * g.random((c["ny"], c["nx"]))
    return k, eps


def gpu_problem(hb, c, k, eps, f):
    return hb.twogrid.Problem(order=c["order"], n_cells=c["nx"], h=c["h"], k=float(k.mean()),
                              k_cells=np.ascontiguousarray(k.ravel()), eps_cells=np.ascontiguousarray(eps.ravel()),
                              side_tags=c["sides"], rhs=f, ny=c["ny"])


@pytest.mark.parametrize("name", list(CASES))
def test_band_subdomains_match_oracle(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_17494_b200 as hb
    c = CASES[name]
    k, eps = hetero(c)
    cfg = dict(l_dd=c["l_dd"])
    ses = po.Session(desc=dict(order=c["order"], nx=c["nx"], ny=c["ny"], h=c["h"], k=k, eps=eps,
                               side_tags=c["sides"]), config=po.SolverConfig(**cfg))
    n = ses.ndof
    f, u = po.random_vector(n, 41), po.random_vector(n, 42)
    ops = hb.setup_two_grid(gpu_problem(hb, c, k, eps, f), hb.SolverConfig(**cfg))
    # every subdomain sees its own coefficients: all of them take the device-factored path
    assert ops.band_subdomains == ops.n_subdomains > 0, (ops.band_subdomains, ops.n_subdomains)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    out = torch.zeros_like(d(u))
    err = rel(ops.dd_step(d(u), d(f), out).cpu().numpy(), ses.dd_step(u, f))
    print(f"{name}: {ops.band_subdomains} band subdomains, dd_step rel err {err:.2e}")
    assert err <= TOL
    ud = d(u)
    ops.csdd_smoother(ud, d(f))
    assert rel(ud.cpu().numpy(), ses.csdd_smoother(u, f)) <= TOL
    ud = d(u)
    ops.two_grid_step(ud, d(f))
    assert rel(ud.cpu().numpy(), ses.two_grid_step(u, f)) <= TOL
    res, ref = ops.solve(d(f)), ses.solve(f)
    assert res.converged == ref.converged and abs(res.iterations - ref.iterations) <= 1
    ops.close()


def test_band_matches_reference_own_subdomain_lu():
    """64 x 48 cells, Q4, random k and eps per cell (768 ... subdomains, each with its own
    factor): dd_step and one sweep against the reference's own per-subdomain SparseLU."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import pyref
    if not os.path.exists(pyref.LIB_PATH):
        pytest.skip("oracle/_ref/libhelmtg_ref.so not built")
    import paper_2509_17494_b200 as hb
    c = dict(order=4, nx=64, ny=48, h=1.0 / 64, sides=(A_, A_, N_, A_), kr=(30.0, 40.0), er=2.0, seed=36)
    k, eps = hetero(c)
    pyref.set_threads(os.cpu_count() or 1)
    ref = pyref.RefSession(desc=dict(order=4, nx=c["nx"], ny=c["ny"], h=c["h"], k=k, eps=eps,
                                     side_tags=c["sides"]), config=po.SolverConfig(coarsening=2))
    assert ref.n_factors == ref.n_subdomains  # the reference factors every subdomain
    n = ref.ndof
    f, u = po.random_vector(n, 43), po.random_vector(n, 44)
    ops = hb.setup_two_grid(gpu_problem(hb, c, k, eps, f), hb.SolverConfig())
    assert ops.band_subdomains == ops.n_subdomains == ref.n_subdomains
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    out = torch.zeros_like(d(u))
    err = rel(ops.dd_step(d(u), d(f), out).cpu().numpy(), ref.dd_step(u, f))
    print(f"64x48 Q4 heterogeneous, {ops.band_subdomains} subdomains: dd_step vs reference {err:.2e}")
    assert err <= TOL
    ud = d(u)
    ops.csdd_smoother(ud, d(f))
    err = rel(ud.cpu().numpy(), ref.csdd_smoother(u, f))
    print(f"  csdd_smoother vs reference {err:.2e}")
    assert err <= TOL
    ops.close()


def test_band_cfg4_size_heterogeneous():
    """A cfg4-size medium (400 x 400 cells, Q4, 2,563,201 dofs) with a random k per cell:
    10,000 subdomains, each factored on the device. Setup in seconds, factors < 5 GB,
    and dd_step / one sweep equal to the reference's own (10,000 SparseLU factors)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import pyref
    if not os.path.exists(pyref.LIB_PATH):
        pytest.skip("oracle/_ref/libhelmtg_ref.so not built")
    import paper_2509_17494_b200 as hb
    c = dict(order=4, nx=400, ny=400, h=1.0 / 400, sides=(A_, A_, A_, A_), seed=37)
    g = np.random.default_rng(c["seed"])
    k = 2 * np.pi * 160 * g.uniform(0.9, 1.1, size=(400, 400))
    eps = np.zeros((400, 400))
    n = (400 * 4 + 1) ** 2
    t0 = time.perf_counter()
    ops = hb.setup_two_grid(gpu_problem(hb, c, k, eps, np.zeros(n, complex)), hb.SolverConfig())
    t_setup = time.perf_counter() - t0
    print(f"cfg4-size heterogeneous: setup {t_setup:.2f} s, {ops.band_subdomains} device-factored subdomains, "
          f"factors {ops.band_factor_bytes / 1e9:.2f} GB")
    assert ops.band_subdomains == ops.n_subdomains == 10000
    assert ops.band_factor_bytes < 5e9
    assert t_setup < 60
    pyref.set_threads(os.cpu_count() or 1)
    ref = pyref.RefSession(desc=dict(order=4, nx=400, ny=400, h=c["h"], k=k, eps=eps, side_tags=c["sides"]),
                           config=po.SolverConfig(coarsening=2))
    rng = np.random.default_rng(38)
    u = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    out = torch.empty_like(d(u))
    err = rel(ops.dd_step(d(u), d(f), out).cpu().numpy(), ref.dd_step(u, f))
    print(f"  dd_step vs the reference: {err:.2e}")
    assert err <= TOL
    ud = d(u)
    ops.csdd_smoother(ud, d(f))
    err = rel(ud.cpu().numpy(), ref.csdd_smoother(u, f))
    print(f"  csdd_smoother vs the reference: {err:.2e}")
    assert err <= TOL
    ops.close()
