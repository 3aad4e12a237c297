"""GPU parity of the FDM subdomain kernel in every team shape it can be launched in.

The default launch picks the shape from the load (eight 2-warp teams, or five 3-warp
teams when an SM gets few subdomains); HTG_FDM_TEAM / HTG_FDM_NTEAMS force the others,
including the lean 24-warp form. Each shape must reproduce the oracle's dd_step and
smoother sweep (relative l2 <= 1e-10, BASELINE.json north_star). The mesh has interior
subdomains of the 6 x 6-cell class (the compile-time path) next to edge and corner
classes (the generic path), and more subdomains per SM than a CTA has teams.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
TOL = 1e-10

SHAPES = [(None, None), ("1", None), ("2", None), ("2", "6"), ("3", "5"), ("3", "6"), ("3", "8"), ("4", None), ("2", "1")]


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


@pytest.fixture(scope="module")
def reference():
    spec = dict(order=4, wavelengths=56, ppw=10)  # 140 x 140 cells: 35 x 35 subdomains, 8.3 per SM
    ses = po.Session(po.ProblemSpec(**spec), po.SolverConfig(coarsening=2))  # no coarse level: sweeps only
    n = ses.ndof
    f = po.random_vector(n, 22)
    u0 = po.random_vector(n, 23)
    return spec, f, u0, ses.dd_step(u0, f), ses.csdd_smoother(u0, f)


@pytest.mark.parametrize("team,nteams", SHAPES)
def test_fdm_team_shapes(reference, team, nteams):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_17494_b200 as hb
    spec, f, u0, want_dd, want_sweep = reference
    saved = {k: os.environ.get(k) for k in ("HTG_FDM_TEAM", "HTG_FDM_NTEAMS")}
    try:
        for k, v in (("HTG_FDM_TEAM", team), ("HTG_FDM_NTEAMS", nteams)):
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        ops = hb.setup_two_grid(hb.build_problem(hb.ProblemSpec(**spec)), hb.SolverConfig(coarsening=hb.twogrid.NONE))
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert ops.fdm_subdomains == 35 * 35
    v = torch.zeros(ops.ndof, dtype=torch.complex128, device="cuda")
    ops.dd_step(torch.from_numpy(u0.copy()).cuda(), torch.from_numpy(f).cuda(), v)
    assert rel(v.cpu().numpy(), want_dd) <= TOL
    u = torch.from_numpy(u0.copy()).cuda()
    ops.csdd_smoother(u, torch.from_numpy(f).cuda())
    assert rel(u.cpu().numpy(), want_sweep) <= TOL
