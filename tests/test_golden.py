"""The committed golden fixtures (tests/golden/, made by tools/make_golden.py from the
pinned oracle) are reproduced by the oracle: guards the checker against drift."""
import ast
import glob
import os

import numpy as np
import pytest

from oracle import pyoracle as po

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_oracle_reproduces_golden(path):
    g = np.load(path)
    spec, cfg = ast.literal_eval(str(g["spec"])), ast.literal_eval(str(g["config"]))
    ses = po.Session(po.ProblemSpec(**spec), po.SolverConfig(**cfg))
    f, u, rc = g["f"], g["u"], g["rc"]
    assert np.array_equal(ses.rhs(), g["rhs"])
    assert rel(ses.residual(f, u), g["residual"]) < 1e-14
    assert rel(ses.residual(f, u, shifted=True), g["residual_shifted"]) < 1e-14
    assert rel(ses.apply(4, f), g["restrict"]) < 1e-14
    assert rel(ses.apply(3, rc), g["prolong"]) < 1e-14
    assert rel(ses.apply(2, rc), g["coarse_apply"]) < 1e-14
    assert rel(ses.coarse_solve(rc), g["coarse_solve"]) < 1e-12
    assert rel(ses.two_grid_step(u, f), g["two_grid_step"]) < 1e-12
    if "dd_step" in g:
        assert rel(ses.dd_step(u, f), g["dd_step"]) < 1e-12
        assert rel(ses.csdd_smoother(u, f), g["csdd_smoother"]) < 1e-12
    res = ses.solve(g["rhs"])
    assert res.iterations == int(g["solve_iterations"])
    assert rel(res.u, g["solve_u"]) < 1e-10
