"""The CUDA path against the committed golden fixtures (tests/golden/), without the
oracle at run time. Tolerance: relative l2 <= 1e-10 per entry point (north star);
solve iteration counts within +-1."""
import ast
import glob
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_gpu_matches_golden(path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_17494_b200 as hb
    g = np.load(path)
    spec, cfg = ast.literal_eval(str(g["spec"])), ast.literal_eval(str(g["config"]))
    prob = hb.build_problem(hb.ProblemSpec(**spec))
    assert np.array_equal(prob.rhs, g["rhs"])
    ops = hb.setup_two_grid(prob, hb.SolverConfig(**cfg))
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    h = lambda t: t.cpu().numpy()  # noqa: E731
    f, u, rc = d(g["f"]), d(g["u"]), d(g["rc"])
    r = torch.zeros_like(f)
    ops.residual(f, u, r)
    assert rel(h(r), g["residual"]) <= TOL
    ops.residual(f, u, r, shifted=True)
    assert rel(h(r), g["residual_shifted"]) <= TOL
    y = torch.zeros_like(rc)
    ops.restrict(f, y)
    assert rel(h(y), g["restrict"]) <= TOL
    ops.coarse_apply(rc, y)
    assert rel(h(y), g["coarse_apply"]) <= TOL
    ops.coarse_solve(rc, y)
    assert rel(h(y), g["coarse_solve"]) <= TOL
    z = torch.zeros_like(f)
    ops.prolong_add(z, rc, 1.0)
    assert rel(h(z), g["prolong"]) <= TOL
    if "dd_step" in g:
        ops.dd_step(u, f, z)
        assert rel(h(z), g["dd_step"]) <= TOL
        uu = u.clone()
        ops.csdd_smoother(uu, f)
        assert rel(h(uu), g["csdd_smoother"]) <= TOL
    uu = u.clone()
    ops.two_grid_step(uu, f)
    assert rel(h(uu), g["two_grid_step"]) <= TOL
    res = ops.solve(d(g["rhs"]))
    assert abs(res.iterations - int(g["solve_iterations"])) <= 1
    ops.close()
