"""BASELINE configs 0 and 1 as specified (seeded complex Gaussian RHS, the
reference's default smoother and coarse level, solved to 1e-6): GPU iteration
counts equal the oracle's within +-1 and the solutions agree. Configs 2-4 are in
test_gpu_parity.py (cfg2 substitute) and test_gpu_fullsize_oracle.py."""
import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
CONFIGS = {
    # cfg0: Q2, 10 wavelengths at 10 dofs/wavelength, n_s = 2, Richardson
    "cfg0": (dict(order=2, wavelengths=10, ppw=10), dict(n_s=2), 1000),
    # cfg1: Q4, 20 wavelengths at 10 dofs/wavelength, defaults (n_s = 1), Richardson
    "cfg1": (dict(order=4, wavelengths=20, ppw=10), dict(), 1001),
}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_baseline_config(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_17494_b200 as hb
    spec, cfg, seed = CONFIGS[name]
    prob = hb.build_problem(hb.ProblemSpec(**spec))
    ops = hb.setup_two_grid(prob, hb.SolverConfig(**cfg))
    ses = po.Session(po.ProblemSpec(**spec), po.SolverConfig(**cfg))
    g = np.random.default_rng(seed)
    f = g.standard_normal(ops.ndof) + 1j * g.standard_normal(ops.ndof)
    ref = ses.solve(f)
    res = ops.solve(torch.from_numpy(f).cuda())
    print(f"{name}: {ops.ndof} dofs, GPU {res.iterations} iterations, oracle {ref.iterations}")
    assert ref.converged and res.converged and abs(res.iterations - ref.iterations) <= 1
    got = res.u.cpu().numpy()
    assert np.linalg.norm(got - ref.u) / np.linalg.norm(ref.u) <= 1e-8
    hist = np.asarray(res.residual_history[: len(ref.residual_history)])
    assert np.allclose(hist, np.asarray(ref.residual_history[: len(hist)]), rtol=1e-8)
    ops.close()
