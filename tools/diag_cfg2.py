"""Per-component parity of the cfg2 substitute (layer) against the oracle."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17494_b200 as hb
from oracle import pyoracle as po
N_, A_ = po.NEUMANN, po.ABSORBING
kw = dict(order=4, wavelengths=40, ppw=12, side_tags=(N_, A_, N_, A_), layer_sides=(po.LEFT, po.BOTTOM))
os_ = po.Session(po.ProblemSpec(**kw), po.SolverConfig())
prob = hb.build_problem(hb.ProblemSpec(**kw))
ops = hb.setup_two_grid(prob, hb.SolverConfig())
print("fdm subs", ops.fdm_subdomains, "of", ops.n_subdomains)
g = np.random.default_rng(1002)
n = ops.ndof
f = prob.rhs + 1e-3 * (g.standard_normal(n) + 1j * g.standard_normal(n))
u0 = po.random_vector(n, 9)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
h = lambda t: t.cpu().numpy()
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
r = torch.empty(n, dtype=torch.complex128, device="cuda"); ops.residual(d(f), d(u0), r)
print("residual", rel(h(r), os_.residual(f, u0)))
o = torch.empty_like(r); ops.dd_step(d(u0), d(f), o)
print("dd_step", rel(h(o), os_.dd_step(u0, f)))
ud = d(u0); ops.csdd_smoother(ud, d(f))
print("smoother", rel(h(ud), os_.csdd_smoother(u0, f)))
nc = ops.coarse_ndof if hasattr(ops, "coarse_ndof") else None
rc0 = po.random_vector(nc, 3) if nc else None
if nc:
    uc = torch.empty(nc, dtype=torch.complex128, device="cuda"); ops.coarse_solve(d(rc0), uc)
    ref = os_.coarse_solve(rc0)
    print("coarse_solve", rel(h(uc), ref), "cond-ish |uc|/|rc|", np.linalg.norm(ref) / np.linalg.norm(rc0))
ud = d(u0); ops.two_grid_step(ud, d(f))
print("two_grid_step", rel(h(ud), os_.two_grid_step(u0, f)))
# coarse solve on the actual restricted post-smoothing residual
ud = d(u0); ops.csdd_smoother(ud, d(f)); ud = d(os_.csdd_smoother(u0, f))
rc = torch.empty(nc, dtype=torch.complex128, device="cuda"); ops.residual_restrict(d(f), ud, rc)
rch = h(rc)
uc = torch.empty_like(rc); ops.coarse_solve(rc, uc); ucg = h(uc)
uco = os_.coarse_solve(rch)
be = lambda x: np.linalg.norm(os_.apply(2, x) - rch) / np.linalg.norm(rch)
print("real rc: rel", rel(ucg, uco), "backward gpu", be(ucg), "backward oracle", be(uco), "|uc|/|rc|", np.linalg.norm(uco)/np.linalg.norm(rch))
be0 = lambda x: np.linalg.norm(os_.apply(2, x) - rc0) / np.linalg.norm(rc0)
uc = torch.empty_like(rc); ops.coarse_solve(d(rc0), uc)
print("random rc: backward gpu", be0(h(uc)), "backward oracle", be0(os_.coarse_solve(rc0)))
