"""Backward error and graph time of the GPU coarse solve (no oracle needed):
||A_c x - r|| / ||r|| with A_c applied by the GPU stencil kernel."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17494_b200 as hb
cases = {
    "cfg4": dict(order=4, wavelengths=160, ppw=10),
    "cfg2sub": dict(order=4, wavelengths=40, ppw=12, side_tags=(1, 2, 1, 2), layer_sides=(0, 2)),
    "cfg3": dict(order=4, wavelengths=80, ppw=10),
}
for name in (sys.argv[1:] or cases):
    prob = hb.build_problem(hb.ProblemSpec(**cases[name]))
    ops = hb.setup_two_grid(prob, hb.SolverConfig())
    g = torch.Generator(device="cuda").manual_seed(5)
    nc = ops.coarse_ndof
    rc = torch.randn(nc, dtype=torch.complex128, device="cuda", generator=g)
    uc = torch.empty_like(rc); y = torch.empty_like(rc)
    ops.coarse_solve(rc, uc); ops.coarse_apply(uc, y)
    be = (torch.linalg.vector_norm(y - rc) / torch.linalg.vector_norm(rc)).item()
    f = torch.from_numpy(prob.rhs).cuda(); u = torch.zeros_like(f)
    p = ops.profile(u, f, reps=10)
    print(name, "coarse backward", be, "coarse_solve_graph ms", p["coarse_solve_graph"], "levels", ops.coarse_levels, flush=True)
