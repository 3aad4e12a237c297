"""Run the cfg4 hot path a few times (for ncu launch lists / captures)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17494_b200 as hb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--wavelengths", type=float, default=160)
ap.add_argument("--order", type=int, default=4)
ap.add_argument("--what", default="step", choices=["sweep", "step", "coarse", "capply", "prolong"])
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
prob = hb.build_problem(hb.ProblemSpec(order=a.order, wavelengths=a.wavelengths, ppw=10))
ops = hb.setup_two_grid(prob, hb.SolverConfig())
g = np.random.default_rng(1)
f = torch.from_numpy(g.standard_normal(ops.ndof) + 1j * g.standard_normal(ops.ndof)).cuda()
u = torch.zeros_like(f)
rc = torch.from_numpy(g.standard_normal(ops.coarse_ndof) + 0j).cuda()
uc = torch.zeros_like(rc)
for _ in range(a.reps):
    if a.what == "sweep":
        ops.csdd_smoother(u, f)
    elif a.what == "step":
        ops.two_grid_step(u, f)
    elif a.what == "capply":
        ops.coarse_apply(rc, uc)
    elif a.what == "prolong":
        ops.prolong_add(u, rc, 1.0)
    else:
        ops.coarse_solve(rc, uc)
torch.cuda.synchronize()
print("ok", ops.ndof, ops.coarse_levels, ops.coarse_factor_bytes / 1e9, "GB coarse factors")
