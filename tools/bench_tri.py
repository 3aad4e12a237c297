"""Triangle-element problem (ElementKind::Triangle) at a BASELINE size: setup time,
smoother sweep and two-grid step times (cold L2), one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17494_b200 as hb  # noqa: E402

W = float(os.environ.get("TRI_W", 80))
prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=W, ppw=10, element_kind=hb.twogrid.TRIANGLE))
t0 = time.perf_counter()
ops = hb.setup_two_grid(prob, hb.SolverConfig())
setup = time.perf_counter() - t0
n = ops.ndof
g = np.random.default_rng(7)
f = torch.from_numpy(g.standard_normal(n) + 1j * g.standard_normal(n)).cuda()
u = torch.zeros_like(f)
prof = ops.profile(u, f, reps=5)
res = ops.solve(torch.from_numpy(prob.rhs).cuda())
print(json.dumps({"workload": f"Q4 triangles (P4 on split cells), {W:.0f} wavelengths, 10 ppw, {n} dofs",
                  "setup_s": setup, "sweep_ms": prof["smoother_sweep_graph"], "sweep_dof_per_s": n / (prof["smoother_sweep_graph"] * 1e-3),
                  "two_grid_step_ms": prof["two_grid_step_graph"], "residual_ms": prof["residual"],
                  "subdomain_solves_ms": prof["dd_gemm"], "iterations": res.iterations,
                  "kernel_ms": {k: round(v, 4) for k, v in prof.items()}}))
