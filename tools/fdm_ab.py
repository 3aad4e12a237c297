"""Time the FDM subdomain kernel (htg_profile, cold L2) at cfg3 and cfg4 for the current
HTG_FDM_* environment; one line per config. Coarse level off (only the sweep kernels run)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17494_b200 as hb  # noqa: E402

tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("HTG_"))
for wl in [float(w) for w in os.environ.get("AB_WL", "80,160").split(",")]:
    prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=wl, ppw=10))
    ops = hb.setup_two_grid(prob, hb.SolverConfig(coarsening=hb.twogrid.NONE))
    g = np.random.default_rng(1)
    f = torch.from_numpy(g.standard_normal(ops.ndof) + 1j * g.standard_normal(ops.ndof)).cuda()
    u = torch.zeros_like(f)
    ms = ops.profile(u, f, reps=20)
    print(f"[{tag}] wl={wl:g} fdm {ms['dd_gemm']*1e3:.1f} us  K1 {ms['residual']*1e3:.1f} us  combine "
          f"{ms['dd_combine']*1e3:.1f} us  sweep(graph) {ms['smoother_sweep_graph']*1e3:.1f} us", flush=True)
    del ops
