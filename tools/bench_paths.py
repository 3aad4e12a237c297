"""Time the alternative hot paths (GalerkinP coarse level, ExactShifted smoother) next
to the default one: setup, seconds per two-grid step (CUDA graph replay, CUDA events)
and the solve to 1e-6 (iterations, seconds). One JSON line per path.

  python tools/bench_paths.py [--out profiles/r01_paths.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17494_b200 as hb  # noqa: E402

PATHS = [
    ("cfg4 Q4 W=160: CSDD + OptimizedFD (default), GMRES", dict(order=4, wavelengths=160, ppw=10), dict(outer=1)),
    ("cfg4 Q4 W=160: CSDD + GalerkinP (acceptance C08 settings: alpha_s=alpha_c=0.02, l_dd=10), GMRES",
     dict(order=4, wavelengths=160, ppw=10), dict(coarsening=1, alpha_s=0.02, alpha_c=0.02, l_dd=10, outer=1)),
    ("cfg3 Q4 W=80: ExactShifted + OptimizedFD, GMRES", dict(order=4, wavelengths=80, ppw=10),
     dict(smoother=1, outer=1)),
    ("cfg3 Q4 W=80: CSDD + OptimizedFD (default), GMRES", dict(order=4, wavelengths=80, ppw=10), dict(outer=1)),
]


def run(name, spec, cfg, reps=10):
    prob = hb.build_problem(hb.ProblemSpec(**spec))
    t0 = time.perf_counter()
    ops = hb.setup_two_grid(prob, hb.SolverConfig(**cfg))
    setup = time.perf_counter() - t0
    g = np.random.default_rng(1004)
    f = torch.from_numpy(g.standard_normal(ops.ndof) + 1j * g.standard_normal(ops.ndof)).cuda()
    u = torch.zeros_like(f)
    for _ in range(2):
        ops.two_grid_step(u, f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ops.two_grid_step(u, f)
    e1.record()
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / reps
    fr = torch.from_numpy(prob.rhs).cuda()
    ops.solve(fr)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = ops.solve(fr)
    torch.cuda.synchronize()
    solve_s = time.perf_counter() - t0
    out = dict(path=name, ndof=ops.ndof, coarse_ndof=ops.coarse_ndof, setup_s=round(setup, 2),
               two_grid_step_ms=round(step_ms, 4), solve_iterations=res.iterations, converged=res.converged,
               solve_s=round(solve_s, 4), device_GB=round(ops.device_bytes / 1e9, 3))
    ops.close()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    lines = []
    for name, spec, cfg in PATHS:
        r = run(name, spec, cfg)
        print(json.dumps(r), flush=True)
        lines.append(r)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(lines, fh, indent=1)
