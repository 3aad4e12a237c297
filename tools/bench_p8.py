"""Setup and sweep time of a high-order problem (default Q8, 40 wavelengths, 8 ppw):
shared-class device factors (default) vs host dense inverses (HTG_BAND=0)."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17494_b200 as hb  # noqa: E402
p = int(os.environ.get("P", 8)); W = float(os.environ.get("W", 40)); ppw = float(os.environ.get("PPW", 8))
prob = hb.build_problem(hb.ProblemSpec(order=p, wavelengths=W, ppw=ppw))
t0 = time.perf_counter()
ops = hb.setup_two_grid(prob, hb.SolverConfig())
setup = time.perf_counter() - t0
f = torch.from_numpy(prob.rhs).cuda(); u = torch.zeros_like(f)
prof = ops.profile(u, f, reps=5)
res = ops.solve(f)
print(json.dumps({"p": p, "W": W, "ndof": ops.ndof, "band_subdomains": ops.band_subdomains, "subdomains": ops.n_subdomains,
                  "setup_s": setup, "sweep_ms": prof["smoother_sweep_graph"], "solves_ms": prof["dd_gemm"],
                  "two_grid_ms": prof["two_grid_step_graph"], "iterations": res.iterations}))
