"""Time the coarse solve (graph replay) for several ND tuning settings (env vars)."""
import json
import os
import subprocess
import sys

settings = []
LEAFS = [int(v) for v in os.environ.get("SWEEP_LEAF", "9,16,36,64").split(",")]
WARPFS = [int(v) for v in os.environ.get("SWEEP_WARPF", "64,96,128").split(",")]
MIDS = [int(v) for v in os.environ.get("SWEEP_MID", "8192,16384,65536").split(",")]
RPTS = [int(v) for v in os.environ.get("SWEEP_RPT", "8").split(",")]
for leaf in LEAFS:
    for warpf in WARPFS:
        for mid in MIDS:
            for rpt in RPTS:
                settings.append(dict(HTG_ND_LEAF=leaf, HTG_ND_WARPF=warpf, HTG_ND_MIDDATA=mid, HTG_ND_RPT=rpt))
code = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2509_17494_b200 as hb
prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=float(sys.argv[1]), ppw=10))
ops = hb.setup_two_grid(prob, hb.SolverConfig())
f = torch.from_numpy(prob.rhs).cuda(); u = torch.zeros_like(f)
p = ops.profile(u, f, reps=10)
print(p["coarse_solve_graph"], ops.coarse_factor_bytes)
'''
W = sys.argv[1] if len(sys.argv) > 1 else "160"
for s in settings:
    env = dict(os.environ, **{k: str(v) for k, v in s.items()})
    out = subprocess.run([sys.executable, "-c", code, W], env=env, capture_output=True, text=True)
    print(json.dumps(s), out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:], flush=True)
