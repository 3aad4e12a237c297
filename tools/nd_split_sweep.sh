for s in 3 4 5 6; do
  HTG_ND_SPLIT=$s python -c "
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2509_17494_b200 as hb
prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=160, ppw=10))
ops = hb.setup_two_grid(prob, hb.SolverConfig())
f = torch.from_numpy(prob.rhs).cuda(); u = torch.zeros_like(f)
p = ops.profile(u, f, reps=10)
print('split', $s, p['coarse_solve_graph'], p['two_grid_step_graph'])
"
done
