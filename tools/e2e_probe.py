"""Where the e2e (host-buffer) smoother time goes at cfg4: copies vs sweep vs call overhead."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17494_b200 as hb
prob = hb.build_problem(hb.ProblemSpec(order=4, wavelengths=160, ppw=10))
ops = hb.setup_two_grid(prob, hb.SolverConfig(coarsening=hb.twogrid.NONE))
n = ops.ndof
g = np.random.default_rng(1)
uh = torch.zeros(n, dtype=torch.complex128).pin_memory().numpy()
fh = torch.from_numpy(g.standard_normal(n) + 1j * g.standard_normal(n)).pin_memory().numpy()
def t(fn, k=20):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
print("csdd_smoother_host", t(lambda: ops.csdd_smoother_host(uh, fh)), "ms")
ud = torch.zeros(n, dtype=torch.complex128, device="cuda"); fd = torch.zeros_like(ud)
ut, ft = torch.from_numpy(uh), torch.from_numpy(fh)
def dev():
    fd.copy_(ft, non_blocking=True); ud.copy_(ut, non_blocking=True); ops.csdd_smoother(ud, fd); ut.copy_(ud, non_blocking=True)
print("torch copies + device sweep", t(dev), "ms")
print("device sweep only", t(lambda: ops.csdd_smoother(ud, fd)), "ms")
