"""One V-cycle of the 27-point 64^3 hierarchy (for ncu launch lists), plus
the event-timed V-cycle (eager launches) for comparison."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, oracle
from oracle import amg
import paper_2112_14681_b200 as nsm
N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
A = inputs.var27(N).to_scipy()
rand_fn = lambda level, n: inputs.uniform(1000 + level, n, 0.0, 1.0)
levels = amg.hierarchy(A, rand_fn, min_coarse=200)
nl = len(levels) - 1
S = [nsm.Smoother(inputs.CSR.from_scipy(levels[l][0])) for l in range(nl)]
M = nsm.Amg(S, [inputs.CSR.from_scipy(levels[l][1]) for l in range(nl)], inputs.CSR.from_scipy(levels[-1][0]))
for l in range(nl):
    M.set_smoother(l, "pgs", 1, 1, 1, 1)
b = torch.from_numpy(inputs.uniform(0, A.shape[0])).cuda()
x = torch.empty_like(b)
for _ in range(3):
    M.vcycle(b, x)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); M.vcycle(b, x); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print("levels", [lv[0].shape[0] for lv in levels], "eager V-cycle ms", round(float(np.median(ts)), 4))
