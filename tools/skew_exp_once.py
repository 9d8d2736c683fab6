"""Run a few fused applications with a given wait window (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs, paper_2112_14681_b200 as nsm
import bench
cfg, w = sys.argv[1], int(sys.argv[2])
A, offsets, kind, k_l, k_u, desc = bench.build_workload(cfg, 0, 1)
F = nsm.ilu0(A) if kind == "ilu" else None
S = nsm.Smoother(A, F)
S.set_fused(1); S.set_fused_window(w)
b = torch.from_numpy(inputs.uniform(0, A.nrows)).cuda()
x = torch.from_numpy(inputs.uniform(1, A.nrows)).cuda()
for _ in range(8):
    S.smooth(b, x, kind, 1, k_l, k_u)
torch.cuda.synchronize(); S.check()
