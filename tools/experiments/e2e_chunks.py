"""C3 e2e (nsm_smooth_host, pinned host vectors) against the number of row
chunks (NSM_HOST_CHUNKS_N, libnsm_exp.so) and without chunking; events around
each call as in bench.py, L2 not flushed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import bench, inputs
import paper_2112_14681_b200 as nsm

nsm.load(variant="exp")
CFG = sys.argv[1] if len(sys.argv) > 1 else "C3"
A, offsets, kind, k_l, k_u, desc = bench.build_workload(CFG, 0, 1)
S = nsm.Smoother(A)
bh = torch.from_numpy(inputs.uniform(inputs.SEED_B, A.nrows)).pin_memory()
xh = torch.from_numpy(inputs.uniform(inputs.SEED_X0, A.nrows)).pin_memory()
xo = torch.empty_like(xh).pin_memory()
st = torch.cuda.current_stream()
for label in (sys.argv[2:] or ["16", "24", "32", "off"]):
    if label == "off":
        S.set_host_chunks(False)
    else:
        os.environ["NSM_HOST_CHUNKS_N"] = label
    S.smooth_host(bh, xh, "pgs", k_l=2, out=xo)
    ts = []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        S.smooth_host(bh, xh, "pgs", k_l=2, out=xo)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{CFG} chunks {label:>5}: {np.median(ts):.3f} ms per step (min {min(ts):.3f})", flush=True)
