"""One-pass windowed pGS (fused_w.cu) probe: ms per application and the
producer's frontier polls for several skew margins D - DT (set_fused_window)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2112_14681_b200 as nsm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
margins = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"])]
A, offsets, kind, k_l, k_u, desc = bench.build_workload(cfg, 0, 1)
S = nsm.Smoother(A)
b = torch.from_numpy(inputs.uniform(0, A.nrows)).cuda()
x = torch.from_numpy(inputs.uniform(1, A.nrows)).cuda()
flush = torch.zeros(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
for mode in ("off", "on"):
    for mg in (margins if mode == "on" else [0]):
        S.set_fused(3 if mode == "on" else 0)
        S.set_fused_window(mg)
        for _ in range(3):
            S.smooth(b, x, "pgs", nu=1, k_l=k_l)
        torch.cuda.synchronize()
        w0 = S.fused_stats()
        ts = []
        for _ in range(10):
            flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            S.smooth(b, x, "pgs", nu=1, k_l=k_l)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        w1 = S.fused_stats()
        S.check()
        print(f"{cfg} fused={mode} margin={mg}: {np.median(ts):.3f} ms/apply; polls/apply "
              f"{(w1[0] - w0[0]) / 10:.0f}, poll time/apply {(w1[1] - w0[1]) / 10 / 1e3:.0f} us (summed over CTAs)",
              flush=True)
