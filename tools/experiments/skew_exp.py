"""Fused-pass experiments: ms per application vs wait window, per config."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2112_14681_b200 as nsm
import bench

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
windows = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"])]
A, offsets, kind, k_l, k_u, desc = bench.build_workload(cfg, 0, 1)
F = nsm.ilu0(A) if kind == "ilu" else None
S = nsm.Smoother(A, F)
b = torch.from_numpy(inputs.uniform(0, A.nrows)).cuda()
x = torch.from_numpy(inputs.uniform(1, A.nrows)).cuda()
flush = torch.zeros(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
for mode, w in [("off", 0)] + [("on", w) for w in windows]:
    S.set_fused(0 if mode == "off" else 1)
    S.set_fused_window(w)
    for _ in range(3):
        S.smooth(b, x, kind, 1, k_l, k_u)
    ts = []
    for _ in range(10):
        bench.flush_l2(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); S.smooth(b, x, kind, 1, k_l, k_u); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    S.check()
    w0 = S.fused_stats()
    S.smooth(b, x, kind, 1, k_l, k_u)
    w1 = S.fused_stats()
    print(json.dumps({"cfg": cfg, "mode": mode, "window": w, "ms": round(float(np.median(ts)), 4),
                      "waits": w1[0] - w0[0], "wait_us": round((w1[1] - w0[1]) / 1e3, 1),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("NSM_DEBUG")}}), flush=True)
