"""Producer counters of the one-pass windowed pGS (nsm_fused_counters) per application."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
import paper_2112_14681_b200 as nsm  # noqa: E402
if os.environ.get("FW_VARIANT"):
    nsm.load(variant=os.environ["FW_VARIANT"])

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
A, offsets, kind, k_l, k_u, desc = bench.build_workload(cfg, 0, 1)
S = nsm.Smoother(A)
if os.environ.get("PLANE_ROWS"):
    S.set_plane_rows(int(os.environ["PLANE_ROWS"]))
S.set_fused(3)
b = torch.from_numpy(inputs.uniform(0, A.nrows)).cuda()
x = torch.from_numpy(inputs.uniform(1, A.nrows)).cuda()
for mg in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"])]:
    S.set_fused_window(mg)
    for _ in range(3):
        S.smooth(b, x, "pgs", nu=1, k_l=k_l)
    torch.cuda.synchronize()
    c0 = S.fused_counters()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        S.smooth(b, x, "pgs", nu=1, k_l=k_l)
    e1.record()
    torch.cuda.synchronize()
    c = (S.fused_counters() - c0) / 10
    ms = e0.elapsed_time(e1) / 10
    G = int(os.environ.get("GRID", "296"))
    print(f"{cfg} margin {mg}: {ms:.3f} ms/apply; per CTA: polls {c[0]/G:.1f} ({c[1]/G/1e3:.1f} us), stage waits "
          f"{c[2]/G/1e3:.1f} us, readiness {c[3]/G/1e3:.1f} us, all units {c[4]/G/1e3:.1f} us, fences {c[5]/G:.1f}",
          flush=True)
