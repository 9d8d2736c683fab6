"""Where the coupled sweeps kernel (coupled.cu) spends its time on C3:
per sweep group, the producer's share in dependency waits / stage waits and
the consumers' share waiting for staged data (nsm_coupled_counters), at a
few throttle distances.  Usage: python tools/experiments/coupled_probe.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import bench
import inputs
import paper_2112_14681_b200 as nsm

A, offsets, kind, k_l, k_u, desc = bench.build_workload("C3", 0, 1)
if os.environ.get("NSM_VARIANT"):
    nsm.load(variant=os.environ["NSM_VARIANT"])
S = nsm.Smoother(A)
b = torch.from_numpy(inputs.uniform(inputs.SEED_B, A.nrows)).cuda()
x = torch.from_numpy(inputs.uniform(inputs.SEED_X0, A.nrows)).cuda()
for lag in [int(a) for a in (sys.argv[1:] or ["1", "150", "300", "600", "1200", "4000"])]:
    S.set_coupled(lag if lag > 0 else 1)
    for _ in range(3):
        S.smooth(b, x, "pgs", k_l=2)
    S.set_profile(True)
    S.profile()
    c0 = S.coupled_counters()
    for _ in range(10):
        S.smooth(b, x, "pgs", k_l=2)
    torch.cuda.synchronize()
    prof = S.profile()
    c = S.coupled_counters() - c0
    S.set_profile(False)
    ms_res = prof["residual"][0] / 10
    ms_sw = prof["sweep"][0] / 10
    out = [f"lag {lag}: residual {ms_res:.3f} ms, sweeps kernel {ms_sw:.3f} ms"]
    for g in range(2):
        tot = max(c[4 * g + 2], 1)
        out.append(f"  g{g}: producer dep-spin {c[4*g]/tot:.2f} fences {c[12+g]/tot:.2f} stage-wait {c[4*g+1]/tot:.2f} "
                   f"consumer data-wait {c[4*g+3]/tot:.2f} (cycles/CTA {tot/148/1e3:.0f}k)")
    print("\n".join(out), flush=True)
S.check()
