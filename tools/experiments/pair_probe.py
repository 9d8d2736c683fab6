"""Paired sweeps (pair.cu; libnsm_exp.so with NSM_CP_PAIR=1): bit-identical to the
oracle / per-pass path on 27-point matrices (ragged, few tiles, C3 full size),
then C3 timing of per-pass vs coupled vs paired (library event pairs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import bench, inputs, oracle
import paper_2112_14681_b200 as nsm

nsm.load(variant="exp")
os.environ["NSM_CP_PAIR"] = "1"
for name, A in [("var27_40", inputs.var27(40)), ("ragged", inputs.var27_grid(130, 20, 6)),
                ("48tiles", inputs.var27_grid(64, 16, 12))]:
    b0, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    want = oracle.pgs_apply(A, b0, x0, 2, nu=2)
    with nsm.Smoother(A) as S:
        S.set_coupled(1)
        S.set_profile(True); S.profile()
        x = torch.from_numpy(x0.copy()).cuda()
        S.smooth(torch.from_numpy(b0).cuda(), x, "pgs", nu=2, k_l=2)
        got = x.cpu().numpy()
        nsweep = S.profile()["sweep"][1]
        S.check()
        print(name, "bitwise" if np.array_equal(got, want) else f"DIFF {np.abs(got - want).max():.3e}", "sweep launches", nsweep, flush=True)
A, offsets, kind, k_l, k_u, desc = bench.build_workload("C3", 0, 1)
b = torch.from_numpy(inputs.uniform(inputs.SEED_B, A.nrows)).cuda()
x0 = torch.from_numpy(inputs.uniform(inputs.SEED_X0, A.nrows)).cuda()
S = nsm.Smoother(A)
ref = None
for mode in ["perpass", "pair", "perpass", "pair"]:
    S.set_coupled(0 if mode == "perpass" else 1)
    x = x0.clone()
    S.smooth(b, x, "pgs", k_l=2)
    torch.cuda.synchronize()
    if ref is None:
        ref = x.cpu().numpy()
    else:
        assert np.array_equal(x.cpu().numpy(), ref), mode
    for _ in range(3):
        S.smooth(b, x, "pgs", k_l=2)
    S.set_profile(True); S.profile()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for e0, e1 in ev:
        e0.record(); S.smooth(b, x, "pgs", k_l=2); e1.record()
    torch.cuda.synchronize()
    pr = S.profile(); S.set_profile(False)
    ms = np.mean([e0.elapsed_time(e1) for e0, e1 in ev])
    print(f"C3 {mode}: {ms:.3f} ms per application (with event pairs), residual {pr['residual'][0]/20:.3f}, sweeps kernel(s) {pr['sweep'][0]/20:.3f} ms", flush=True)
S.check()
print("C3 full size: pair == per-pass bitwise")
