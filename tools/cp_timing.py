"""Set-up cost: host IKJ ILU(0) (nsm_ilu0) vs GPU Chow-Patel sweeps
(nsm_ilu0_fixed_point), wall time of the C-ABI calls incl. transfers, and the
ILU smoother quality with the approximate factors (C2 / C4)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_2112_14681_b200 as nsm

for cfg in sys.argv[1:] or ["C2", "C4"]:
    A = inputs.config_matrix(cfg)
    nsm.ilu0_fixed_point(A, 1)  # warm the device / module
    t0 = time.perf_counter(); host = nsm.ilu0(A); t_host = time.perf_counter() - t0
    b = torch.from_numpy(inputs.uniform(0, A.nrows)).cuda()
    res = {}
    for sw in [1, 2, 3, 5, 10]:
        t0 = time.perf_counter(); F = nsm.ilu0_fixed_point(A, sw); t_dev = time.perf_counter() - t0
        rel = float(np.linalg.norm(F - host) / np.linalg.norm(host))
        # smoother quality: ||b - A x|| after 3 ILU(2,2) applications from 0
        with nsm.Smoother(A, F) as S:
            x = torch.zeros_like(b)
            S.smooth(b, x, "ilu", nu=3, k_l=2, k_u=2, x_is_zero=True)
            r = torch.empty_like(b); S.residual(b, x, r)
            rr = float(torch.linalg.norm(r) / torch.linalg.norm(b))
        res[sw] = {"s": round(t_dev, 3), "factor_relerr": rel, "smoother_relres": rr}
    with nsm.Smoother(A, host) as S:
        x = torch.zeros_like(b)
        S.smooth(b, x, "ilu", nu=3, k_l=2, k_u=2, x_is_zero=True)
        r = torch.empty_like(b); S.residual(b, x, r)
        rr_exact = float(torch.linalg.norm(r) / torch.linalg.norm(b))
    print(json.dumps({"cfg": cfg, "n": A.nrows, "nnz": A.nnz, "host_ilu0_s": round(t_host, 3),
                      "exact_smoother_relres": rr_exact, "fixed_point": res}), flush=True)
