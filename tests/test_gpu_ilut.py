"""ILUT(droptol, lfil) + Ruiz smoothing on the GPU (-m gpu; Algorithm 2 in
full) against the oracle's
ilu_ruiz_apply / ilu_apply on the same host factors — bitwise."""
import numpy as np
import pytest
import torch

import inputs
import oracle
import paper_2112_14681_b200 as nsm
from oracle import ilut as oilut

pytestmark = pytest.mark.gpu

MATS = {
    "convdiff12": lambda: inputs.convdiff(12),
    "var27_10": lambda: inputs.var27(10),
    "laplace7_20": lambda: inputs.laplace(20, 20, 20),
}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


@pytest.mark.parametrize("mat", list(MATS))
@pytest.mark.parametrize("kl,ku", [(0, 0), (1, 0), (0, 2), (2, 2), (3, 5)])
@pytest.mark.parametrize("fresh", [False, True])
def test_ruiz_ilu_smooth_bitwise(mat, kl, ku, fresh):
    A = MATS[mat]()
    F = nsm.ilut(A, 1e-3, 6)
    Fr, sr, sc = nsm.ruiz(F)
    n = A.nrows
    b, x0 = inputs.uniform(0, n), inputs.uniform(1, n)
    want = oilut.ilu_ruiz_apply(A, (Fr.rowptr, Fr.col, Fr.val), sr, sc, b, x0, kl, ku, nu=2, x_is_zero=fresh)
    S = nsm.Smoother(A, Fr)
    try:
        S.set_ruiz(sr, sc)
        for mode in ("fused", "fusedw1", "pipelined", "plain"):
            S.set_pipeline(mode != "plain")
            S.set_fused(1 if mode.startswith("fused") else 0)
            S.set_fused_window(1 if mode == "fusedw1" else 0)
            x = dev(np.full(n, np.nan) if fresh else x0)
            S.smooth(dev(b), x, "ilu", 2, kl, ku, x_is_zero=fresh)
            got = x.cpu().numpy()
            assert np.array_equal(got, want), (mat, kl, ku, fresh, mode, np.max(np.abs(got - want)))
        S.check()
    finally:
        S.close()


@pytest.mark.parametrize("mat", list(MATS))
def test_ilut_factors_unscaled_bitwise(mat):
    """ILUT factors through the ordinary ILU path (no Ruiz) vs oracle.ilu_apply."""
    A = MATS[mat]()
    F = nsm.ilut(A, 1e-2, 4)
    n = A.nrows
    b, x0 = inputs.uniform(0, n), inputs.uniform(1, n)
    want = oracle.ilu_apply(A, (F.rowptr, F.col, F.val), b, x0, 3, 3, nu=1)
    S = nsm.Smoother(A, F)
    try:
        for fused in (1, 0):
            S.set_fused(fused)
            x = dev(x0)
            S.smooth(dev(b), x, "ilu", 1, 3, 3)
            assert np.array_equal(x.cpu().numpy(), want), f"fused={fused}"
    finally:
        S.close()
