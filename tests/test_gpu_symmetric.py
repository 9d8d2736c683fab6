"""Symmetric residual (transpose.cu + stream.cu k_residual_tma_ws, DESIGN.md
§6): when A is bitwise symmetric the windowed residual reads U = L^T from L's
values through U's transpose map.  The map exists exactly when every value it
produces equals U's stored one; results are bit-identical to the oracle and to
the streaming-U kernels (-m gpu)."""
import numpy as np
import pytest
import torch

import bench
import inputs
import oracle
import paper_2112_14681_b200 as nsm

pytestmark = pytest.mark.gpu


def dev(v):
    return torch.from_numpy(np.ascontiguousarray(v)).cuda()


def host(t):
    return t.cpu().numpy()


def perturbed(A, i, j, ulps=1):
    """A with the stored value of (i, j) moved by `ulps` units in the last place."""
    val = A.val.copy()
    p = A.rowptr[i] + int(np.flatnonzero(A.col[A.rowptr[i]:A.rowptr[i + 1]] == j)[0])
    val[p] = np.nextafter(val[p], np.inf) if ulps > 0 else np.nextafter(val[p], -np.inf)
    return inputs.CSR(A.nrows, A.ncols, A.rowptr, A.col, val, A.row_begin)


MATS = {
    "var27_40": lambda: inputs.var27(40),                          # 64,000 rows: 250 tiles
    "var27_ragged": lambda: inputs.var27_grid(130, 20, 6),         # 15,600 rows: a ragged last tile
    "var27_lines": lambda: inputs.var27_grid(256, 8, 10),          # C3's structure: a tile = one grid line
}


@pytest.mark.parametrize("name", list(MATS))
def test_symmetric_residual_parity(name):
    A = MATS[name]()
    b, x = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    with nsm.Smoother(A) as S:
        assert S.layout()["Ut"], name                               # the map exists
        want_r = oracle.residual(A, b, x)
        want_ax = oracle.spmv(A, x)
        for sym in (True, False, True):
            S.set_symmetric(sym)
            assert np.array_equal(host(S.residual(dev(b), dev(x))), want_r), (name, sym)
            assert np.array_equal(host(S.spmv(dev(x))), want_ax), (name, sym)
        for k, nu, xz in ((0, 1, False), (1, 1, False), (2, 1, False), (3, 2, False), (2, 2, True)):
            x0 = np.zeros(A.nrows) if xz else x
            want = oracle.pgs_apply(A, b, x0, k, nu=nu, x_is_zero=xz)
            xd = dev(x0)
            S.smooth(dev(b), xd, "pgs", nu=nu, k_l=k, x_is_zero=xz)
            assert np.array_equal(host(xd), want), (name, k, nu, xz)


@pytest.mark.parametrize("where", ["first_row", "interior", "last_row"])
def test_one_ulp_asymmetry_disables_the_map(where):
    """A single U value one ulp off its mirror (or one L value): no map, and
    the residual (streaming U) is still bit-identical to the oracle."""
    A = inputs.var27_grid(256, 8, 6)     # offset-aligned, 256-row lines
    n = A.nrows
    i = {"first_row": 0, "interior": n // 2, "last_row": n - 2}[where]
    j = i + 1                                                    # (i, i + 1) is in U
    B = perturbed(A, i, j) if where != "interior" else perturbed(A, j, i, -1)   # interior: perturb the L side
    assert not bench.symmetric_local(B)
    b, x = inputs.uniform(0, n), inputs.uniform(1, n)
    with nsm.Smoother(B) as S:
        assert S.layout()["L"] and S.layout()["U"] and not S.layout()["Ut"]
        assert np.array_equal(host(S.residual(dev(b), dev(x))), oracle.residual(B, b, x))


def test_signed_zero_asymmetry_disables_the_map():
    """+0.0 against -0.0 stored at mirrored positions is not bitwise symmetric."""
    A = inputs.var27_grid(64, 12, 10)
    val = A.val.copy()
    i = 300
    p = A.rowptr[i] + int(np.flatnonzero(A.col[A.rowptr[i]:A.rowptr[i + 1]] == i + 1)[0])
    q = A.rowptr[i + 1] + int(np.flatnonzero(A.col[A.rowptr[i + 1]:A.rowptr[i + 2]] == i)[0])
    val[p], val[q] = 0.0, -0.0
    B = inputs.CSR(A.nrows, A.ncols, A.rowptr, A.col, val)
    with nsm.Smoother(B) as S:
        assert not S.layout()["Ut"]
        b, x = inputs.uniform(0, B.nrows), inputs.uniform(1, B.nrows)
        assert np.array_equal(host(S.residual(dev(b), dev(x))), oracle.residual(B, b, x))


def test_nonsymmetric_and_short_rows_have_no_map():
    for A in (inputs.convdiff(12), inputs.laplace(64, 16, 8), inputs.var27(9)):
        with nsm.Smoother(A) as S:
            assert not S.layout()["Ut"]
            assert S.layout()["Ut"] == bench.aligned_parts(A)["Ut"]


def test_ilu_residual_uses_the_map_with_factors():
    """The ILU application's residual on a symmetric A (factors nonsymmetric
    in general) also reads U from L; the whole application stays exact."""
    A = inputs.var27_grid(64, 12, 10)
    F = oracle.ilu0(A)[2]
    b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    want = oracle.ilu_apply(A, (A.rowptr, A.col, F), b, x0, 2, 2)
    with nsm.Smoother(A, F) as S:
        assert S.layout()["Ut"]
        x = dev(x0)
        S.smooth(dev(b), x, "ilu", nu=1, k_l=2, k_u=2)
        assert np.array_equal(host(x), want)


@pytest.mark.slow
def test_symmetric_residual_full_size_c3():
    """C3 at full size (16.7 M rows): the map exists and the residual through
    it equals the streaming-U residual bit for bit (both equal the oracle in
    test_gpu_parity's full-size case); sampled rows against the oracle's
    row-by-row definition."""
    A = inputs.config_matrix("C3")
    b, x = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    with nsm.Smoother(A) as S:
        assert S.layout()["Ut"]
        r_sym = host(S.residual(dev(b), dev(x)))
        S.set_symmetric(False)
        r_str = host(S.residual(dev(b), dev(x)))
    assert np.array_equal(r_sym, r_str)
    rng = np.random.default_rng(7)
    for i in np.concatenate([[0, 1, A.nrows - 1], rng.integers(0, A.nrows, 64)]):
        sub = A.rows(int(i), int(i) + 1)
        assert r_sym[i] == oracle.residual(sub, b[i:i + 1], x)[0], i
