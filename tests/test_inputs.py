"""The seeded input generators (inputs/) produce matrices with the structure
SURVEY.md §8(d) and DESIGN.md §3 state (-m "not gpu")."""
import numpy as np
import pytest

import inputs


def test_nnz_closed_forms():
    L = inputs._L()
    # C1: 5-point N^2: 5N^2 - 4N
    assert inputs.config_matrix("C1").nnz == 20224
    # C2 / C4 / C5: 7-point N^3: 7N^3 - 6N^2
    assert L.gen_lap_nnz(128, 128, 128, 3, 0, 128 ** 3) == 14581760
    assert L.gen_cd_nnz(256, 256, 256, 0, 256 ** 3) == 117047296
    # C3: 27-point N^3: (3N-2)^3
    assert L.gen_var27_nnz(256, 256, 256, 0, 256 ** 3) == 449455096


@pytest.mark.parametrize("gen", ["lap", "var27", "cd"])
def test_mmatrix_structure(gen):
    A = {"lap": lambda: inputs.laplace(6, 5, 4), "var27": lambda: inputs.var27(6),
         "cd": lambda: inputs.convdiff(6, rcm=False)}[gen]()
    M = A.to_scipy().toarray()
    off = M - np.diag(np.diag(M))
    assert np.all(off <= 0)
    assert np.all(np.diag(M) > 0)
    assert np.all(np.diag(M) >= -off.sum(1) - 1e-9 * np.diag(M))
    # columns strictly ascending
    for i in range(A.nrows):
        c = A.col[A.rowptr[i]:A.rowptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    if gen in ("lap", "var27"):
        np.testing.assert_allclose(M, M.T, rtol=1e-15, atol=0)
    else:
        assert np.array_equal(M != 0, (M != 0).T) and not np.allclose(M, M.T)


def test_var27_interior_zero_rowsum_and_anisotropy():
    N = 6
    A = inputs.var27(N)
    M = A.to_scipy().toarray()
    i = 2 + N * (2 + N * 2)
    assert abs(M[i].sum()) < 1e-9 * M[i, i]
    # pure-z face coupling carries the factor 100 relative to x faces
    assert -M[i, i + N * N] > 20 * -M[i, i + 1] or -M[i, i + N * N] > 20 * -M[i, i - 1]


def test_partition_invariance():
    """Rows [r0, r1) of a generator equal the same rows of the global matrix."""
    G = inputs.laplace(4, 4, 8)
    S = inputs.weak_slab(4, 2, 1)
    assert S.row_begin == 64 and S.nrows == 64
    B = G.rows(64, 128)
    assert np.array_equal(S.rowptr, B.rowptr) and np.array_equal(S.col, B.col) and np.array_equal(S.val, B.val)
    u = inputs.uniform(0, 100)
    assert np.array_equal(inputs.uniform(0, 40, idx0=60), u[60:])


def test_rcm_valid_and_reduces_bandwidth():
    A = inputs.convdiff(8, rcm=False)
    order = inputs.rcm_order(A)
    assert np.array_equal(np.sort(order), np.arange(A.nrows))
    B = inputs.permute(A, order)
    M, P = A.to_scipy().toarray(), B.to_scipy().toarray()
    np.testing.assert_array_equal(P, M[np.ix_(order, order)])
    # 2-D 8x8: bandwidth of an RCM ordering is <= 8 + slack of a level
    A2 = inputs.laplace(8, 8, 1)
    B2 = inputs.permute(A2, inputs.rcm_order(A2))
    assert inputs.bandwidth(B2) <= 8


def test_uniform_int_exact():
    v = inputs.uniform_int(0, 10000, 20)
    assert np.all(v == np.round(v)) and v.min() >= -2 ** 20 and v.max() < 2 ** 20
