"""Pins of the oracle's ILUT(droptol, lfil) and Ruiz scaling (Alg. 2,
P:L1020-1045; NEXT-3) (-m "not gpu"), and parity of the product's host
ILUT / Ruiz setup (nsm_ilut, nsm_ruiz) with the oracle."""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

import inputs
import oracle
import paper_2112_14681_b200 as nsm
from oracle import ilut as oilut


def dense_factors(n, F):
    W = sp.csr_matrix((F[2], F[1], F[0]), shape=(n, n)).toarray()
    return np.eye(n) + np.tril(W, -1), np.triu(W)


def dd_random(n, seed, density=0.4):
    rng = np.random.default_rng(seed)
    M = rng.uniform(-1, 1, (n, n)) * (rng.uniform(0, 1, (n, n)) < density)
    M += np.diag(np.abs(M).sum(1) + 1.0)
    return sp.csr_matrix(M)


def test_ilut_no_dropping_is_exact_lu():
    """droptol = 0, lfil >= n: the complete (unpivoted) LU, L U = A."""
    A = dd_random(12, 1)
    F = oilut.ilut(A, 0.0, 12)
    L, U = dense_factors(12, F)
    np.testing.assert_allclose(L @ U, A.toarray(), rtol=1e-13, atol=1e-13)


def test_ilut_diagonal_and_caps():
    A = sp.diags(np.arange(1.0, 7.0)).tocsr()
    F = oilut.ilut(A, 0.1, 2)
    L, U = dense_factors(6, F)
    assert np.array_equal(L, np.eye(6)) and np.array_equal(U, A.toarray())
    B = inputs.convdiff(6).to_scipy()
    lfil = 3
    rp, col, val = oilut.ilut(B, 1e-3, lfil)
    rows = np.repeat(np.arange(B.shape[0]), np.diff(rp))
    assert np.all(np.bincount(rows[col < rows], minlength=B.shape[0]) <= lfil)
    assert np.all(np.bincount(rows[col > rows], minlength=B.shape[0]) <= lfil)


def test_ilut_drop_monotone_and_ilu0_relation():
    B = inputs.convdiff(6).to_scipy()
    sizes = [len(oilut.ilut(B, t, 50)[1]) for t in (0.0, 1e-4, 1e-2, 1e-1)]
    assert all(a >= b for a, b in zip(sizes, sizes[1:]))
    # without dropping ILUT keeps every entry of A's pattern (plus fill)
    rp, col, _ = oilut.ilut(B, 0.0, 10 ** 6)
    full = sp.csr_matrix((np.ones(len(col)), col, rp), shape=B.shape).toarray() != 0
    assert np.all(full[B.toarray() != 0])


def test_ruiz_properties():
    B = inputs.convdiff(6).to_scipy()
    F = oilut.ilut(B, 1e-3, 5)
    v, sr, sc = oilut.ruiz_upper(*F, max_iters=5)
    n = B.shape[0]
    rows = np.repeat(np.arange(n), np.diff(F[0]))
    up = F[1] >= rows
    diag = F[1] == rows
    assert np.all(v[diag] == 1.0)                       # exact unit diagonal
    U = sp.csr_matrix((np.where(up, F[2], 0.0), F[1], F[0]), shape=(n, n)).toarray()
    Ut = sp.csr_matrix((np.where(up, v, 0.0), F[1], F[0]), shape=(n, n)).toarray()
    np.testing.assert_allclose(np.diag(sr) @ Ut @ np.diag(sc), U, rtol=1e-13, atol=1e-13)
    assert np.max(np.abs(Ut - np.diag(np.diag(Ut)))) <= 1.0 + 1e-12
    assert np.array_equal(v[~up], F[2][~up])            # L_s unchanged


def test_ilu_ruiz_apply_limits():
    """k >= n-1 on both factors: the direct ILUT solve x + U^-1 L^-1 (b - A x)."""
    B = inputs.convdiff(4).to_scipy()
    n = B.shape[0]
    F = oilut.ilut(B, 1e-2, 4)
    v, sr, sc = oilut.ruiz_upper(*F)
    L, U = dense_factors(n, F)
    b, x0 = inputs.uniform(0, n), inputs.uniform(1, n)
    r = b - B @ x0
    want = x0 + sla.solve_triangular(U, sla.solve_triangular(L, r, lower=True, unit_diagonal=True), lower=False)
    got = oilut.ilu_ruiz_apply(inputs.CSR.from_scipy(B), (F[0], F[1], v), sr, sc, b, x0, n - 1, n - 1)
    np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("which", ["convdiff", "var27", "random"])
@pytest.mark.parametrize("droptol,lfil", [(0.0, 1000), (1e-3, 5), (1e-2, 2)])
def test_product_ilut_ruiz_match_oracle(which, droptol, lfil):
    A = {"convdiff": lambda: inputs.convdiff(6), "var27": lambda: inputs.var27(5),
         "random": lambda: inputs.CSR.from_scipy(dd_random(40, 3))}[which]()
    Fo = oilut.ilut(A.to_scipy(), droptol, lfil)
    Fp = nsm.ilut(A, droptol, lfil)
    assert np.array_equal(Fp.rowptr, Fo[0]) and np.array_equal(Fp.col, Fo[1])
    assert np.array_equal(Fp.val, Fo[2])
    vo, sro, sco = oilut.ruiz_upper(*Fo)
    Fr, srp, scp = nsm.ruiz(Fp)
    assert np.array_equal(Fr.val, vo) and np.array_equal(srp, sro) and np.array_equal(scp, sco)
