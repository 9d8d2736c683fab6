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


# ------------------------------------------- departure from normality ---
# P:L847-855 (Henrici), Theorem 3, Definition 2 / Theorem 4
# (P:L1234-1265), the Ruiz early termination.
def unit_upper_with_strict_norm(n, target, seed=0):
    """A unit upper-triangular CSR of size n whose strictly-upper part has
    Frobenius norm `target` (entries on the first superdiagonal)."""
    rng = np.random.default_rng(seed)
    m = min(n - 1, 400)
    w = rng.uniform(0.5, 1.0, m)
    w *= target / np.linalg.norm(w)
    U = sp.eye(n, format="lil")
    for i in range(m):
        U[i, i + 1] = w[i]
    U = U.tocsr()
    U.sort_indices()
    return U


def read_table5():
    import os
    rows, n = [], None
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "table5_depU.txt")):
        t = line.split()
        if not t or t[0].startswith("#"):
            continue
        if t[0] == "n":
            n = int(t[1])
        else:
            rows.append((int(t[0]), float(t[1]), float(t[2]), float(t[3])))
    return n, rows


def test_table5_theorem3_bound_row():
    """Table 5's bound row follows from its dep(U)-after row and N = 14186
    when Theorem 3's nu is evaluated as ||U||_F = sqrt(N + dep^2) of the
    unit-diagonal scaled U (reading R20); with the theorem's nu = ||U_s||_F
    the bound is smaller (still a bound).  Checked through dep_info on unit
    upper-triangular matrices with exactly those norms, oracle and product."""
    n, rows = read_table5()
    for fill, _, dep_after, bound in rows:
        U = unit_upper_with_strict_norm(n, dep_after, seed=fill)
        for info in (oilut.dep_info(U.indptr, U.indices, U.data, True),
                     nsm.dep(inputs.CSR.from_scipy(U), upper=True)):
            assert abs(info["dep"] - dep_after) < 1e-9
            assert round(info["bound_table5"], 2) == bound, (fill, info["bound_table5"], bound)
            assert info["dep"] <= info["bound_thm3"] < info["bound_table5"]


def test_theorem3_worked_example():
    """n = 1e9 and ||U_s|| = 0.8 give dep(U) <= 225."""
    sq = np.sqrt(1e9)
    assert np.sqrt((2 * sq + 0.8) * 0.8) <= 225.0 < np.sqrt((2 * sq + 0.8) * 0.8) + 0.1
    U = unit_upper_with_strict_norm(50, 0.8)
    info = oilut.dep_info(U.indptr, U.indices, U.data, True)
    assert abs(info["bound_thm3"] - np.sqrt((2 * np.sqrt(50) + 0.8) * 0.8)) < 1e-12


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_dep_triangular_equals_definition(seed):
    """Henrici's definition via eigenvalues (dep_dense) = the strictly-upper
    Frobenius norm (dep_upper) on triangular matrices; 0 on normal matrices;
    |a| on [[1, a], [0, 1]]."""
    rng = np.random.default_rng(seed)
    n = 9
    T = np.triu(rng.uniform(-1, 1, (n, n)) * (rng.uniform(0, 1, (n, n)) < 0.6)) + np.diag(rng.uniform(1, 2, n))
    S = sp.csr_matrix(T)
    S.sort_indices()
    assert abs(oilut.dep_dense(T) - oilut.dep_upper(S.indptr, S.indices, S.data)) < 1e-12
    assert abs(oilut.dep_dense(T) - np.linalg.norm(np.triu(T, 1))) < 1e-12
    M = rng.uniform(-1, 1, (n, n))
    assert oilut.dep_dense(M + M.T) < 1e-6                  # symmetric: normal
    Q, _ = np.linalg.qr(M)
    assert oilut.dep_dense(Q) < 1e-6                        # orthogonal: normal
    assert abs(oilut.dep_dense(np.array([[1.0, 3.0], [0.0, 1.0]])) - 3.0) < 1e-12


@pytest.mark.parametrize("which", ["convdiff", "random"])
def test_dep_bounds_hold_after_ruiz(which):
    """Theorems 3 and 4 on ILUT + Ruiz factors (unit-diagonal U~): dep <=
    sqrt((2 sqrt(n) + nu) nu) and dep <= sqrt(n) (1 + delta); the product's
    diagnostics equal the oracle's."""
    A = {"convdiff": lambda: inputs.convdiff(6).to_scipy(), "random": lambda: dd_random(60, 5, 0.2)}[which]()
    rp, col, val = oilut.ilut(A, 1e-3, 5)
    v, _, _ = oilut.ruiz_upper(rp, col, val)
    F = nsm.FactorCSR(A.shape[0], rp, col, v)
    for upper in (True, False):
        o = oilut.dep_info(rp, col, v, upper)
        p = nsm.dep(F, upper=upper)
        assert o["dep"] <= o["bound_thm3"] + 1e-12 and o["dep"] <= o["bound_thm4"] + 1e-12
        for k in o:
            assert p[k] == o[k] if k in ("n", "dep", "fro", "fro_strict") else abs(p[k] - o[k]) <= 1e-12 * max(1, abs(o[k])), k
        dense = sp.csr_matrix((v, col, rp), shape=A.shape).toarray()
        T = np.triu(dense) if upper else np.eye(A.shape[0]) + np.tril(dense, -1)
        assert abs(o["dep"] - oilut.dep_dense(T)) < 1e-9 * max(1.0, o["dep"])


def test_ruiz_early_termination():
    """nsm_ruiz_dep / ruiz_upper_dep: the dep history of the scaled U, rounds
    stop once it is below the tolerance, bit-for-bit equal between product and
    oracle; tolerance 0 is plain Ruiz."""
    A = inputs.convdiff(6).to_scipy()
    F = oilut.ilut(A, 1e-3, 5)
    v0, sr0, sc0, it0, h0 = oilut.ruiz_upper_dep(*F, max_iters=5, dep_tol=0.0)
    assert it0 == 5 and len(h0) == 6
    assert np.array_equal(v0, oilut.ruiz_upper(*F)[0])
    Fc = nsm.FactorCSR(A.shape[0], *F)
    Fr, sr, sc, (itp, hp) = nsm.ruiz(Fc, 5, history=True)
    assert itp == 5 and np.array_equal(hp, np.array(h0)) and np.array_equal(Fr.val, v0)
    tol = h0[1] * (1 + 1e-9) if h0[1] < h0[0] else h0[0]
    v1, sr1, sc1, it1, h1 = oilut.ruiz_upper_dep(*F, max_iters=5, dep_tol=tol)
    Fr1, sr1p, sc1p, (it1p, h1p) = nsm.ruiz(Fc, 5, dep_tol=tol)
    assert it1 == it1p and it1 <= 2 and np.array_equal(Fr1.val, v1) and np.array_equal(sr1p, sr1)
    assert h1[-1] < tol
    rows = np.repeat(np.arange(A.shape[0]), np.diff(F[0]))
    assert np.all(v1[F[1] == rows] == 1.0)                   # still an exact unit diagonal
