"""Pins of the oracle's Chow-Patel fixed-point ILU(0) (oracle.ilu0_fixed_point,
reading R19; the set-up algorithm the paper names as future work,
P:L1578-1582) against what does not depend on it:

* the textbook ILU(0) (Saad's IKJ variant, oracle.ilu0, itself pinned by the
  defining property (LU)_ij = a_ij on the pattern in test_oracle_pins.py):
  the fixed point of the sweeps IS that factorisation, and because every
  entry is formed with the same subtractions in the same ascending-k order,
  the converged sweeps reproduce it bit for bit;
* the dependency structure of synchronous sweeps, computed here by a plain
  graph recursion: after m sweeps exactly the entries whose inputs settle
  within m - 1 sweeps are final (one "level" per sweep);
* the 1-D closed form u_ii = (i+2)/(i+1), l_{i+1,i} = -(i+1)/(i+2): one more
  entry of the chain becomes exact per sweep.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import inputs
import oracle


def tridiag(n):
    return inputs.CSR.from_scipy(sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]))


def random_sparse_dd(n, seed, per_row=4):
    rng = np.random.default_rng(seed)
    M = sp.lil_matrix((n, n))
    for i in range(n):
        for j in rng.choice(n, size=per_row, replace=False):
            if j != i:
                M[i, j] = rng.uniform(-1, 1)
    M = M.tocsr()
    M = M + sp.diags(np.abs(M).sum(1).A1 + 1.0)
    return inputs.CSR.from_scipy(M)


MATS = {
    "tridiag": lambda: tridiag(12),
    "lap2d": lambda: inputs.laplace(7, 6, 1),
    "lap3d": lambda: inputs.laplace(4, 4, 3),
    "cd_rcm": lambda: inputs.convdiff(5),
    "random": lambda: random_sparse_dd(40, 3),
}


def settle_level(A):
    """Sweep after which each entry (CSR position) is final, from the
    dependency graph of the fixed-point equations: entry (i,j) reads (i,k) and
    (k,j) for k < min(i,j) in the pattern, and an L entry also u_jj.  Level 0
    = the initial guess is already final (no k-terms; for an L entry also
    u_jj = a_jj)."""
    n, rp, ci = A.nrows, A.rowptr, A.col
    pos = {}
    for i in range(n):
        for p in range(rp[i], rp[i + 1]):
            pos[(i, int(ci[p]))] = p
    level = {}

    def lev(i, j):
        if (i, j) in level:
            return level[(i, j)]
        deps = []
        for k in range(min(i, j)):
            if (i, k) in pos and (k, j) in pos:
                deps += [(i, k), (k, j)]
        if j < i:
            if not deps and lev(j, j) == 0:
                level[(i, j)] = 0
                return 0
            deps.append((j, j))
        level[(i, j)] = 0 if not deps else 1 + max(lev(a, b) for a, b in deps)
        return level[(i, j)]

    return np.array([lev(i, int(ci[p])) for i in range(n) for p in range(rp[i], rp[i + 1])])


@pytest.mark.parametrize("name", list(MATS))
def test_converges_to_ikj_ilu0_bitwise(name):
    A = MATS[name]()
    want = oracle.ilu0(A)[2]
    lev = settle_level(A)
    got = oracle.ilu0_fixed_point(A, int(lev.max()))[2]
    assert np.array_equal(got, want)
    # the fixed point is a fixed point: one more sweep changes nothing
    assert np.array_equal(oracle.ilu0_fixed_point(A, int(lev.max()) + 3)[2], want)


@pytest.mark.parametrize("name", list(MATS))
def test_one_level_settles_per_sweep(name):
    """Synchronous sweeps: after m sweeps the entries of level <= m are final;
    before the last level, some entry is not (the iteration did not finish
    early, i.e. updates really use the previous sweep only)."""
    A = MATS[name]()
    want = oracle.ilu0(A)[2]
    lev = settle_level(A)
    for m in range(int(lev.max()) + 1):
        got = oracle.ilu0_fixed_point(A, m)[2]
        done = lev <= m
        assert np.array_equal(got[done], want[done]), f"sweep {m}: a level-<=m entry is not final"
        if m < lev.max():
            assert np.any(got[~done] != want[~done]), f"sweep {m}: converged earlier than the levels allow"


def test_1d_closed_form_one_entry_per_sweep():
    """Tridiagonal (-1, 2, -1): u_00 = 2 and l_10 = -1/2 are exact from the
    initial guess; then the chain u_11 <- l_21 <- u_22 <- ... settles one
    entry per sweep: u_ii = (i+2)/(i+1) after sweep 2i - 1, l_{i+1,i} =
    -(i+1)/(i+2) after sweep 2i."""
    n = 7
    A = tridiag(n)
    for m in range(0, 2 * n):
        rp, ci, w = oracle.ilu0_fixed_point(A, m)
        F = sp.csr_matrix((w, ci, rp), shape=(n, n)).toarray()
        for i in range(n):
            u_exact = abs(F[i, i] - (i + 2) / (i + 1)) < 1e-15
            assert u_exact == (m >= max(0, 2 * i - 1)), (m, i, F[i, i])
            if i + 1 < n:
                l_exact = abs(F[i + 1, i] + (i + 1) / (i + 2)) < 1e-15
                assert l_exact == (m >= 2 * i), (m, i, F[i + 1, i])
                assert F[i, i + 1] == -1.0


def test_initial_guess_and_zero_diagonal():
    A = MATS["lap2d"]()
    rp, ci, w = oracle.ilu0_fixed_point(A, 0)
    M = sp.csr_matrix((A.val, A.col, A.rowptr), shape=(A.nrows, A.nrows))
    d = M.diagonal()
    rows = np.repeat(np.arange(A.nrows), np.diff(rp))
    want = np.where(ci < rows, A.val / d[ci], A.val)
    assert np.array_equal(w, want)
    Z = inputs.CSR.from_scipy(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 1.0]])))
    with pytest.raises(oracle.OracleError):
        oracle.ilu0_fixed_point(Z, 2)
