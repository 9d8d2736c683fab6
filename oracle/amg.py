"""CPU ORACLE — classical AMG hierarchy, V-cycle and right-preconditioned
GMRES for the iteration-count parity driver (north_star: "iteration counts
must be identical in a GMRES + one-V-cycle driver").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy/scipy, fp64,
one function per step in the paper's order:

  strength      |a_ij| >= theta max_{k != i} |a_ik|
  pmis          parallel maximal independent set, Luby-style
  bamg_direct   w_ij = -(a_ij + beta_i / n_Cs) / (a_ii + sum_{N_i^w} a_ik)
                                                                
  galerkin      A_c = P^T A P
  vcycle        pre-smooth, residual, restrict, recurse, prolong, post-smooth,
                coarse direct solve
  gmres         right-preconditioned MGS-GMRES with Givens rotations
                (the classical form of Alg. 1's solver; the
                low-synchronisation variant is NEXT-1, out of scope)

Readings: R11 stopping rule relres < tol; R13 BAMG-direct
sets: beta_i sums the strong F-neighbours and the weak C-neighbours, the
denominator the weak F-neighbours (the only assignment that interpolates
constants exactly for zero-row-sum rows, the stated purpose of f = 1); R14
PMIS measure = number of points strongly influenced + a random number in
[0, 1) that is passed in (drawn by inputs/, not by the oracle); F-points with
no strong C-neighbour get an empty interpolation row.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp


def strength(A: sp.csr_matrix, theta: float = 0.25) -> sp.csr_matrix:
    """S_ij = 1 iff j != i and |a_ij| >= theta * max_{k != i} |a_ik|."""
    A = sp.csr_matrix(A)
    n = A.shape[0]
    rows, cols, vals = [], [], []
    for i in range(n):
        lo, hi = A.indptr[i], A.indptr[i + 1]
        c = A.indices[lo:hi]
        a = np.abs(A.data[lo:hi])
        off = c != i
        if not np.any(off):
            continue
        m = a[off].max()
        keep = off & (a >= theta * m) & (m > 0)
        rows += [i] * int(keep.sum())
        cols += list(c[keep])
    return sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(n, n))


def pmis(S: sp.csr_matrix, rand: np.ndarray) -> np.ndarray:
    """PMIS C/F splitting (De Sterck et al., Luby's algorithm).
    Returns cf (1 = C, 0 = F).  measure_i = |{j : j strongly depends on i}| +
    rand_i.  Points influencing nobody become F; then repeatedly every
    undecided point whose measure beats all undecided neighbours in the
    symmetrised strong graph becomes C, and undecided points strongly
    depending on a new C point become F."""
    n = S.shape[0]
    ST = S.T.tocsr()
    meas = np.asarray(ST.sum(axis=1)).ravel() + rand
    G = (S + ST).tocsr()
    state = np.full(n, -1)  # -1 undecided, 0 F, 1 C
    state[np.asarray(ST.sum(axis=1)).ravel() == 0] = 0
    while np.any(state < 0):
        und = state < 0
        newc = []
        for i in np.nonzero(und)[0]:
            nb = G.indices[G.indptr[i]:G.indptr[i + 1]]
            nb = nb[und[nb]]
            if np.all(meas[i] > meas[nb]):
                newc.append(i)
        if not newc:  # ties cannot happen with distinct random parts; guard anyway
            newc = [int(np.nonzero(und)[0][np.argmax(meas[und])])]
        state[newc] = 1
        isc = np.zeros(n, dtype=bool)
        isc[newc] = True
        for i in np.nonzero(state < 0)[0]:
            deps = S.indices[S.indptr[i]:S.indptr[i + 1]]
            if np.any(isc[deps]):
                state[i] = 0
    return state


def bamg_direct(A: sp.csr_matrix, S: sp.csr_matrix, cf: np.ndarray) -> sp.csr_matrix:
    """BAMG-direct interpolation for f = 1, reading R13."""
    A = sp.csr_matrix(A)
    n = A.shape[0]
    cidx = -np.ones(n, dtype=np.int64)
    cidx[cf == 1] = np.arange(int((cf == 1).sum()))
    rows, cols, vals = [], [], []
    for i in range(n):
        if cf[i] == 1:
            rows.append(i)
            cols.append(cidx[i])
            vals.append(1.0)
            continue
        lo, hi = A.indptr[i], A.indptr[i + 1]
        strong = set(S.indices[S.indptr[i]:S.indptr[i + 1]].tolist())
        aii = 0.0
        cs, acs = [], []
        beta = 0.0
        den_w = 0.0
        for p in range(lo, hi):
            j, a = A.indices[p], A.data[p]
            if j == i:
                aii = a
            elif j in strong and cf[j] == 1:
                cs.append(j)
                acs.append(a)
            elif j in strong:          # strong F-neighbour
                beta += a
            elif cf[j] == 1:           # weak C-neighbour
                beta += a
            else:                      # weak F-neighbour
                den_w += a
        if not cs:
            continue                   # F-point without strong C-neighbour: empty row
        den = aii + den_w
        for j, a in zip(cs, acs):
            rows.append(i)
            cols.append(cidx[j])
            vals.append(-(a + beta / len(cs)) / den)
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, int((cf == 1).sum())))


def galerkin(A, P):
    """A_c = P^T A P, R = P^T."""
    Ac = (P.T @ (A @ P)).tocsr()
    Ac.sum_duplicates()
    Ac.sort_indices()
    return Ac


def hierarchy(A, rand_fn, theta: float = 0.25, max_levels: int = 25, min_coarse: int = 200):
    """[(A_0, P_1), (A_1, P_2), ..., (A_m, None)] — stops at <= min_coarse rows,
    max_levels, or when coarsening stagnates.  rand_fn(level, n) supplies the
    PMIS random numbers (from inputs/)."""
    A = sp.csr_matrix(A)
    A.sort_indices()
    levels = []
    for lev in range(max_levels):
        n = A.shape[0]
        if n <= min_coarse or lev == max_levels - 1:
            levels.append((A, None))
            break
        S = strength(A, theta)
        cf = pmis(S, rand_fn(lev, n))
        nc = int(cf.sum())
        if nc == 0 or nc >= n:
            levels.append((A, None))
            break
        P = bamg_direct(A, S, cf)
        levels.append((A, P))
        A = galerkin(A, P)
    return levels


def vcycle(levels, smooth, b, lev: int = 0, lu=None):
    """One V(1,1) cycle from x = 0.  smooth(lev, A,
    b, x, x_is_zero) returns the smoothed x.  lu: cached dense LU of the
    coarsest matrix."""
    A, P = levels[lev]
    if P is None:
        return sla.lu_solve(lu, b)
    x = smooth(lev, A, b, np.zeros(A.shape[0]), True)         # pre-smoothing
    r = b - A @ x
    xc = vcycle(levels, smooth, P.T @ r, lev + 1, lu)         # restrict, recurse
    x = x + P @ xc                                            # prolong
    return smooth(lev, A, b, x, False)                        # post-smoothing


def coarse_lu(levels):
    return sla.lu_factor(levels[-1][0].toarray())


def gmres(A, b, precond, tol: float = 1e-5, maxit: int = 200):
    """Right-preconditioned MGS-GMRES, x0 = 0, no restart, Givens QR; stops
    when the implicit relative residual |g_{k+1}| / ||b|| < tol (R11).
    Returns (x, iterations, history of implicit relres)."""
    n = len(b)
    beta = np.linalg.norm(b)
    V = np.zeros((maxit + 1, n))
    Z = np.zeros((maxit, n))
    H = np.zeros((maxit + 1, maxit))
    cs, sn = np.zeros(maxit), np.zeros(maxit)
    g = np.zeros(maxit + 1)
    g[0] = beta
    V[0] = b / beta
    hist = [1.0]
    k = 0
    for k in range(maxit):
        Z[k] = precond(V[k])
        w = A @ Z[k]
        for j in range(k + 1):                     # modified Gram-Schmidt
            H[j, k] = np.dot(V[j], w)
            w = w - H[j, k] * V[j]
        H[k + 1, k] = np.linalg.norm(w)
        if H[k + 1, k] > 0:
            V[k + 1] = w / H[k + 1, k]
        for j in range(k):                         # apply previous rotations
            t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
            H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
            H[j, k] = t
        den = np.hypot(H[k, k], H[k + 1, k])
        cs[k], sn[k] = H[k, k] / den, H[k + 1, k] / den
        H[k, k] = den
        H[k + 1, k] = 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        hist.append(abs(g[k + 1]) / beta)
        if hist[-1] < tol:
            break
    m = k + 1
    y = sla.solve_triangular(H[:m, :m], g[:m])
    x = Z[:m].T @ y
    return x, m, hist
