"""CPU ORACLE — ILUT(droptol, lfil) factors and Ruiz scaling of the U factor
(Algorithm 2).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain Python loops
(small matrices only), fp64, in the order of Saad's dual-threshold ILUT
(the factorisation Alg. 2 names, "Compute A ~ LU with droptol and lfill
imposed"):

  for each row i:   w = a_i*,  tau_i = droptol * ||a_i||_2
    for k < i, nonzeros of w in ascending column order (fill included):
        w_k = w_k / u_kk ;  if |w_k| < tau_i: drop w_k
        else: w_j = w_j - w_k * u_kj  for every j > k in row k of U
    drop every off-diagonal w_j with |w_j| < tau_i; keep the lfil largest
    in the L part and the lfil largest in the U part (ties: smaller column
    first); the diagonal is always kept; zero pivot -> error.

Ruiz (Knight et al.; Alg. 2 line "Apply the Ruiz strategy"):
iterated sup-norm row/column equilibration of U, then an exact diagonal
normalisation of the rows, so that U~ = diag(1/s_r) U diag(1/s_c) has a unit
diagonal; the scaling is kept as the DIVISORS s_r, s_c (reading R18).
"""
from __future__ import annotations

import math

import numpy as np


class IlutError(RuntimeError):
    pass


def ilut(A, droptol: float, lfil: int):
    """A: scipy CSR (square).  Returns (rowptr, col, val) of the factors on
    ONE pattern: strictly-lower = L_s (unit-lower L), upper incl. diagonal = U."""
    import scipy.sparse as sp
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    Urows = []                       # per row: dict col -> value (j >= i)
    rows_out = []
    for i in range(n):
        lo, hi = A.indptr[i], A.indptr[i + 1]
        w = {int(j): float(v) for j, v in zip(A.indices[lo:hi], A.data[lo:hi])}
        tau = droptol * math.sqrt(sum(v * v for v in A.data[lo:hi]))
        done = set()
        while True:
            cand = [k for k in w if k < i and k not in done]
            if not cand:
                break
            k = min(cand)
            done.add(k)
            ukk = Urows[k][k]
            wk = w[k] / ukk
            if abs(wk) < tau:
                del w[k]
                continue
            w[k] = wk
            for j, ukj in sorted(Urows[k].items()):
                if j <= k:
                    continue
                w[j] = w.get(j, 0.0) - wk * ukj
        if i not in w or w[i] == 0.0:
            raise IlutError(f"zero pivot at row {i}")
        keep_l = [(j, v) for j, v in w.items() if j < i and abs(v) >= tau]
        keep_u = [(j, v) for j, v in w.items() if j > i and abs(v) >= tau]
        keep_l = sorted(keep_l, key=lambda t: (-abs(t[1]), t[0]))[:lfil]
        keep_u = sorted(keep_u, key=lambda t: (-abs(t[1]), t[0]))[:lfil]
        row = sorted(keep_l + [(i, w[i])] + keep_u)
        Urows.append({j: v for j, v in row if j >= i})
        rows_out.append(row)
    rp = np.zeros(n + 1, dtype=np.int64)
    for i, row in enumerate(rows_out):
        rp[i + 1] = rp[i] + len(row)
    col = np.array([j for row in rows_out for j, _ in row], dtype=np.int64)
    val = np.array([v for row in rows_out for _, v in row], dtype=np.float64)
    return rp, col, val


def ruiz_upper(rp, col, val, max_iters: int = 5):
    """Ruiz scaling of the upper part (incl. diagonal) of the factor CSR.
    Returns (val_scaled, s_r, s_c): on the upper entries u~_ij = u_ij / s_r_i /
    s_c_j, then rows divided by their diagonal (s_r_i *= u~_ii) so u~_ii = 1;
    strictly-lower entries (L_s) are returned unchanged."""
    n = len(rp) - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    up = col >= rows
    v = val.copy()
    s_r = np.ones(n)
    s_c = np.ones(n)
    for _ in range(max_iters):
        rmax = np.zeros(n)
        cmax = np.zeros(n)
        for p in np.nonzero(up)[0]:
            rmax[rows[p]] = max(rmax[rows[p]], abs(v[p]))
            cmax[col[p]] = max(cmax[col[p]], abs(v[p]))
        dr = np.sqrt(rmax)
        dc = np.sqrt(cmax)
        dr[dr == 0] = 1.0
        dc[dc == 0] = 1.0
        for p in np.nonzero(up)[0]:
            v[p] = v[p] / dr[rows[p]] / dc[col[p]]
        s_r = s_r * dr
        s_c = s_c * dc
    # exact unit diagonal: divide each row by its diagonal
    diag = np.ones(n)
    for p in np.nonzero(up & (col == rows))[0]:
        diag[rows[p]] = v[p]
    for p in np.nonzero(up)[0]:
        v[p] = v[p] / diag[rows[p]]
    s_r = s_r * diag
    return v, s_r, s_c


def ilu_ruiz_apply(A, F, s_r, s_c, b, x, kL, kU, nu=1, x_is_zero=False):
    """Alg. 2 with Ruiz: r = b - A x; y = kL Jacobi sweeps on the unit-lower
    L (y0 = r); y~ = y / s_r; v = kU Jacobi sweeps on the unit-diagonal
    U~ (v0 = y~); x += v / s_c.  F = (rowptr, col, val) with U~ on the upper part."""
    from oracle import residual, tri_jacobi  # the C oracle's residual and sweeps
    import scipy.sparse as sp
    n = len(b)
    Fs = sp.csr_matrix((F[2], F[1], F[0]), shape=(n, n))
    x = np.zeros(n) if x_is_zero else np.array(x, dtype=np.float64, copy=True)   # contents ignored
    for it in range(nu):
        r = np.array(b, dtype=np.float64, copy=True) if (it == 0 and x_is_zero) else residual(A, b, x)
        y = tri_jacobi(Fs, r, kL, lower=True, unit=True)
        yt = y / s_r
        v = tri_jacobi(Fs, yt, kU, lower=False)          # diagonal of U~ is exactly 1
        x = x + v / s_c
    return x
