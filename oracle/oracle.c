/*
 * oracle/oracle.c — the CPU ORACLE for the Neumann-series smoothers of
 * arXiv 2112.14681 ("Neumann series in GMRES and algebraic multigrid
 * smoothers", PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2112_14681_b200/) never links, imports or calls it, and
 * it shares no code, header or helper with that path.
 *
 * Rules this file follows (DESIGN.md §4 "Oracle"):
 *   - plain, slow, obviously correct: one loop per formula, in the paper's
 *     order and notation; fp64; compiled with -O2 -ffp-contract=off (no FMA
 *     contraction, no fast-math);
 *   - every row sum is accumulated from 0 in ASCENDING column order
 *     (reading R10);
 *   - Jacobi inner iterations are OUT-OF-PLACE (previous iterate only,
 *     eq:jacobi P:L757-764; reading R2);
 *   - a "partition" (nblocks, bounds[nblocks+1]) restricts the inner
 *     triangular couplings to j with owner(j) == owner(i): HYBRID semantics
 *     (P:L733-741).  nblocks == 1 is the exact global method (GLOBAL mode).
 *     The residual always uses the full matrix (boundary values
 *     are exchanged before the local relaxation).
 *
 * Matrices are CSR: rowptr[n+1] (int64), col[nnz] (int64, strictly ascending
 * per row), val[nnz] (double).  Return codes: 0 ok, -1 bad argument,
 * -(2 + row) missing/zero diagonal (or zero pivot) at `row`.
 *
 * Parity status of each function: see the table in DESIGN.md §4; every
 * function here is pinned by a -m "not gpu" test in tests/test_oracle_pins.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* Row-parallel loops (each row's arithmetic is independent of the others and
 * keeps its own ascending order, so results do not depend on the thread
 * count).  The parity oracle is built WITHOUT -fopenmp (pragma ignored,
 * single thread); bench.py's all-cores CPU baseline loads the same source
 * built with -fopenmp (liboracle_omp.so).  tests/test_oracle_pins.py checks
 * the two builds agree bit for bit. */
#ifdef _OPENMP
#define ORC_ROWS _Pragma("omp parallel for schedule(static)")
#else
#define ORC_ROWS
#endif

/* owner block of row/column j under the partition (bounds ascending) */
static i64 owner(i64 j, int nblocks, const i64 *bounds) {
    if (nblocks <= 1) return 0;
    i64 lo = 0, hi = nblocks - 1;
    while (lo < hi) {                      /* largest b with bounds[b] <= j */
        i64 mid = (lo + hi + 1) / 2;
        if (bounds[mid] <= j) lo = mid; else hi = mid - 1;
    }
    return lo;
}

/* d_i = a_ii (A = L + D + U).  Missing or zero diagonal is an
 * error (reading R9). */
static int diagonal(i64 n, const i64 *rp, const i64 *ci, const double *va, double *d) {
    ORC_ROWS
    for (i64 i = 0; i < n; ++i) {
        d[i] = 0.0;
        for (i64 p = rp[i]; p < rp[i + 1]; ++p)
            if (ci[p] == i) d[i] = va[p];
    }
    for (i64 i = 0; i < n; ++i)
        if (d[i] == 0.0) return (int)(-(2 + i));
    return 0;
}

/* r = b - A x :  r_i = b_i - (sum_{j ascending} a_ij x_j)
 * ("r^(k) = b - A x^(k)"). */
int orc_residual(i64 n, const i64 *rp, const i64 *ci, const double *va,
                 const double *b, const double *x, double *r) {
    ORC_ROWS
    for (i64 i = 0; i < n; ++i) {
        double s = 0.0;
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) s = s + va[p] * x[ci[p]];
        r[i] = b[i] - s;
    }
    return 0;
}

/* y = A x  (plain SpMV, ascending columns; used by the driver tests) */
int orc_spmv(i64 n, const i64 *rp, const i64 *ci, const double *va, const double *x, double *y) {
    ORC_ROWS
    for (i64 i = 0; i < n; ++i) {
        double s = 0.0;
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) s = s + va[p] * x[ci[p]];
        y[i] = s;
    }
    return 0;
}

/*
 * Jacobi-iterated triangular solve  T g = r  with k inner sweeps
 * (P:L753-764 eq:jr-initial-guess, eq:jacobi; P:L826-829 eq:LUiterMat):
 *
 *   g^(0)   = D_T^{-1} r
 *   g^(j+1) = D_T^{-1} ( r - T_s g^(j) ),   j = 0 .. k-1
 *
 * T is the lower (lower=1) or upper (lower=0) triangle of the CSR matrix
 * (entries on the other side are ignored), T_s its strict part and D_T its
 * diagonal; with unit=1 the diagonal is the identity and stored diagonal
 * entries are ignored (unit-lower ILU factor).  After k sweeps
 * g = sum_{j=0..k} (-D_T^{-1} T_s)^j D_T^{-1} r.
 * Couplings to other partition blocks are dropped (HYBRID, nblocks > 1).
 */
int orc_tri_jacobi(i64 n, const i64 *rp, const i64 *ci, const double *va, int lower, int unit,
                   const double *r, int k, int nblocks, const i64 *bounds, double *g) {
    if (k < 0) return -1;
    double *d = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    double *gn = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!d || !gn) { free(d); free(gn); return -1; }
    int rc = 0;
    if (unit) { for (i64 i = 0; i < n; ++i) d[i] = 1.0; }
    else if ((rc = diagonal(n, rp, ci, va, d)) != 0) { free(d); free(gn); return rc; }
    ORC_ROWS
    for (i64 i = 0; i < n; ++i) g[i] = r[i] / d[i];
    for (int s = 0; s < k; ++s) {
        ORC_ROWS
        for (i64 i = 0; i < n; ++i) {
            i64 oi = owner(i, nblocks, bounds);
            double acc = 0.0;
            for (i64 p = rp[i]; p < rp[i + 1]; ++p) {
                i64 j = ci[p];
                if ((lower ? j < i : j > i) && owner(j, nblocks, bounds) == oi) acc = acc + va[p] * g[j];
            }
            gn[i] = (r[i] - acc) / d[i];
        }
        memcpy(g, gn, (size_t)n * sizeof(double));
    }
    free(d); free(gn);
    return 0;
}

/* Direct (exact) triangular solve  T y = r  by forward (lower) or backward
 * (upper) substitution: the classical recurrences the paper replaces
 * (P:L729-731).  Same triangle/unit/partition conventions. */
int orc_tri_direct(i64 n, const i64 *rp, const i64 *ci, const double *va, int lower, int unit,
                   const double *r, int nblocks, const i64 *bounds, double *y) {
    double *d = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!d) return -1;
    int rc = 0;
    if (unit) { for (i64 i = 0; i < n; ++i) d[i] = 1.0; }
    else if ((rc = diagonal(n, rp, ci, va, d)) != 0) { free(d); return rc; }
    for (i64 t = 0; t < n; ++t) {
        i64 i = lower ? t : n - 1 - t;
        i64 oi = owner(i, nblocks, bounds);
        double acc = 0.0;
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) {
            i64 j = ci[p];
            if ((lower ? j < i : j > i) && owner(j, nblocks, bounds) == oi) acc = acc + va[p] * y[j];
        }
        y[i] = (r[i] - acc) / d[i];
    }
    free(d);
    return 0;
}

/*
 * Polynomial Gauss-Seidel smoother, nu outer iterations:
 *   r     = b - A x                                   (eq:polynomial)
 *   g     = k Jacobi sweeps on (D + L) g = r from g^(0) = D^{-1} r
 *   x     = x + g
 * k = 0 is Jacobi.  x_is_zero: the caller asserts x == 0 on
 * entry, so the first residual is b (reading R3; exact).
 */
int orc_pgs_apply(i64 n, const i64 *rp, const i64 *ci, const double *va, const double *b,
                  double *x, int k, int nu, int x_is_zero, int nblocks, const i64 *bounds) {
    double *r = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    double *g = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!r || !g) { free(r); free(g); return -1; }
    int rc = 0;
    for (int it = 0; it < nu && rc == 0; ++it) {
        if (it == 0 && x_is_zero) memcpy(r, b, (size_t)n * sizeof(double));
        else orc_residual(n, rp, ci, va, b, x, r);
        rc = orc_tri_jacobi(n, rp, ci, va, 1, 0, r, k, nblocks, bounds, g);
        if (rc) break;
        ORC_ROWS
        for (i64 i = 0; i < n; ++i) x[i] = x[i] + g[i];
    }
    free(r); free(g);
    return rc;
}

/* Polynomial GS with the backward splitting M = D + U (eq:one-stage,
 * P:L726-727 "M = U + D ... backward sweeps"), same Neumann construction
 * with the upper triangle: x = x + sum_{j<=k} (-D^{-1}U)^j D^{-1} (b - A x). */
int orc_pgs_backward_apply(i64 n, const i64 *rp, const i64 *ci, const double *va, const double *b,
                           double *x, int k, int nu, int x_is_zero, int nblocks, const i64 *bounds) {
    double *r = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    double *g = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!r || !g) { free(r); free(g); return -1; }
    int rc = 0;
    for (int it = 0; it < nu && rc == 0; ++it) {
        if (it == 0 && x_is_zero) memcpy(r, b, (size_t)n * sizeof(double));
        else orc_residual(n, rp, ci, va, b, x, r);
        rc = orc_tri_jacobi(n, rp, ci, va, 0, 0, r, k, nblocks, bounds, g);
        if (rc) break;
        ORC_ROWS
        for (i64 i = 0; i < n; ++i) x[i] = x[i] + g[i];
    }
    free(r); free(g);
    return rc;
}

/* l1-Jacobi (named by the paper as the comparison smoother; the
 * definition is hypre's as fixed by S:L354-359):
 *   d_i = a_ii + sum_{j != i} |a_ij|  (ascending columns, summed from 0)
 *   x = x + D_l1^{-1} (b - A x), nu times. */
int orc_l1_jacobi_apply(i64 n, const i64 *rp, const i64 *ci, const double *va, const double *b, double *x,
                        int nu, int x_is_zero) {
    double *r = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    double *d = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!r || !d) { free(r); free(d); return -1; }
    int rc = diagonal(n, rp, ci, va, d);
    if (rc) { free(r); free(d); return rc; }
    for (i64 i = 0; i < n; ++i) {
        double s = 0.0;
        for (i64 p = rp[i]; p < rp[i + 1]; ++p)
            if (ci[p] != i) s = s + (va[p] < 0 ? -va[p] : va[p]);
        d[i] = d[i] + s;
    }
    for (int it = 0; it < nu; ++it) {
        if (it == 0 && x_is_zero) memcpy(r, b, (size_t)n * sizeof(double));
        else orc_residual(n, rp, ci, va, b, x, r);
        for (i64 i = 0; i < n; ++i) x[i] = x[i] + r[i] / d[i];
    }
    free(r); free(d);
    return 0;
}

/* Classical (direct) forward Gauss-Seidel, nu sweeps: x = x + (D+L)^{-1}(b - Ax)
 * (eq:one-stage).  With a partition this is hypre's hybrid GS
 * (P:L733-741).  It is the exact operator pGS approximates (config C1). */
int orc_gs_apply(i64 n, const i64 *rp, const i64 *ci, const double *va, const double *b,
                 double *x, int nu, int nblocks, const i64 *bounds) {
    double *r = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    double *y = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!r || !y) { free(r); free(y); return -1; }
    int rc = 0;
    for (int it = 0; it < nu && rc == 0; ++it) {
        orc_residual(n, rp, ci, va, b, x, r);
        rc = orc_tri_direct(n, rp, ci, va, 1, 0, r, nblocks, bounds, y);
        if (rc) break;
        for (i64 i = 0; i < n; ++i) x[i] = x[i] + y[i];
    }
    free(r); free(y);
    return rc;
}

/*
 * ILU(0): incomplete LU with the sparsity pattern of A, IKJ variant, no
 * pivoting (the "ILU(0)" building block of P:L193-196).
 * Writes the factor values on the pattern of A into w: strictly-lower part =
 * L_s of the unit-lower L = I + L_s, upper part incl. diagonal = U.
 *   for i = 1..n-1, for k in row i with k < i (ascending):
 *       w_ik <- w_ik / w_kk
 *       for j in row k with j > k and (i,j) in pattern: w_ij <- w_ij - w_ik * w_kj
 * Zero pivot or missing diagonal -> -(2 + row).
 */
int orc_ilu0(i64 n, const i64 *rp, const i64 *ci, const double *va, double *w) {
    i64 nnz = rp[n];
    memcpy(w, va, (size_t)nnz * sizeof(double));
    i64 *pos = (i64 *)malloc((size_t)(n > 0 ? n : 1) * sizeof(i64));
    i64 *dpos = (i64 *)malloc((size_t)(n > 0 ? n : 1) * sizeof(i64));
    if (!pos || !dpos) { free(pos); free(dpos); return -1; }
    for (i64 j = 0; j < n; ++j) pos[j] = -1;
    for (i64 i = 0; i < n; ++i) {
        dpos[i] = -1;
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) if (ci[p] == i) dpos[i] = p;
        if (dpos[i] < 0) { free(pos); free(dpos); return (int)(-(2 + i)); }
    }
    int rc = 0;
    for (i64 i = 0; i < n && rc == 0; ++i) {
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) pos[ci[p]] = p;
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) {
            i64 k = ci[p];
            if (k >= i) break;
            double piv = w[dpos[k]];
            if (piv == 0.0) { rc = (int)(-(2 + k)); break; }
            w[p] = w[p] / piv;
            for (i64 q = rp[k]; q < rp[k + 1]; ++q) {
                i64 j = ci[q];
                if (j <= k) continue;
                if (pos[j] >= 0) w[pos[j]] = w[pos[j]] - w[p] * w[q];
            }
        }
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) pos[ci[p]] = -1;
        if (rc == 0 && w[dpos[i]] == 0.0) rc = (int)(-(2 + i));
    }
    free(pos); free(dpos);
    return rc;
}

/*
 * Chow-Patel fixed-point ILU(0) — the set-up algorithm the paper names as
 * future work ("fixed-point iteration algorithms of Chow and
 * Patel [Chow2015] ... to compute the ILU(0) ... factorizations").  The paper
 * does not restate it; this is the standard definition (reading R19):
 * the ILU(0) factors are the solution of the nonlinear equations
 *     (L U)_ij = a_ij   for every (i,j) in S = pattern(A),  L unit lower,
 * written as the fixed point
 *     l_ij = ( a_ij - sum_{k<j} l_ik u_kj ) / u_jj     (i > j)
 *     u_ij =   a_ij - sum_{k<i} l_ik u_kj              (i <= j)
 * (sums over k with (i,k), (k,j) in S, ascending k, one subtraction each) and
 * iterated SYNCHRONOUSLY: every entry of sweep s+1 uses only sweep-s values.
 * Initial guess (reading R19): l_ij = a_ij / a_jj, u_ij = a_ij.
 * Output layout as orc_ilu0 (strict lower = L_s, upper incl. diagonal = U).
 * Pinned in tests/test_oracle_chow_patel.py: n sweeps reproduce orc_ilu0
 * (Saad's IKJ ILU(0)) bit for bit; the 1-D closed form becomes exact one
 * entry per sweep.
 */
int orc_ilu0_fixed_point(i64 n, const i64 *rp, const i64 *ci, const double *va, int sweeps, double *w) {
    i64 nnz = rp[n];
    i64 *dpos = (i64 *)malloc((size_t)(n > 0 ? n : 1) * sizeof(i64));
    double *old = (double *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
    if (!dpos || !old) { free(dpos); free(old); return -1; }
    for (i64 i = 0; i < n; ++i) {
        dpos[i] = -1;
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) if (ci[p] == i) dpos[i] = p;
        if (dpos[i] < 0 || va[dpos[i]] == 0.0) { free(dpos); free(old); return (int)(-(2 + i)); }
    }
    /* initial guess */
    for (i64 i = 0; i < n; ++i)
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) {
            i64 j = ci[p];
            w[p] = (j < i) ? va[p] / va[dpos[j]] : va[p];
        }
    int rc = 0;
    for (int s = 0; s < sweeps && rc == 0; ++s) {
        memcpy(old, w, (size_t)nnz * sizeof(double));
        for (i64 i = 0; i < n && rc == 0; ++i) {
            for (i64 p = rp[i]; p < rp[i + 1]; ++p) {
                i64 j = ci[p];
                i64 m = j < i ? j : i;          /* k < min(i, j) */
                double sum = va[p];
                for (i64 q = rp[i]; q < rp[i + 1]; ++q) {
                    i64 k = ci[q];              /* l_ik, ascending k */
                    if (k >= m) break;
                    for (i64 t = rp[k]; t < rp[k + 1]; ++t) {  /* u_kj, if (k,j) in S */
                        if (ci[t] == j) { sum = sum - old[q] * old[t]; break; }
                        if (ci[t] > j) break;
                    }
                }
                if (j < i) {
                    double ujj = old[dpos[j]];
                    if (ujj == 0.0) { rc = (int)(-(2 + j)); break; }
                    w[p] = sum / ujj;
                } else {
                    w[p] = sum;
                }
            }
        }
    }
    free(dpos); free(old);
    return rc;
}

/*
 * ILU smoother with Jacobi-iterated triangular solves, nu outer iterations
 * (Algorithm 2, with LDU row scaling of U in place of Ruiz,
 * P:L1012-1013):
 *   r = b - A x
 *   y = kL Jacobi sweeps on (I + L_s) y = r     from y^(0) = r
 *   z = kU Jacobi sweeps on U z = y             from z^(0) = D_U^{-1} y
 *   x = x + z
 * F holds the factors on its own pattern (orc_ilu0 output: strict lower =
 * L_s, upper incl. diagonal = U).  Sweep-count reading R1: Alg. 2's m_L is
 * kL + 1 (its y^(0) = 0 first sweep produces y = r).
 */
int orc_ilu_apply(i64 n, const i64 *rp, const i64 *ci, const double *va,
                  const i64 *frp, const i64 *fci, const double *fva, const double *b, double *x,
                  int kL, int kU, int nu, int x_is_zero, int direct, int nblocks, const i64 *bounds) {
    double *r = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    double *y = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    double *z = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!r || !y || !z) { free(r); free(y); free(z); return -1; }
    int rc = 0;
    for (int it = 0; it < nu && rc == 0; ++it) {
        if (it == 0 && x_is_zero) memcpy(r, b, (size_t)n * sizeof(double));
        else orc_residual(n, rp, ci, va, b, x, r);
        if (direct) {
            rc = orc_tri_direct(n, frp, fci, fva, 1, 1, r, nblocks, bounds, y);
            if (!rc) rc = orc_tri_direct(n, frp, fci, fva, 0, 0, y, nblocks, bounds, z);
        } else {
            rc = orc_tri_jacobi(n, frp, fci, fva, 1, 1, r, kL, nblocks, bounds, y);
            if (!rc) rc = orc_tri_jacobi(n, frp, fci, fva, 0, 0, y, kU, nblocks, bounds, z);
        }
        if (rc) break;
        ORC_ROWS
        for (i64 i = 0; i < n; ++i) x[i] = x[i] + z[i];
    }
    free(r); free(y); free(z);
    return rc;
}
