"""Pins of the CPU oracle against what the paper and the mathematics fix
(-m "not gpu").  None of these re-types the oracle's recurrence: each check
uses a different route to the same value (explicit matrix powers, textbook
substitution via scipy, closed forms, spectra, exact integer arithmetic) so
that a dropped term, a wrong sign or index, or a transposed operand in
oracle/oracle.c fails at least one of them.  DESIGN.md §4 lists which pin
covers which oracle function.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

import inputs
import oracle


def dense(A):
    return A.to_scipy().toarray()


def split(M):
    D = np.diag(np.diag(M))
    return D, np.tril(M, -1), np.triu(M, 1)


def neumann_powers(B, v, k):
    """sum_{j=0..k} (-B)^j v with explicit dense matrix powers."""
    out = np.zeros_like(v)
    for j in range(k + 1):
        out += np.linalg.matrix_power(-B, j) @ v
    return out


# ---------------------------------------------------------------- pin (a) ---
# k inner sweeps from g0 = D^-1 r give the (k+1)-term Neumann sum.
@pytest.mark.parametrize("n", [1, 2, 5, 8])
@pytest.mark.parametrize("density", [1.0, 0.5])
def test_pgs_equals_neumann_powers(n, density):
    A = inputs.random_dense(n, seed=100 + n, density=density)
    M = dense(A)
    D, L, U = split(M)
    Dinv = np.diag(1.0 / np.diag(M))
    b = inputs.uniform(0, n)
    x0 = inputs.uniform(1, n)
    for k in range(0, n + 1):
        # from x = 0 (north_star pin (a))
        got = oracle.pgs_apply(A, b, np.zeros(n), k, x_is_zero=True)
        want = neumann_powers(Dinv @ L, Dinv @ b, k)
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-14)
        # from a nonzero x: x + S_k D^-1 (b - A x)
        got = oracle.pgs_apply(A, b, x0, k)
        want = x0 + neumann_powers(Dinv @ L, Dinv @ (b - M @ x0), k)
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("k", [0, 1, 3])
def test_upper_jacobi_equals_neumann_powers(k):
    n = 7
    A = inputs.random_dense(n, seed=7, density=0.6)
    M = dense(A)
    D, L, U = split(M)
    Dinv = np.diag(1.0 / np.diag(M))
    r = inputs.uniform(3, n)
    got = oracle.tri_jacobi(A, r, k, lower=False)
    np.testing.assert_allclose(got, neumann_powers(Dinv @ U, Dinv @ r, k), rtol=1e-13, atol=1e-14)


def test_unit_lower_jacobi_equals_neumann_powers():
    # unit-lower L = I + L_s: stored diagonal ignored, D = I
    n = 8
    A = inputs.random_dense(n, seed=11, density=0.7)
    Ls = np.tril(dense(A), -1)
    r = inputs.uniform(4, n)
    for k in range(n):
        got = oracle.tri_jacobi(A, r, k, lower=True, unit=True)
        np.testing.assert_allclose(got, neumann_powers(Ls, r, k), rtol=1e-13, atol=1e-13)


# ---------------------------------------------------------------- pin (b) ---
# D^-1 L is nilpotent, so n-1 sweeps reproduce forward substitution.
@pytest.mark.parametrize("n", [3, 6, 8])
def test_nilpotence_equals_forward_substitution(n):
    A = inputs.random_dense(n, seed=200 + n)
    M = dense(A)
    b = inputs.uniform(0, n)
    x0 = inputs.uniform(1, n)
    r = b - M @ x0
    want = x0 + sla.solve_triangular(np.tril(M), r, lower=True)
    got = oracle.pgs_apply(A, b, x0, n - 1)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-13)
    # the classical GS oracle is the same textbook substitution
    np.testing.assert_allclose(oracle.gs_apply(A, b, x0), want, rtol=1e-12, atol=1e-13)
    # upper: backward substitution
    np.testing.assert_allclose(oracle.tri_jacobi(A, r, n - 1, lower=False),
                               sla.solve_triangular(np.triu(M), r, lower=False), rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(oracle.tri_direct(A, r, lower=False),
                               sla.solve_triangular(np.triu(M), r, lower=False), rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("shape", [(9, 1, 1), (8, 8, 1), (5, 5, 5)])
def test_stencil_nilpotency_index(shape):
    """For a d-dimensional lexicographic stencil the nilpotency index of D^-1 L
    is d(N-1)+1: k = d(N-1) sweeps are exact, k = d(N-1)-1 are not."""
    nx, ny, nz = shape
    if ny == 1:  # 1-D tridiagonal (2, -1)
        A = inputs.CSR.from_scipy(sp.diags([-np.ones(nx - 1), 2 * np.ones(nx), -np.ones(nx - 1)], [-1, 0, 1]))
        d = 1
    else:
        A = inputs.laplace(nx, ny, nz)
        d = 2 if nz == 1 else 3
    n = A.nrows
    M = dense(A)
    r = inputs.uniform(0, n, 0.0, 1.0)  # positive r: every Neumann term is > 0
    exact = sla.solve_triangular(np.tril(M), r, lower=True)
    kmax = d * (nx - 1)
    g = oracle.tri_jacobi(A, r, kmax)
    np.testing.assert_allclose(g, exact, rtol=1e-13)
    g1 = oracle.tri_jacobi(A, r, kmax - 1)
    assert np.max(np.abs(g1 - exact) / exact) > 1e-12


def test_poisson64_exact_at_k126():
    """Config C1 (2-D 64x64): exact forward substitution at k = 2*63 = 126."""
    A = inputs.config_matrix("C1")
    b = inputs.uniform(0, A.nrows)
    exact = sla.solve_triangular(np.tril(dense(A)), b, lower=True)
    got = oracle.pgs_apply(A, b, np.zeros(A.nrows), 126, x_is_zero=True)
    assert np.linalg.norm(got - exact) / np.linalg.norm(exact) < 1e-14


# ---------------------------------------------------------------- pin (c) ---
# 2-D 5-point Dirichlet Poisson: rho_J = cos(pi h), rho_GS = cos^2(pi h),
# h = 1/(N+1) (textbook).  For an M-matrix the pGS error operator E_k = I -
# M_k^-1 A satisfies rho_GS <= rho(E_{k+1}) <= rho(E_k) <= rho_J (comparison
# theorem for weak regular splittings; DESIGN.md pin (c)).
def error_operator(A, k):
    n = A.nrows
    E = np.empty((n, n))
    zero = np.zeros(n)
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1.0
        E[:, i] = oracle.pgs_apply(A, zero, e, k)  # b = 0: x_new = E_k x
    return E


# survey-check values of rho(E_k), k = 0..3 (SURVEY.md §8(c) pin (c) rows)
SURVEY_RHO = {8: [0.939693, 0.910563, 0.896112, 0.888981], 16: [0.982973, 0.974537, 0.970327, 0.968229]}


@pytest.mark.parametrize("N", [8, 16])
def test_poisson_spectrum_bracket(N):
    A = inputs.laplace(N, N, 1)
    h = 1.0 / (N + 1)
    rho_j, rho_gs = math.cos(math.pi * h), math.cos(math.pi * h) ** 2
    rhos = []
    for k in range(0, 4):
        rhos.append(max(abs(np.linalg.eigvals(error_operator(A, k)))))
    assert abs(rhos[0] - rho_j) < 1e-10          # k = 0 is Jacobi
    for a, b in zip(rhos, rhos[1:]):
        assert b <= a + 1e-12
    for r in rhos:
        assert rho_gs - 1e-12 <= r <= rho_j + 1e-12
    np.testing.assert_allclose(rhos, SURVEY_RHO[N], atol=2e-6)
    # k at the nilpotency index reproduces GS exactly
    rho_inf = max(abs(np.linalg.eigvals(error_operator(A, 2 * (N - 1)))))
    assert abs(rho_inf - rho_gs) < 1e-8


def test_truncation_bound_config1():
    """||D^-1 L||_2 <= 1/2 for the 5-point stencil, so
    ||g_k - (D+L)^-1 r|| <= 2^-k ||D^-1 r||  (closed-form bound)."""
    A = inputs.config_matrix("C1")
    M = dense(A)
    r = inputs.uniform(0, A.nrows)
    exact = sla.solve_triangular(np.tril(M), r, lower=True)
    for k in range(1, 4):
        g = oracle.tri_jacobi(A, r, k)
        assert np.linalg.norm(g - exact) <= 2.0 ** (-k) * np.linalg.norm(r / 4.0) * (1 + 1e-12)


def test_config1_dyadic_exact():
    """C1 has D = 4I: with integer b (|b| < 2^20) and x = 0 every quantity up
    to k = 3 is a dyadic rational, so fp64 is exact.  Compare bit-for-bit with
    4^{k+1} g_k = sum_j 4^{k-j} (-L)^j b evaluated in int64."""
    A = inputs.config_matrix("C1")
    n = A.nrows
    b = inputs.uniform_int(0, n, 20)
    Lint = sp.tril(A.to_scipy(), -1).astype(np.int64).tocsr()
    bint = b.astype(np.int64)
    for k in range(0, 4):
        h = np.zeros(n, dtype=np.int64)
        t = bint.copy()
        for j in range(k + 1):
            h += (4 ** (k - j)) * t
            t = -(Lint @ t)
        want = h.astype(np.float64) / float(4 ** (k + 1))
        assert np.all(np.abs(h) < 2 ** 52)
        got = oracle.pgs_apply(A, b, np.zeros(n), k, x_is_zero=True)
        assert np.array_equal(got, want)


def test_monotone_in_k_mmatrix():
    """M-matrix, r >= 0: every Neumann term (-B)^j D^-1 r >= 0, so g_k is
    entrywise nondecreasing in k and bounded by (D+L)^-1 r."""
    A = inputs.var27(6)
    M = dense(A)
    r = inputs.uniform(0, A.nrows, 0.0, 1.0)
    exact = sla.solve_triangular(np.tril(M), r, lower=True)
    prev = None
    for k in range(0, 6):
        g = oracle.tri_jacobi(A, r, k)
        assert np.all(g <= exact * (1 + 1e-12))
        if prev is not None:
            assert np.all(g >= prev * (1 - 1e-15))
        prev = g


# ------------------------------------------------------------- 1-D closed form
def test_1d_closed_form():
    """Tridiagonal (-1, 2, -1): D^-1 L = -(1/2) shift, so
    g_{k,i} = sum_{j=0..min(k,i)} 2^{-j-1} r_{i-j}."""
    n = 12
    A = inputs.CSR.from_scipy(sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]))
    r = inputs.uniform(5, n)
    for k in range(0, 5):
        want = np.array([sum(2.0 ** (-j - 1) * r[i - j] for j in range(min(k, i) + 1)) for i in range(n)])
        np.testing.assert_allclose(oracle.tri_jacobi(A, r, k), want, rtol=1e-15, atol=1e-16)


def test_1d_ilu0_closed_form():
    """ILU(0) of a tridiagonal matrix is its exact LU: u_ii = (i+2)/(i+1),
    l_{i+1,i} = -(i+1)/(i+2) (0-based)."""
    n = 10
    A = inputs.CSR.from_scipy(sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]))
    rp, ci, w = oracle.ilu0(A)
    F = sp.csr_matrix((w, ci, rp), shape=(n, n)).toarray()
    for i in range(n):
        assert abs(F[i, i] - (i + 2) / (i + 1)) < 1e-15
        if i + 1 < n:
            assert abs(F[i + 1, i] + (i + 1) / (i + 2)) < 1e-15
            assert F[i, i + 1] == -1.0


# --------------------------------------------------------------------- ILU(0)
def factors_dense(A, F):
    n = A.nrows
    W = sp.csr_matrix((F[2], F[1], F[0]), shape=(n, n)).toarray()
    return np.eye(n) + np.tril(W, -1), np.triu(W)


@pytest.mark.parametrize("which", ["lap2d", "lap3d", "cd_rcm", "rand"])
def test_ilu0_defining_property(which):
    """(L U)_ij = a_ij on pattern(A) (Saad's ILU(0) definition)."""
    if which == "lap2d":
        A = inputs.laplace(8, 8, 1)
    elif which == "lap3d":
        A = inputs.laplace(5, 5, 5)
    elif which == "cd_rcm":
        A = inputs.convdiff(6)
    else:
        A = inputs.random_dense(8, seed=3, density=0.5, diag_shift=4.0)
    M = dense(A)
    L, U = factors_dense(A, oracle.ilu0(A))
    P = L @ U
    mask = M != 0
    mask |= np.eye(A.nrows, dtype=bool)
    np.testing.assert_allclose(P[mask], M[mask], rtol=1e-13, atol=1e-13)
    if which == "lap2d":
        assert np.max(np.abs((P - M)[~mask])) > 0.1  # fill is dropped in 2-D


def test_ilu0_exact_when_no_fill():
    """A = L0 U0 with a dense pattern: ILU(0) is the exact LU."""
    rng = np.random.default_rng(9)
    n = 6
    L0 = np.eye(n) + np.tril(rng.uniform(-0.5, 0.5, (n, n)), -1)
    U0 = np.triu(rng.uniform(-0.5, 0.5, (n, n)), 1) + np.diag(rng.uniform(2, 3, n))
    A = inputs.CSR.from_scipy(sp.csr_matrix(L0 @ U0))
    L, U = factors_dense(A, oracle.ilu0(A))
    np.testing.assert_allclose(L, L0, atol=1e-13)
    np.testing.assert_allclose(U, U0, atol=1e-13)


def test_ilu0_zero_pivot_error():
    A = inputs.CSR.from_scipy(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 1.0]])))
    with pytest.raises(oracle.OracleError):
        oracle.ilu0(A)


@pytest.mark.parametrize("which", ["lap3d", "cd_rcm"])
def test_ilu_apply_limits(which):
    A = inputs.laplace(4, 4, 4) if which == "lap3d" else inputs.convdiff(4)
    n = A.nrows
    M = dense(A)
    F = oracle.ilu0(A)
    L, U = factors_dense(A, F)
    b = inputs.uniform(0, n)
    x0 = inputs.uniform(1, n)
    r = b - M @ x0
    direct = x0 + sla.solve_triangular(U, sla.solve_triangular(L, r, lower=True, unit_diagonal=True), lower=False)
    np.testing.assert_allclose(oracle.ilu_apply(A, F, b, x0, 0, 0, direct=True), direct, rtol=1e-12, atol=1e-13)
    # nilpotence: k >= n-1 sweeps equal the direct solves
    np.testing.assert_allclose(oracle.ilu_apply(A, F, b, x0, n - 1, n - 1), direct, rtol=1e-11, atol=1e-12)
    # closed form at small k: L-solve sum (-L_s)^j r, U-solve Neumann in D_U^-1 U_s
    Ls = L - np.eye(n)
    DU = np.diag(np.diag(U))
    DUi = np.linalg.inv(DU)
    for kL, kU in [(0, 0), (2, 2), (3, 1)]:
        y = neumann_powers(Ls, r, kL)
        z = neumann_powers(DUi @ (U - DU), DUi @ y, kU)
        np.testing.assert_allclose(oracle.ilu_apply(A, F, b, x0, kL, kU), x0 + z, rtol=1e-12, atol=1e-13)


def test_ilu_identity_exact():
    n = 5
    A = inputs.CSR.from_scipy(sp.identity(n, format="csr"))
    b = inputs.uniform(0, n)
    got = oracle.ilu_apply(A, oracle.ilu0(A), b, np.zeros(n), 2, 2, x_is_zero=True)
    assert np.array_equal(got, b)


def test_ilu_sweeps_residual_decreases():
    """Table-1-style triangular relative residuals decrease with k (RCM
    convection-diffusion)."""
    A = inputs.convdiff(10)
    n = A.nrows
    F = oracle.ilu0(A)
    L, U = factors_dense(A, F)
    b = inputs.uniform(0, n)
    prevL = prevU = None
    for k in [1, 2, 3, 5, 10]:
        y = oracle.tri_jacobi(sp.csr_matrix((F[2], F[1], F[0]), shape=(n, n)), b, k, lower=True, unit=True)
        z = oracle.tri_jacobi(sp.csr_matrix((F[2], F[1], F[0]), shape=(n, n)), y, k, lower=False)
        rl = np.linalg.norm(b - L @ y) / np.linalg.norm(b)
        ru = np.linalg.norm(y - U @ z) / np.linalg.norm(y)
        if prevL is not None:
            assert rl < prevL and ru < prevU
        prevL, prevU = rl, ru


# ------------------------------------------------------- smoother as operator
def test_jacobi_special_case():
    """k = 0: x + D^-1 (b - A x)."""
    A = inputs.var27(5)
    M = dense(A)
    b = inputs.uniform(0, A.nrows)
    x0 = inputs.uniform(1, A.nrows)
    want = x0 + (b - M @ x0) / np.diag(M)
    np.testing.assert_allclose(oracle.pgs_apply(A, b, x0, 0), want, rtol=1e-14, atol=1e-15)


def test_residual_and_spmv_dense():
    A = inputs.random_dense(8, seed=5, density=0.6)
    M = dense(A)
    x = inputs.uniform(1, 8)
    b = inputs.uniform(0, 8)
    np.testing.assert_allclose(oracle.residual(A, b, x), b - M @ x, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(oracle.spmv(A, x), M @ x, rtol=1e-14, atol=1e-15)


def test_hybrid_partition_special_cases():
    """HYBRID: one block == GLOBAL; singleton blocks == Jacobi;
    two blocks == Neumann sum of the block-diagonal lower part."""
    A = inputs.laplace(6, 6, 1)
    n = A.nrows
    M = dense(A)
    b = inputs.uniform(0, n)
    x0 = inputs.uniform(1, n)
    k = 3
    g = oracle.pgs_apply(A, b, x0, k)
    assert np.array_equal(oracle.pgs_apply(A, b, x0, k, bounds=[0, n]), g)
    jac = oracle.pgs_apply(A, b, x0, 0)
    np.testing.assert_allclose(oracle.pgs_apply(A, b, x0, k, bounds=np.arange(n + 1)), jac, rtol=0, atol=0)
    bounds = [0, 14, n]
    own = np.searchsorted(bounds, np.arange(n), side="right") - 1
    Lh = np.tril(M, -1) * (own[:, None] == own[None, :])
    Dinv = np.diag(1.0 / np.diag(M))
    want = x0 + neumann_powers(Dinv @ Lh, Dinv @ (b - M @ x0), k)
    np.testing.assert_allclose(oracle.pgs_apply(A, b, x0, k, bounds=bounds), want, rtol=1e-13, atol=1e-14)
    # hybrid direct GS: block forward substitution
    want = x0 + sla.solve_triangular(np.diag(np.diag(M)) + Lh, b - M @ x0, lower=True)
    np.testing.assert_allclose(oracle.gs_apply(A, b, x0, bounds=bounds), want, rtol=1e-13, atol=1e-14)


def test_nu_outer_iterations_compose():
    """nu outer iterations == nu single applications (eq:one-stage)."""
    A = inputs.laplace(5, 5, 5)
    b = inputs.uniform(0, A.nrows)
    x = np.zeros(A.nrows)
    once = x
    for _ in range(3):
        once = oracle.pgs_apply(A, b, once, 2)
    assert np.array_equal(oracle.pgs_apply(A, b, x, 2, nu=3), once)
    assert np.array_equal(oracle.pgs_apply(A, b, x, 2, nu=3, x_is_zero=True), once)


def test_zero_diagonal_error():
    A = inputs.CSR.from_scipy(sp.csr_matrix(np.array([[1.0, 1.0], [1.0, 0.0]])))
    with pytest.raises(oracle.OracleError):
        oracle.pgs_apply(A, np.ones(2), np.zeros(2), 1)


# ------------------------------------------- backward / symmetric / l1-Jacobi
@pytest.mark.parametrize("n", [4, 7])
def test_backward_pgs_neumann_and_nilpotence(n):
    """M = D + U: k sweeps = (k+1)-term Neumann series in
    D^-1 U (dense powers); k = n-1 = backward substitution."""
    A = inputs.random_dense(n, seed=300 + n, density=0.7)
    M = dense(A)
    D, L, U = split(M)
    Dinv = np.diag(1.0 / np.diag(M))
    b, x0 = inputs.uniform(0, n), inputs.uniform(1, n)
    r = b - M @ x0
    for k in range(n):
        want = x0 + neumann_powers(Dinv @ U, Dinv @ r, k)
        np.testing.assert_allclose(oracle.pgs_backward_apply(A, b, x0, k), want, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(oracle.pgs_backward_apply(A, b, x0, n - 1),
                               x0 + sla.solve_triangular(np.triu(M), r, lower=False), rtol=1e-12, atol=1e-13)


def test_symmetric_pgs_is_forward_then_backward_operator():
    """Symmetric pGS error operator = E_back E_fwd with the dense Neumann
    operators M_k^{-1} = S_k D^{-1} of each direction."""
    n = 8
    A = inputs.random_dense(n, seed=17, density=0.6)
    M = dense(A)
    D, L, U = split(M)
    Dinv = np.diag(1.0 / np.diag(M))
    k = 2
    Mf = sum(np.linalg.matrix_power(-Dinv @ L, j) for j in range(k + 1)) @ Dinv
    Mb = sum(np.linalg.matrix_power(-Dinv @ U, j) for j in range(k + 1)) @ Dinv
    I = np.eye(n)
    E = (I - Mb @ M) @ (I - Mf @ M)
    x0 = inputs.uniform(1, n)
    # b = 0: x_new = E x0
    np.testing.assert_allclose(oracle.pgs_symmetric_apply(A, np.zeros(n), x0, k), E @ x0, rtol=1e-12, atol=1e-13)


def test_l1_jacobi_properties():
    # diagonal matrix: exact in one sweep
    A = inputs.CSR.from_scipy(sp.diags(np.arange(1.0, 9.0)).tocsr())
    b = inputs.uniform(0, 8)
    np.testing.assert_allclose(oracle.l1_jacobi_apply(A, b, np.zeros(8)), b / np.arange(1.0, 9.0), rtol=1e-15)
    # zero-row-sum interior rows of an M-matrix: D_l1 = 2 a_ii
    A = inputs.var27(6)
    M = dense(A)
    x0 = inputs.uniform(1, A.nrows)
    b = inputs.uniform(0, A.nrows)
    dl1 = np.diag(M) + np.abs(M - np.diag(np.diag(M))).sum(1)
    i = 2 + 6 * (2 + 6 * 2)
    assert abs(dl1[i] - 2 * M[i, i]) < 1e-9 * M[i, i]
    got = oracle.l1_jacobi_apply(A, b, x0)
    np.testing.assert_allclose(got, x0 + (b - M @ x0) / dl1, rtol=1e-13, atol=1e-14)
    # unconditionally convergent for SPD A (Baker et al. 2011): rho(I - D_l1^-1 A) < 1
    rho = max(abs(np.linalg.eigvals(np.eye(A.nrows) - M / dl1[:, None])))
    assert rho < 1.0


# ------------------------------------------------ all-cores oracle build ---
# bench.py's all-cores CPU baseline (SURVEY.md §8(d) "Oracle timing") loads the
# same oracle.c built with -fopenmp.  Its row loops keep each row's ascending
# order, so it must agree with the single-thread parity build bit for bit.
def test_all_cores_build_is_bitwise_serial():
    A = inputs.var27(20)
    F = oracle.ilu0(A)
    b, x = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    bounds = np.array([0, 3000, 5100, A.nrows], dtype=np.int64)
    want = [oracle.residual(A, b, x), oracle.pgs_apply(A, b, x, 3, nu=2),
            oracle.pgs_backward_apply(A, b, x, 2), oracle.ilu_apply(A, F, b, x, 2, 3),
            oracle.pgs_apply(A, b, x, 2, bounds=bounds), oracle.l1_jacobi_apply(A, b, x, nu=2)]
    try:
        assert oracle.use_all_cores(True) >= 1
        got = [oracle.residual(A, b, x), oracle.pgs_apply(A, b, x, 3, nu=2),
               oracle.pgs_backward_apply(A, b, x, 2), oracle.ilu_apply(A, F, b, x, 2, 3),
               oracle.pgs_apply(A, b, x, 2, bounds=bounds), oracle.l1_jacobi_apply(A, b, x, nu=2)]
    finally:
        oracle.use_all_cores(False)
    for w, g in zip(want, got):
        assert np.array_equal(w, g)
