"""Pins of the oracle's low-synchronisation truncated-Neumann MGS-GMRES
(Algorithm 1) (-m "not gpu"): it must reproduce the classical
MGS-GMRES (Saad-Schultz, oracle.amg.gmres, an independent implementation of
the textbook algorithm) — the paper's claim that the convergence history is
identical — and solve the system."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import inputs
import oracle
from oracle import amg, krylov


def rand_fn(level, n):
    return inputs.uniform(1000 + level, n, 0.0, 1.0)


def graded(N):
    """2-D Poisson with a graded diagonal scaling: kappa ~ 1e6."""
    A = inputs.laplace(N, N, 1).to_scipy()
    s = np.logspace(0, 2, A.shape[0])
    return sp.csr_matrix(sp.diags(s) @ A @ sp.diags(s))


CASES = {
    "poisson32_noprec": (lambda: inputs.laplace(32, 32, 1).to_scipy(), None),
    "graded24_noprec": (lambda: graded(24), None),
    "convdiff8_noprec": (lambda: inputs.convdiff(8).to_scipy(), None),
    "poisson32_amg": (lambda: inputs.laplace(32, 32, 1).to_scipy(), "amg"),
}


def precond_for(A, which):
    if which is None:
        return lambda v: v
    levels = amg.hierarchy(A, rand_fn, min_coarse=50)
    lu = amg.coarse_lu(levels)
    sm = lambda lev, M, b, x, z: oracle.pgs_apply(M, b, x, 2, x_is_zero=z)
    return lambda v: amg.vcycle(levels, sm, v, lu=lu)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("t_mode", ["neumann", "inverse"])
def test_lowsync_matches_classical_mgs(case, t_mode):
    A = CASES[case][0]()
    M = precond_for(A, CASES[case][1])
    b = inputs.uniform(0, A.shape[0])
    tol = 1e-10
    x_ref, m_ref, h_ref = amg.gmres(A, b, M, tol=tol, maxit=300)
    x, m, h = krylov.gmres_lowsync(A, b, M, tol=tol, maxit=300, t_mode=t_mode)
    assert m == m_ref
    # identical convergence history to 1e-8 relative
    np.testing.assert_allclose(h, h_ref, rtol=1e-8, atol=0)
    # same attainable accuracy as the classical algorithm (kappa * eps floor)
    res = lambda v: np.linalg.norm(b - A @ v) / np.linalg.norm(b)
    assert res(x) <= 10 * res(x_ref) + 1e-12


def test_lowsync_solution_matches_direct():
    A = inputs.convdiff(6).to_scipy()
    b = inputs.uniform(0, A.shape[0])
    x, m, h = krylov.gmres_lowsync(A, b, lambda v: v, tol=1e-13, maxit=A.shape[0] + 1)
    np.testing.assert_allclose(x, spla.spsolve(A.tocsc(), b), rtol=1e-9)


def test_truncation_error_is_second_order():
    """T = I - L differs from (I + L)^{-1} by O(||L||^2): the two
    variants' Arnoldi coefficients differ far less than ||L||."""
    A = graded(16)
    b = inputs.uniform(0, A.shape[0])
    _, m1, h1 = krylov.gmres_lowsync(A, b, lambda v: v, tol=1e-12, t_mode="neumann")
    _, m2, h2 = krylov.gmres_lowsync(A, b, lambda v: v, tol=1e-12, t_mode="inverse")
    assert m1 == m2
    np.testing.assert_allclose(h1, h2, rtol=1e-10)
