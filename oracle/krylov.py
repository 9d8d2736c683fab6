"""CPU ORACLE — low-synchronisation MGS-GMRES with the truncated Neumann
correction matrix (Algorithm 1; §2; §4
P:L442-474).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy, fp64.

One iteration k (0-based) of the one-reduce ICWY MGS-GMRES with lagged
normalisation, in the paper's notation (L = strictly lower part of V^T V,
T = (I + L)^{-1}, eq:GS P:L149-152):

  w   = A M u                        (u = unnormalised candidate v_k; Alg.1 step 5)
  [a, nu, c, mu] = [V_k, u]^T [u, w] (ONE global reduction; step 6)
  rho = sqrt(nu); v_k = u / rho      (lagged normalisation; steps 7-8)
  H[k, k-1] = rho                    (completes Arnoldi column k-1; Givens, check)
  L[k, :k] = a / rho                 (step 10: one row of L, eq:matvec P:L316-318)
  z = [c, mu / rho] / rho            (step 9: scale for Arnoldi)
  h = T z,   T = I - L (Neumann, truncated: the paper's choice, step 11)
             or T = (I + L)^{-1} (exact triangular solve)
  H[:k+1, k] = h ;  u <- w / rho - V_{k+1} h   (step 12)

Convergence is tested on the implicit residual |g_{m}| / ||b|| of the
completed columns, so column k-1 is tested at iteration k (one iteration of
lag, the price of the single reduction).  x = M (V_m y_m), x0 = 0.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def gmres_lowsync(A, b, precond, tol: float = 1e-5, maxit: int = 200, t_mode: str = "neumann"):
    """Returns (x, iterations m, implicit relres history [1, ...])."""
    n = len(b)
    beta = np.linalg.norm(b)
    V = np.zeros((maxit + 1, n))
    Lm = np.zeros((maxit + 1, maxit + 1))
    H = np.zeros((maxit + 1, maxit))
    cs, sn = np.zeros(maxit), np.zeros(maxit)
    g = np.zeros(maxit + 1)
    g[0] = beta
    hist = [1.0]
    u = np.array(b, dtype=np.float64, copy=True)
    m = 0

    def complete_column(j, rho):
        """H[j+1, j] = rho; rotate column j; update g."""
        H[j + 1, j] = rho
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        den = np.hypot(H[j, j], H[j + 1, j])
        cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
        H[j, j] = den
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        hist.append(abs(g[j + 1]) / beta)

    for k in range(maxit + 1):
        w = A @ precond(u) if k < maxit else None
        # the single reduction: [V_k, u]^T [u, w]
        a = V[:k] @ u
        nu = float(u @ u)
        rho = np.sqrt(nu)
        if k > 0:
            complete_column(k - 1, rho)
            if hist[-1] < tol or k == maxit:
                m = k
                break
        c = V[:k] @ w
        mu = float(u @ w)
        V[k] = u / rho
        Lm[k, :k] = a / rho
        z = np.concatenate([c, [mu / rho]]) / rho
        Lk = Lm[:k + 1, :k + 1]
        if t_mode == "neumann":
            h = z - Lk @ z                      # T = I - L (truncated Neumann)
        elif t_mode == "inverse":
            h = sla.solve_triangular(np.eye(k + 1) + Lk, z, lower=True)
        else:
            raise ValueError(t_mode)
        H[:k + 1, k] = h
        u = w / rho - V[:k + 1].T @ h
    y = sla.solve_triangular(H[:m, :m], g[:m])
    x = precond(V[:m].T @ y)
    return x, m, hist


def loss_of_orthogonality(V):
    """||I - V^T V||_F of the computed basis."""
    G = V @ V.T
    return np.linalg.norm(np.eye(len(V)) - G)
