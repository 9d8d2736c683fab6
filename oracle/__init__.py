"""CPU ORACLE for the Neumann-series smoothers of arXiv 2112.14681.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares
no code with the CUDA path (paper_2112_14681_b200/) and never imports it.

The arithmetic lives in oracle.c (plain C, fp64, -O2 -ffp-contract=off, one
loop per formula in the paper's order); this file is ctypes marshalling only.
Function-by-function citations are in oracle.c and DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


class OracleError(RuntimeError):
    pass


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
_libs = {}
_variant = "serial"
_CFLAGS = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall", "-Wno-unknown-pragmas"]


def _build_one(path: str, extra: list, force: bool) -> str:
    if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_SRC):
        tmp = path + f".tmp{os.getpid()}"
        subprocess.check_call(_CFLAGS + extra + ["-o", tmp, _SRC])
        os.replace(tmp, path)
    return path


def build(force: bool = False) -> str:
    """liboracle.so (single thread: the parity oracle) and liboracle_omp.so
    (the same source with -fopenmp: its row loops run on all cores with
    per-row arithmetic unchanged; used only for bench.py's all-cores CPU
    baseline)."""
    _build_one(_LIB_OMP, ["-fopenmp"], force)
    return _build_one(_LIB, [], force)


def use_all_cores(on: bool = True) -> int:
    """Switch every function of this module to the -fopenmp build (on) or
    back to the single-thread parity build (off).  Returns the number of
    threads the row loops use (1 when off)."""
    global _variant
    _variant = "omp" if on else "serial"
    if not on:
        return 1
    _L()
    return len(os.sched_getaffinity(0)) if not os.environ.get("OMP_NUM_THREADS") else int(os.environ["OMP_NUM_THREADS"])


def _L():
    lib = _libs.get(_variant)
    if lib is None:
        build()
        lib = ctypes.CDLL(_LIB_OMP if _variant == "omp" else _LIB)
        i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        lib.orc_residual.argtypes = [i64, vp, vp, vp, vp, vp, vp]
        lib.orc_spmv.argtypes = [i64, vp, vp, vp, vp, vp]
        lib.orc_tri_jacobi.argtypes = [i64, vp, vp, vp, ci, ci, vp, ci, ci, vp, vp]
        lib.orc_tri_direct.argtypes = [i64, vp, vp, vp, ci, ci, vp, ci, vp, vp]
        lib.orc_pgs_apply.argtypes = [i64, vp, vp, vp, vp, vp, ci, ci, ci, ci, vp]
        lib.orc_gs_apply.argtypes = [i64, vp, vp, vp, vp, vp, ci, ci, vp]
        lib.orc_pgs_backward_apply.argtypes = [i64, vp, vp, vp, vp, vp, ci, ci, ci, ci, vp]
        lib.orc_l1_jacobi_apply.argtypes = [i64, vp, vp, vp, vp, vp, ci, ci]
        lib.orc_ilu0.argtypes = [i64, vp, vp, vp, vp]
        lib.orc_ilu0_fixed_point.argtypes = [i64, vp, vp, vp, ci, vp]
        lib.orc_ilu_apply.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp, vp, ci, ci, ci, ci, ci, ci, vp]
        _libs[_variant] = lib
    return lib


def _p(a):
    return 0 if a is None else a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _csr(A):
    """Accept inputs.CSR or a scipy sparse matrix (square, rows 0..n-1)."""
    if hasattr(A, "rowptr"):
        return A.nrows, np.ascontiguousarray(A.rowptr, np.int64), np.ascontiguousarray(A.col, np.int64), _f64(A.val)
    m = A.tocsr()
    m.sort_indices()
    return m.shape[0], m.indptr.astype(np.int64), m.indices.astype(np.int64), _f64(m.data)


def _part(bounds):
    if bounds is None:
        return 1, None
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    return len(b) - 1, b


def _check(rc, what):
    if rc == -1:
        raise OracleError(f"{what}: bad argument")
    if rc <= -2:
        raise OracleError(f"{what}: zero or missing diagonal / pivot at row {-rc - 2}")


def residual(A, b, x):
    n, rp, ci, va = _csr(A)
    b, x = _f64(b), _f64(x)
    r = np.empty(n)
    _L().orc_residual(n, _p(rp), _p(ci), _p(va), _p(b), _p(x), _p(r))
    return r


def spmv(A, x):
    n, rp, ci, va = _csr(A)
    x = _f64(x)
    y = np.empty(n)
    _L().orc_spmv(n, _p(rp), _p(ci), _p(va), _p(x), _p(y))
    return y


def tri_jacobi(T, r, k, lower=True, unit=False, bounds=None):
    """k inner Jacobi sweeps on the lower/upper triangle of T from D^{-1} r."""
    n, rp, ci, va = _csr(T)
    nb, bd = _part(bounds)
    r = _f64(r)
    g = np.empty(n)
    _check(_L().orc_tri_jacobi(n, _p(rp), _p(ci), _p(va), int(lower), int(unit), _p(r), int(k), nb, _p(bd), _p(g)),
           "tri_jacobi")
    return g


def tri_direct(T, r, lower=True, unit=False, bounds=None):
    n, rp, ci, va = _csr(T)
    nb, bd = _part(bounds)
    r = _f64(r)
    y = np.empty(n)
    _check(_L().orc_tri_direct(n, _p(rp), _p(ci), _p(va), int(lower), int(unit), _p(r), nb, _p(bd), _p(y)),
           "tri_direct")
    return y


def pgs_apply(A, b, x, k, nu=1, x_is_zero=False, bounds=None):
    """Returns the new x (input x is not modified)."""
    n, rp, ci, va = _csr(A)
    nb, bd = _part(bounds)
    b = _f64(b)
    x = np.array(x, dtype=np.float64, copy=True)
    _check(_L().orc_pgs_apply(n, _p(rp), _p(ci), _p(va), _p(b), _p(x), int(k), int(nu), int(x_is_zero), nb, _p(bd)),
           "pgs_apply")
    return x


def pgs_backward_apply(A, b, x, k, nu=1, x_is_zero=False, bounds=None):
    """Backward pGS (M = D + U); returns the new x."""
    n, rp, ci, va = _csr(A)
    nb, bd = _part(bounds)
    b = _f64(b)
    x = np.array(x, dtype=np.float64, copy=True)
    _check(_L().orc_pgs_backward_apply(n, _p(rp), _p(ci), _p(va), _p(b), _p(x), int(k), int(nu), int(x_is_zero),
                                       nb, _p(bd)), "pgs_backward_apply")
    return x


def pgs_symmetric_apply(A, b, x, k, nu=1, x_is_zero=False, bounds=None):
    """nu x (forward pGS, then backward pGS)."""
    x = np.array(x, dtype=np.float64, copy=True)
    for it in range(nu):
        x = pgs_apply(A, b, x, k, x_is_zero=x_is_zero and it == 0, bounds=bounds)
        x = pgs_backward_apply(A, b, x, k, bounds=bounds)
    return x


def l1_jacobi_apply(A, b, x, nu=1, x_is_zero=False):
    n, rp, ci, va = _csr(A)
    b = _f64(b)
    x = np.array(x, dtype=np.float64, copy=True)
    _check(_L().orc_l1_jacobi_apply(n, _p(rp), _p(ci), _p(va), _p(b), _p(x), int(nu), int(x_is_zero)),
           "l1_jacobi_apply")
    return x


def gs_apply(A, b, x, nu=1, bounds=None):
    n, rp, ci, va = _csr(A)
    nb, bd = _part(bounds)
    b = _f64(b)
    x = np.array(x, dtype=np.float64, copy=True)
    _check(_L().orc_gs_apply(n, _p(rp), _p(ci), _p(va), _p(b), _p(x), int(nu), nb, _p(bd)), "gs_apply")
    return x


def ilu0(A):
    """ILU(0) factor values on the pattern of A (strict lower = L_s, upper incl.
    diagonal = U).  Returns (rowptr, col, val) sharing A's pattern."""
    n, rp, ci, va = _csr(A)
    w = np.empty_like(va)
    _check(_L().orc_ilu0(n, _p(rp), _p(ci), _p(va), _p(w)), "ilu0")
    return rp, ci, w


def ilu0_fixed_point(A, sweeps):
    """Chow-Patel fixed-point ILU(0) after `sweeps` synchronous sweeps (reading
    R19); (rowptr, col, val) on A's pattern, the ilu0 layout."""
    n, rp, ci, va = _csr(A)
    w = np.empty_like(va)
    _check(_L().orc_ilu0_fixed_point(n, _p(rp), _p(ci), _p(va), int(sweeps), _p(w)), "ilu0_fixed_point")
    return rp, ci, w


def ilu_apply(A, F, b, x, kL, kU, nu=1, x_is_zero=False, direct=False, bounds=None):
    """F = (rowptr, col, val) of the factors (ilu0 output)."""
    n, rp, ci, va = _csr(A)
    frp, fci, fva = (np.ascontiguousarray(F[0], np.int64), np.ascontiguousarray(F[1], np.int64), _f64(F[2]))
    nb, bd = _part(bounds)
    b = _f64(b)
    x = np.array(x, dtype=np.float64, copy=True)
    _check(_L().orc_ilu_apply(n, _p(rp), _p(ci), _p(va), _p(frp), _p(fci), _p(fva), _p(b), _p(x),
                              int(kL), int(kU), int(nu), int(x_is_zero), int(direct), nb, _p(bd)), "ilu_apply")
    return x


def block_ilu0(A, bounds):
    """ILU(0) of the block-diagonal part of A under a row partition (HYBRID
    ILU, reading R5): factor of each diagonal block A_pp, off-block entries of
    the returned pattern carry 0 and are ignored by ilu_apply(bounds=...)."""
    n, rp, ci, va = _csr(A)
    b = np.asarray(bounds, dtype=np.int64)
    own = np.searchsorted(b, np.arange(n), side="right") - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    keep = own[rows] == own[ci]
    import scipy.sparse as sp
    Ab = sp.csr_matrix((va[keep], ci[keep], np.concatenate([[0], np.cumsum(np.bincount(rows[keep], minlength=n))])),
                       shape=(n, n))
    return ilu0(Ab)
