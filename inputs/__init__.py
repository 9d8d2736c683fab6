"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and
bench.py (SURVEY.md §8(d) "Synthetic inputs"; DESIGN.md §3 "Input recipe").

This module holds none of the method's arithmetic: it assembles stencil
matrices shaped like the paper's workloads (§6), draws
counter-based random vectors keyed by (seed, global row), and computes the RCM
ordering used as preprocessing.  Both the oracle side and the
CUDA side read what it produces; neither is imported here.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libnsm_inputs.so")
_lib = None

SEED_B, SEED_X0, SEED_FIELD = 0, 1, 2   # b seed 0, x0 seed 1, coefficients seed 2


def build(force: bool = False) -> str:
    """Compile gen.c into libnsm_inputs.so (plain gcc, host only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i64, dbl, u64, vp = ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, ctypes.c_void_p
        _lib.gen_uniform.argtypes = [u64, i64, i64, dbl, dbl, vp]
        _lib.gen_uniform_int.argtypes = [u64, i64, i64, ctypes.c_int, vp]
        _lib.gen_kappa_field.argtypes = [i64, i64, i64, u64, dbl, vp]
        _lib.gen_lap_nnz.argtypes = [i64, i64, i64, ctypes.c_int, i64, i64]
        _lib.gen_lap_nnz.restype = i64
        _lib.gen_lap_fill.argtypes = [i64, i64, i64, ctypes.c_int, i64, i64, vp, vp, vp]
        _lib.gen_var27_nnz.argtypes = [i64, i64, i64, i64, i64]
        _lib.gen_var27_nnz.restype = i64
        _lib.gen_var27_fill.argtypes = [i64, i64, i64, vp, i64, i64, vp, vp, vp]
        _lib.gen_cd_velocity.argtypes = [u64, dbl, vp]
        _lib.gen_cd_nnz.argtypes = [i64, i64, i64, i64, i64]
        _lib.gen_cd_nnz.restype = i64
        _lib.gen_cd_fill.argtypes = [i64, i64, i64, vp, vp, i64, i64, vp, vp, vp]
        _lib.gen_rcm.argtypes = [i64, vp, vp, vp]
        _lib.gen_permute.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp]
        _lib.gen_bandwidth.argtypes = [i64, vp, vp]
        _lib.gen_bandwidth.restype = i64
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass
class CSR:
    """Host CSR block of rows [row_begin, row_begin + nrows) of an ncols-column
    matrix; int64 rowptr (starting at 0) and GLOBAL int64 column ids."""
    nrows: int
    ncols: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    row_begin: int = 0

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.rowptr), shape=(self.nrows, self.ncols))

    @staticmethod
    def from_scipy(m, row_begin: int = 0) -> "CSR":
        m = m.tocsr()
        m.sort_indices()
        return CSR(m.shape[0], m.shape[1], m.indptr.astype(np.int64), m.indices.astype(np.int64),
                   m.data.astype(np.float64), row_begin)

    def rows(self, r0: int, r1: int) -> "CSR":
        """Rows [r0, r1) (local indices) as a new CSR block."""
        a, b = int(self.rowptr[r0]), int(self.rowptr[r1])
        return CSR(r1 - r0, self.ncols, (self.rowptr[r0:r1 + 1] - a).copy(), self.col[a:b].copy(),
                   self.val[a:b].copy(), self.row_begin + r0)


# ------------------------------------------------------------------ vectors --
def uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0, idx0: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _L().gen_uniform(seed, idx0, n, lo, hi, _p(out))
    return out


def uniform_int(seed: int, n: int, bits: int = 20, idx0: int = 0) -> np.ndarray:
    """Integers uniform in [-2^bits, 2^bits) stored as float64 (exact)."""
    out = np.empty(n, dtype=np.float64)
    _L().gen_uniform_int(seed, idx0, n, bits, _p(out))
    return out


# ----------------------------------------------------------------- matrices --
def _fill(nnz_fn, fill_fn, nrows, ncols, row_begin, *args) -> CSR:
    nnz = nnz_fn()
    rp = np.empty(nrows + 1, dtype=np.int64)
    ci = np.empty(nnz, dtype=np.int64)
    va = np.empty(nnz, dtype=np.float64)
    fill_fn(rp, ci, va)
    return CSR(nrows, ncols, rp, ci, va, row_begin)


def laplace(nx: int, ny: int, nz: int = 1, r0: int = 0, r1: int | None = None) -> CSR:
    """Dirichlet Laplacian: 2-D 5-point (nz == 1; stencil 4, -1) or 3-D 7-point
    (stencil 6, -1), rows [r0, r1) of the lexicographic (x fastest) ordering."""
    n = nx * ny * nz
    r1 = n if r1 is None else r1
    dim = 2 if nz == 1 else 3
    L = _L()
    return _fill(lambda: L.gen_lap_nnz(nx, ny, nz, dim, r0, r1),
                 lambda rp, ci, va: L.gen_lap_fill(nx, ny, nz, dim, r0, r1, _p(rp), _p(ci), _p(va)),
                 r1 - r0, n, r0)


def kappa_field(nx: int, ny: int, nz: int, seed: int = SEED_FIELD, contrast: float = 1e4) -> np.ndarray:
    k = np.empty(nx * ny * nz, dtype=np.float64)
    if _L().gen_kappa_field(nx, ny, nz, seed, contrast, _p(k)) != 0:
        raise MemoryError("gen_kappa_field")
    return k


def var27(N: int, seed: int = SEED_FIELD, contrast: float = 1e4, r0: int = 0, r1: int | None = None) -> CSR:
    """27-point variable-coefficient pressure matrix on N^3 (Nalu-Wind shaped, C3)."""
    n = N ** 3
    r1 = n if r1 is None else r1
    kap = kappa_field(N, N, N, seed, contrast)
    L = _L()
    return _fill(lambda: L.gen_var27_nnz(N, N, N, r0, r1),
                 lambda rp, ci, va: L.gen_var27_fill(N, N, N, _p(kap), r0, r1, _p(rp), _p(ci), _p(va)),
                 r1 - r0, n, r0)


def var27_grid(nx: int, ny: int, nz: int, r0: int = 0, r1: int | None = None, seed: int = SEED_FIELD,
               contrast: float = 1e4) -> CSR:
    """Rows [r0, r1) of the 27-point pressure matrix on an nx x ny x nz grid
    (the C3 recipe; var27(N) is var27_grid(N, N, N))."""
    n = nx * ny * nz
    r1 = n if r1 is None else r1
    kap = kappa_field(nx, ny, nz, seed, contrast)
    L = _L()
    return _fill(lambda: L.gen_var27_nnz(nx, ny, nz, r0, r1),
                 lambda rp, ci, va: L.gen_var27_fill(nx, ny, nz, _p(kap), r0, r1, _p(rp), _p(ci), _p(va)),
                 r1 - r0, n, r0)


def var27_slab(N: int, nranks: int, rank: int) -> CSR:
    """Weak-scaled C3: the 27-point pressure matrix on the global
    N x N x (N * nranks) grid (one coefficient field over the whole grid);
    rank p owns the z-slab of rows [p N^3, (p+1) N^3).  nranks == 1 is C3."""
    n_loc = N ** 3
    return var27_grid(N, N, N * nranks, rank * n_loc, (rank + 1) * n_loc)


def rcm_order(A: CSR) -> np.ndarray:
    order = np.empty(A.nrows, dtype=np.int64)
    rc = _L().gen_rcm(A.nrows, _p(A.rowptr), _p(A.col), _p(order))
    if rc != 0:
        raise RuntimeError(f"gen_rcm failed ({rc})")
    return order


def permute(A: CSR, order: np.ndarray) -> CSR:
    """B = A(order, order), i.e. b_{k,m} = a_{order[k], order[m]}."""
    rp = np.empty(A.nrows + 1, dtype=np.int64)
    ci = np.empty(A.nnz, dtype=np.int64)
    va = np.empty(A.nnz, dtype=np.float64)
    order = np.ascontiguousarray(order, dtype=np.int64)
    if _L().gen_permute(A.nrows, _p(A.rowptr), _p(A.col), _p(A.val), _p(order), _p(rp), _p(ci), _p(va)) != 0:
        raise MemoryError("gen_permute")
    return CSR(A.nrows, A.ncols, rp, ci, va, 0)


def bandwidth(A: CSR) -> int:
    return int(_L().gen_bandwidth(A.nrows, _p(A.rowptr), _p(A.col)))


def convdiff(N: int, seed: int = SEED_FIELD, contrast: float = 1e3, rcm: bool = True) -> CSR:
    """Nonsymmetric upwind convection-diffusion on N^3 (PeleLM shaped, C4),
    optionally RCM-reordered (P:L942 'symrcm')."""
    n = N ** 3
    kap = kappa_field(N, N, N, seed, contrast)
    v = np.empty(3, dtype=np.float64)
    L = _L()
    L.gen_cd_velocity(seed, contrast, _p(v))
    A = _fill(lambda: L.gen_cd_nnz(N, N, N, 0, n),
              lambda rp, ci, va: L.gen_cd_fill(N, N, N, _p(kap), _p(v), 0, n, _p(rp), _p(ci), _p(va)),
              n, n, 0)
    if rcm:
        A = permute(A, rcm_order(A))
    return A


def weak_slab(N: int, nranks: int, rank: int) -> CSR:
    """Config C5: 7-point Laplacian on the global N x N x (N * nranks) grid;
    rank p owns the z-slab of rows [p N^3, (p+1) N^3) (global column ids)."""
    n_loc = N ** 3
    return laplace(N, N, N * nranks, rank * n_loc, (rank + 1) * n_loc)


def random_dense(n: int, seed: int, density: float = 1.0, diag_shift: float = 2.0) -> CSR:
    """Tiny random matrix (pins on n <= 8): entries U[-1,1) with the given
    pattern density, diagonal shifted away from zero."""
    rng = np.random.default_rng(seed)
    M = rng.uniform(-1.0, 1.0, (n, n))
    if density < 1.0:
        M *= rng.uniform(0, 1, (n, n)) < density
    M[np.arange(n), np.arange(n)] = diag_shift + rng.uniform(0, 1, n)
    import scipy.sparse as sp
    return CSR.from_scipy(sp.csr_matrix(M))


# ------------------------------------------------------------------ configs --
CONFIGS = {
    "C1": "2D 5-point Poisson 64x64 (4096 rows), poly-GS k=1..3 vs direct forward substitution, fp64",
    "C2": "3D 7-point Laplacian 128^3, ILU(0) factors, Jacobi-iterated L and U solves (k=2)",
    "C3": "3D 27-point variable-coefficient pressure matrix 256^3 (Nalu-Wind-shaped), pGS",
    "C4": "nonsymmetric convection-diffusion 256^3 (PeleLM-shaped) + RCM, ILU(0) Jacobi solves",
    "C5": "weak-scaled 7-point Laplacian 256^3 rows per GPU, row-block partition + halo exchange",
}


def config_matrix(name: str, scale: int | None = None, nranks: int = 1, rank: int = 0) -> CSR:
    """Matrix of a BASELINE.json config; `scale` overrides the grid edge N for
    reduced-size parity cases (same generator, same recipe)."""
    if name == "C1":
        N = scale or 64
        return laplace(N, N, 1)
    if name == "C2":
        N = scale or 128
        return laplace(N, N, N)
    if name == "C3":
        return var27_slab(scale or 256, nranks, rank)
    if name == "C4":
        return convdiff(scale or 256)
    if name == "C5":
        return weak_slab(scale or 256, nranks, rank)
    raise KeyError(name)
