"""The generators' symmetry flag (inputs.CSR.symmetric, metadata bench.py
uses to count the symmetric residual's bytes) against an exhaustive bitwise
check, and bench.py's mirror of the transpose-map decision on small grids."""
import numpy as np

import bench
import inputs


def bitwise_symmetric(A):
    B = inputs.CSR(A.nrows, A.ncols, A.rowptr, A.col, A.val, A.row_begin)   # symmetric unknown: checked
    return bench.symmetric_local(B)


def test_generator_flags_are_true():
    for A in (inputs.var27(9), inputs.var27_grid(13, 7, 5), inputs.laplace(11, 7, 5), inputs.laplace(9, 8)):
        assert A.symmetric is True
        assert bitwise_symmetric(A)


def test_row_blocks_of_symmetric_grids_are_locally_symmetric():
    for r0, r1 in ((0, 150), (91, 400), (300, 455)):
        A = inputs.var27_grid(13, 7, 5, r0, r1)
        assert A.symmetric and bitwise_symmetric(A)


def test_check_detects_one_ulp_and_signed_zero():
    A = inputs.var27(6)
    i = 40
    p = A.rowptr[i] + int(np.flatnonzero(A.col[A.rowptr[i]:A.rowptr[i + 1]] == i + 1)[0])
    v = A.val.copy()
    v[p] = np.nextafter(v[p], 0.0)
    assert not bitwise_symmetric(inputs.CSR(A.nrows, A.ncols, A.rowptr, A.col, v))
    q = A.rowptr[i + 1] + int(np.flatnonzero(A.col[A.rowptr[i + 1]:A.rowptr[i + 2]] == i)[0])
    v = A.val.copy()
    v[p], v[q] = 0.0, -0.0
    assert not bitwise_symmetric(inputs.CSR(A.nrows, A.ncols, A.rowptr, A.col, v))


def test_nonsymmetric_generator_is_detected():
    assert not bitwise_symmetric(inputs.convdiff(6))


def test_transpose_map_mirror():
    """27-point grids with 256-row tiles get a map; 7-point grids have no
    residual window (too few gathers per window value); a nonsymmetric matrix
    has none."""
    assert bench.aligned_parts(inputs.var27(40))["Ut"]
    assert bench.aligned_parts(inputs.var27_grid(130, 20, 6))["Ut"]
    assert not bench.aligned_parts(inputs.laplace(64, 16, 8))["Ut"]
    assert not bench.aligned_parts(inputs.convdiff(12))["Ut"]


def test_byte_model_counts_the_map():
    n, nl, nu = 1000, 13000, 13000
    plain = bench.algorithmic_bytes("pgs", n, nl + nu, nl, nu, 2, 0, 0, {"L": True, "U": True})
    sym = bench.algorithmic_bytes("pgs", n, nl + nu, nl, nu, 2, 0, 0, {"L": True, "U": True, "Ut": True})
    assert plain["residual"] - sym["residual"] == (8 * nu + (nu + 31) // 32 * 4) - (nu + 31) // 32 * 20
    assert plain["sweeps"] == sym["sweeps"]
