"""GPU Chow-Patel fixed-point ILU(0) (nsm_ilu0_fixed_point, reading R19)
against the oracle's sweeps, through the C-ABI (-m gpu).  Both form every
entry with the same IEEE operations in the same order, so the comparison is
bit for bit at every sweep count; converged, it is the host ILU(0)."""
import numpy as np
import pytest
import scipy.sparse as sp

import inputs
import oracle
import paper_2112_14681_b200 as nsm

pytestmark = pytest.mark.gpu


def random_sparse_dd(n, seed, per_row=6):
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n), per_row)
    cols = rng.integers(0, n, size=n * per_row)
    M = sp.csr_matrix((rng.uniform(-1, 1, size=n * per_row), (rows, cols)), shape=(n, n))
    M.setdiag(0)
    M.eliminate_zeros()
    M = M + sp.diags(np.abs(M).sum(1).A1 + 1.0)
    return inputs.CSR.from_scipy(M.tocsr())


MATS = {
    "lap2d": lambda: inputs.laplace(31, 17, 1),
    "lap3d_ragged": lambda: inputs.laplace(13, 11, 7),
    "var27": lambda: inputs.var27(9),
    "cd_rcm": lambda: inputs.convdiff(10),
    "random": lambda: random_sparse_dd(997, 5),
}


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("sweeps", [0, 1, 2, 5, 17])
def test_sweeps_bitwise(name, sweeps):
    A = MATS[name]()
    want = oracle.ilu0_fixed_point(A, sweeps)[2]
    got = nsm.ilu0_fixed_point(A, sweeps)
    assert np.array_equal(got, want), f"{name} sweeps={sweeps}: {np.sum(got != want)} entries differ"


@pytest.mark.parametrize("name", ["lap2d", "cd_rcm"])
def test_converged_equals_host_ilu0(name):
    """Enough sweeps (>= the dependency depth, at most nnz) reproduce the host
    IKJ factorisation nsm_ilu0 exactly; the factors then drive the smoother."""
    A = MATS[name]()
    host = nsm.ilu0(A)
    sweeps = 1
    while True:
        got = nsm.ilu0_fixed_point(A, sweeps)
        if np.array_equal(got, host):
            break
        assert sweeps < 4 * A.nrows, "did not converge"
        sweeps *= 2
    assert np.array_equal(got, oracle.ilu0(A)[2])


def test_block_partition_matches_host():
    """row_begin: the factorisation of the local diagonal block A_pp (HYBRID
    reading R5), off-block entries 0 — the layout of nsm_ilu0."""
    N = 8
    A = inputs.laplace(N, N, 2 * N, N ** 3, 2 * N ** 3)   # rank 1 of 2 z-slabs
    host = nsm.ilu0(A, row_begin=A.row_begin)
    got = nsm.ilu0_fixed_point(A, 4 * N ** 3, row_begin=A.row_begin)
    assert np.array_equal(got, host)


def test_zero_diagonal_error():
    Z = inputs.CSR.from_scipy(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 1.0]])))
    with pytest.raises(nsm.NsmError) as e:
        nsm.ilu0_fixed_point(Z, 2)
    assert e.value.name == "NSM_ERR_ZERO_DIAG"


@pytest.mark.slow
def test_full_size_c2_three_sweeps():
    """BASELINE config C2 (128^3): three sweeps, the whole factor vs oracle."""
    A = inputs.config_matrix("C2")
    want = oracle.ilu0_fixed_point(A, 3)[2]
    got = nsm.ilu0_fixed_point(A, 3)
    assert np.array_equal(got, want)
