"""The device-side split / SELL-32 builder (nsm_setup_device, builder_gpu.cu;
SURVEY.md §8(f) NEXT-4) against the host builder (nsm_setup,
builder.cpp): every device array of the handle identical entry by entry, and
the smoothers on top of it bit-identical to the oracle (-m gpu)."""
import time

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import inputs
import oracle
import paper_2112_14681_b200 as nsm

pytestmark = pytest.mark.gpu


def random_sparse(n, seed, avg=9, maxrow=70):
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(n):
        m = int(min(maxrow, rng.geometric(1.0 / avg)))
        c = rng.choice(n, size=min(m, n), replace=False)
        rows += [i] * len(c)
        cols += list(c)
    M = sp.csr_matrix((rng.uniform(-1, 1, len(rows)), (rows, cols)), shape=(n, n))
    M = M + sp.diags(np.abs(M).sum(1).A1 + 1.0)
    return inputs.CSR.from_scipy(M)


MATS = {
    "C1": lambda: inputs.config_matrix("C1"),
    "lap3d_ragged": lambda: inputs.laplace(13, 11, 7),
    "var27_9": lambda: inputs.var27(9),
    "cd_rcm_10": lambda: inputs.convdiff(10),            # RCM: compact layout
    "random_irregular": lambda: random_sparse(997, 5),   # scattered: compact layout
    "lap_aligned_ragged": lambda: inputs.laplace(100, 9, 3),
    "var27_aligned_40": lambda: inputs.var27(40),
    "n1": lambda: inputs.CSR.from_scipy(sp.csr_matrix(np.array([[3.0]]))),
    "diagonal": lambda: inputs.CSR.from_scipy(sp.diags(np.arange(1.0, 100.0)).tocsr()),
    "dense40": lambda: inputs.random_dense(40, 3),
}


def device_csr(A, fval=None):
    rp = torch.from_numpy(np.ascontiguousarray(A.rowptr, np.int64)).cuda()
    ci = torch.from_numpy(np.ascontiguousarray(A.col, np.int64)).cuda()
    va = torch.from_numpy(np.ascontiguousarray(A.val, np.float64)).cuda()
    fv = torch.from_numpy(np.ascontiguousarray(fval, np.float64)).cuda() if fval is not None else None
    return rp, ci, va, fv


def assert_same_handles(Sh, Sd, nparts):
    for p in range(nparts):
        a, b = Sh.part(p), Sd.part(p)
        for k in ("ptr", "col", "val", "off"):
            assert np.array_equal(a[k], b[k]), (p, k)
        assert (a["nnz"], a["maxw"], a["aligned"]) == (b["nnz"], b["maxw"], b["aligned"]), p
    for w in ((0, 1, 2) if nparts > 4 else (0, 1)):
        assert np.array_equal(Sh.diag(w), Sd.diag(w)), w


@pytest.mark.parametrize("name", list(MATS))
def test_device_builder_matches_host(name):
    A = MATS[name]()
    F = oracle.ilu0(A)[2]
    with nsm.Smoother(A, F) as Sh:
        Sd = nsm.Smoother.from_device_csr(*device_csr(A, F))
        try:
            assert_same_handles(Sh, Sd, 8)
            assert (Sd.n, Sd.nnz_offdiag, Sd.layout()) == (Sh.n, Sh.nnz_offdiag, Sh.layout())
            # the smoothers on the device-built handle: bit-identical to the oracle
            b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
            for kind, want in (("pgs", oracle.pgs_apply(A, b, x0, 2)),
                               ("ilu", oracle.ilu_apply(A, (A.rowptr, A.col, F), b, x0, 2, 2))):
                x = torch.from_numpy(x0.copy()).cuda()
                Sd.smooth(torch.from_numpy(b).cuda(), x, kind, nu=1, k_l=2, k_u=2)
                assert np.array_equal(x.cpu().numpy(), want), (name, kind)
            Sd.check()
        finally:
            Sd.close()


def test_device_builder_without_factor():
    A = inputs.var27(12)
    with nsm.Smoother(A) as Sh:
        Sd = nsm.Smoother.from_device_csr(*device_csr(A)[:3])
        try:
            assert_same_handles(Sh, Sd, 4)
        finally:
            Sd.close()


def test_device_builder_errors():
    """The host builder's errors, with the first offending row."""
    A = inputs.laplace(6, 6, 6).to_scipy().tolil()
    A[77, 77] = 0.0
    A = inputs.CSR.from_scipy(A.tocsr())
    A.val[A.rowptr[77]:A.rowptr[78]][A.col[A.rowptr[77]:A.rowptr[78]] == 77] = 0.0
    with pytest.raises(nsm.NsmError) as e:
        nsm.Smoother.from_device_csr(*device_csr(A)[:3])
    assert e.value.name == "NSM_ERR_ZERO_DIAG" and "row 77" in str(e.value)
    B = inputs.laplace(6, 6, 6)
    c = B.col.copy()
    r0 = B.rowptr[100]
    c[r0], c[r0 + 1] = c[r0 + 1], c[r0]          # unsorted row 100
    B = inputs.CSR(B.nrows, B.ncols, B.rowptr, c, B.val)
    with pytest.raises(nsm.NsmError) as e:
        nsm.Smoother.from_device_csr(*device_csr(B)[:3])
    assert e.value.name == "NSM_ERR_PATTERN" and "row 100" in str(e.value)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_device_builder_full_size(cfg):
    """Full BASELINE sizes: identical arrays; set-up times of both builders
    (host: nsm_setup incl. upload; device: nsm_setup_device from a device CSR
    already resident) are printed for profiles/."""
    A = inputs.config_matrix(cfg)
    F = oracle.ilu0(A)[2] if cfg == "C4" else None
    dev = device_csr(A, F)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Sh = nsm.Smoother(A, F)
    t_host = time.perf_counter() - t0
    t0 = time.perf_counter()
    Sd = nsm.Smoother.from_device_csr(*dev)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    try:
        assert_same_handles(Sh, Sd, 8 if F is not None else 4)
        print(f"{cfg}: n={A.nrows} nnz={A.nnz} host set-up {t_host:.3f} s, device set-up {t_dev:.3f} s")
    finally:
        Sd.close()
        Sh.close()
