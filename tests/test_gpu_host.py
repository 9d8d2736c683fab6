"""nsm_smooth_host (the end-to-end C-ABI call on host vectors): bit-identical
to nsm_smooth on device vectors, for pageable numpy and pinned CPU tensors,
with and without x_is_zero; argument errors."""
import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _smoother(A, F=None):
    import paper_2112_14681_b200 as nsm
    return nsm.Smoother(A, F, device=0)


@pytest.mark.parametrize("kind", ["pgs", "ilu", "pgs_symmetric"])
@pytest.mark.parametrize("host", ["numpy", "pinned"])
@pytest.mark.parametrize("x_is_zero", [False, True])
def test_smooth_host_matches_device(kind, host, x_is_zero):
    A = inputs.laplace(20, 13, 7)  # 1820 rows: a ragged last slice
    F = oracle.ilu0(A)[2] if kind == "ilu" else None
    b, x0 = inputs.uniform(3, A.nrows), inputs.uniform(4, A.nrows)
    with _smoother(A, F) as S:
        xd = torch.from_numpy(x0.copy()).cuda()
        S.smooth(torch.from_numpy(b).cuda(), xd, kind, nu=2, k_l=2, k_u=3, x_is_zero=x_is_zero)
        want = xd.cpu().numpy()
        if host == "numpy":
            bh, xh = b.copy(), x0.copy()
        else:
            bh = torch.from_numpy(b).pin_memory()
            xh = torch.from_numpy(x0.copy()).pin_memory()
        for _ in range(2):  # the second call reuses the staging vectors
            xs = xh.copy() if host == "numpy" else xh.clone().pin_memory()
            S.smooth_host(bh, xs, kind, nu=2, k_l=2, k_u=3, x_is_zero=x_is_zero)
            got = xs if host == "numpy" else xs.numpy()
            assert np.array_equal(got, want)
        # out-of-place: x_in untouched, the result in out
        xin = xh.copy() if host == "numpy" else xh.clone().pin_memory()
        out = np.empty_like(x0) if host == "numpy" else torch.empty(A.nrows, dtype=torch.float64).pin_memory()
        S.smooth_host(bh, xin, kind, nu=2, k_l=2, k_u=3, x_is_zero=x_is_zero, out=out)
        assert np.array_equal(out if host == "numpy" else out.numpy(), want)
        assert np.array_equal(xin if host == "numpy" else xin.numpy(), x0)
        # b is untouched
        assert np.array_equal(bh if host == "numpy" else bh.numpy(), b)
        # and against the oracle (one more, independent check of the path)
        if kind == "pgs" and not x_is_zero:
            ref = oracle.pgs_apply(A, b, oracle.pgs_apply(A, b, x0, 2), 2)
            np.testing.assert_allclose(got, ref, rtol=1e-13, atol=0)


def test_smooth_host_errors():
    import paper_2112_14681_b200 as nsm
    A = inputs.laplace(8, 8, 2)
    b = inputs.uniform(0, A.nrows)
    with _smoother(A) as S:
        with pytest.raises(TypeError):
            S.smooth_host(b.astype(np.float32), b.copy())
        with pytest.raises(TypeError):
            S.smooth_host(b, torch.zeros(A.nrows, dtype=torch.float64, device="cuda"))
        with pytest.raises(nsm.NsmError):
            S.smooth_host(b, b)  # aliased
        with pytest.raises(nsm.NsmError):
            y = np.zeros(A.nrows + 1)
            S.smooth_host(b, y[:-1], out=y[1:])  # partial overlap of x_in and out
        with pytest.raises(nsm.NsmError):
            S.smooth_host(b, b.copy(), "ilu")  # no factors on this handle


def test_smooth_host_nu_zero():
    """nu = 0: no application, the result is the start vector (x_in, or zeros
    with x_is_zero) — never the staging buffer's stale contents."""
    A = inputs.laplace(8, 8, 2)
    b = inputs.uniform(0, A.nrows)
    x0 = inputs.uniform(1, A.nrows)
    with _smoother(A) as S:
        out = np.full(A.nrows, 7.0)
        S.smooth_host(b, x0.copy(), nu=1, out=out)              # fills the staging vectors
        out2 = np.full(A.nrows, 7.0)
        S.smooth_host(b, x0, nu=0, x_is_zero=True, out=out2)
        assert np.array_equal(out2, np.zeros(A.nrows))
        out3 = np.full(A.nrows, 7.0)
        S.smooth_host(b, x0, nu=0, out=out3)
        assert np.array_equal(out3, x0)


def _wide_band(n=100_000, w=20_000, seed=3):
    """A matrix whose bandwidth (20,000 rows) exceeds n / 32: the chunk length
    follows the bandwidth, not the chunk count (a CPU model of the chunk
    schedule with chunks shorter than the bandwidth gives a wrong x)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    offs = [-w, -1, 1, w]
    diags = [rng.uniform(-1, 1, n - abs(o)) for o in offs]
    M = sp.diags(diags, offs, shape=(n, n), format="csr")
    M = M + sp.diags(np.abs(M).sum(1).A1 + 1.0)
    return inputs.CSR.from_scipy(M.tocsr())


@pytest.mark.parametrize("mat", ["var27_64", "lap_96", "cd_rcm_40", "wide_band"])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_smooth_host_chunked_matches_device(mat, k):
    """nsm_smooth_host in row chunks (copies overlapped with the passes,
    NSM_OPT_HOST_CHUNKS, the default) is bit-identical to the device call and
    to the unchunked host call; pinned host vectors."""
    A = {"var27_64": lambda: inputs.var27(64), "lap_96": lambda: inputs.laplace(96, 96, 96),
         "cd_rcm_40": lambda: inputs.convdiff(40), "wide_band": _wide_band}[mat]()
    b = torch.from_numpy(inputs.uniform(0, A.nrows)).pin_memory()
    x0 = torch.from_numpy(inputs.uniform(1, A.nrows)).pin_memory()
    with _smoother(A) as S:
        xd = x0.cuda()
        S.smooth(b.cuda(), xd, "pgs", nu=1, k_l=k)
        want = xd.cpu().numpy()
        out = torch.empty_like(x0).pin_memory()
        l0 = S.stats()[0]
        S.smooth_host(b, x0, "pgs", nu=1, k_l=k, out=out)
        assert S.stats()[0] - l0 > 2 * (k + 1), "the chunked path did not run"   # (k + 1) launches per chunk
        assert np.array_equal(out.numpy(), want), f"{mat} k={k} chunked"
        # a pageable result buffer: the chunked path copies x back instead of
        # writing it over PCIe from the last sweep
        outp = np.full(A.nrows, 7.0)
        S.smooth_host(b, x0, "pgs", nu=1, k_l=k, out=outp)
        assert np.array_equal(outp, want), f"{mat} k={k} chunked, pageable out"
        S.set_host_chunks(False)
        out2 = torch.empty_like(x0).pin_memory()
        S.smooth_host(b, x0, "pgs", nu=1, k_l=k, out=out2)
        assert np.array_equal(out2.numpy(), want)
        assert np.array_equal(x0.numpy(), inputs.uniform(1, A.nrows))   # x_in untouched
        S.check()
