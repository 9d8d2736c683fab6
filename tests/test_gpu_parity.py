"""Parity of the CUDA path (through the C-ABI) with the CPU oracle on the same
seeded inputs (-m gpu).

Bar (BASELINE.json north_star): normwise relative error <= 1e-12 per smoother
application.  Because the kernels reproduce the oracle's rounding sequence
(per-row ascending sums, no FMA, IEEE division — DESIGN.md R10), the tests
also assert bit-for-bit equality; the 1e-12 check is the contract, the
bitwise check guards the design claim.
"""
import numpy as np
import pytest
import scipy.sparse as sp
import torch

import inputs
import oracle
import paper_2112_14681_b200 as nsm

pytestmark = pytest.mark.gpu
TOL = 1e-12


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def start(x0, xz):
    """Device start vector; with x_is_zero its contents must be ignored, so
    hand the library NaNs (the oracle gets the zeros)."""
    return torch.full((len(x0),), float("nan"), dtype=torch.float64, device="cuda") if xz else dev(x0)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def relerr(got, want):
    nw = np.linalg.norm(want)
    return np.linalg.norm(got - want) / (nw if nw > 0 else 1.0)


def agree(got, want, what=""):
    e = relerr(got, want)
    assert e <= TOL, f"{what}: relerr {e:.3e}"
    nbad = int(np.sum(got != want))
    assert nbad == 0, f"{what}: {nbad} of {len(want)} entries differ (relerr {e:.2e})"


def random_sparse(n, seed, avg=9, maxrow=70):
    """Irregular rows (lengths 1 .. maxrow): exercises SELL padding."""
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


SMALL = {
    "C1": lambda: inputs.config_matrix("C1"),
    "lap3d_ragged": lambda: inputs.laplace(13, 11, 7),           # n = 1001
    "var27_9": lambda: inputs.var27(9),
    "cd_rcm_10": lambda: inputs.convdiff(10),
    "random_irregular": lambda: random_sparse(997, 5),
    # offset-aligned layout (nsm_layout): stencil rows, ragged tail / 27-point
    "lap_aligned_ragged": lambda: inputs.laplace(100, 9, 3),
    "var27_aligned_40": lambda: inputs.var27(40),
}


KERNELS = ("fused", "fusedw1", "onepass", "onepassw1", "coupled", "coupledlag", "pipelined", "nowindow", "plain")


def set_kernels(S, mode):
    """fused: phase-skewed fused passes wherever possible (pGS one pass, ILU
    two) + pipelined kernels; fusedw1: the same with wait distance 1 (every
    item waits for its predecessor, rings wrap after a few tiles: stresses the
    synchronisation); pipelined: one cp.async.bulk pipelined kernel per pass,
    gathering from shared-memory windows where the layout allows (the
    default); nowindow: the same gathering through L1/L2; plain:
    register-blocked; onepass(w1): the one-pass windowed pGS (NSM_OPT_FUSED = 3)
    where the matrix allows it, else as fused (w1: skew margin 1); coupled: the
    k = 2, 3 sweeps of a forward pGS application on windowed matrices as
    concurrent CTA groups of one kernel (NSM_OPT_COUPLED), the rest pipelined;
    coupledlag: the same at throttle distance 2 (group 0 waits for the last
    sweep group almost every tile: stresses the synchronisation)."""
    S.set_coupled(1 if mode == "coupled" else (2 if mode == "coupledlag" else 0))
    S.set_pipeline(mode != "plain")
    S.set_window(mode != "nowindow")
    S.set_fused(1 if mode.startswith("fused") else (3 if mode.startswith("onepass") else 0))
    S.set_fused_window(1 if mode.endswith("w1") else 0)


@pytest.fixture(scope="module", params=[(c, p) for c in SMALL for p in KERNELS], ids=lambda v: f"{v[0]}-{v[1]}")
def case(request):
    name, pipe = request.param
    A = SMALL[name]()
    F = oracle.ilu0(A)[2]
    S = nsm.Smoother(A, F)
    set_kernels(S, pipe)   # every kernel family must agree with the oracle
    yield f"{name}/{pipe}", A, F, S
    S.close()


def test_residual_spmv(case):
    name, A, F, S = case
    b, x = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    agree(host(S.residual(dev(b), dev(x))), oracle.residual(A, b, x), name + " residual")
    agree(host(S.spmv(dev(x))), oracle.spmv(A, x), name + " spmv")


@pytest.mark.parametrize("k", [0, 1, 2, 3, 7])
def test_tri_solves(case, k):
    name, A, F, S = case
    r = inputs.uniform(3, A.nrows)
    # handle with factors: lsolve/usolve act on the ILU factors
    Ff = (A.rowptr, A.col, F)
    Fs = sp.csr_matrix((F, A.col, A.rowptr), shape=(A.nrows, A.nrows))
    agree(host(S.lsolve(dev(r), k)), oracle.tri_jacobi(Fs, r, k, lower=True, unit=True), f"{name} ilu lsolve k={k}")
    agree(host(S.usolve(dev(r), k)), oracle.tri_jacobi(Fs, r, k, lower=False), f"{name} ilu usolve k={k}")
    del Ff


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_pgs_tri_solves(k):
    A = inputs.var27(7)
    with nsm.Smoother(A) as S:
        r = inputs.uniform(3, A.nrows)
        agree(host(S.lsolve(dev(r), k)), oracle.tri_jacobi(A, r, k, lower=True), f"pgs lsolve k={k}")
        agree(host(S.usolve(dev(r), k)), oracle.tri_jacobi(A, r, k, lower=False), f"pgs usolve k={k}")


@pytest.mark.parametrize("k,nu,xz", [(0, 1, False), (1, 1, False), (2, 1, False), (3, 1, False), (2, 3, False),
                                     (0, 2, True), (2, 1, True), (3, 2, True)])
def test_pgs_smooth(case, k, nu, xz):
    name, A, F, S = case
    b = inputs.uniform(0, A.nrows)
    x0 = np.zeros(A.nrows) if xz else inputs.uniform(1, A.nrows)
    x = start(x0, xz)
    S.smooth(dev(b), x, "pgs", nu=nu, k_l=k, x_is_zero=xz)
    agree(host(x), oracle.pgs_apply(A, b, x0, k, nu=nu, x_is_zero=xz), f"{name} pgs k={k} nu={nu} xz={xz}")


@pytest.mark.parametrize("kl,ku,nu,xz", [(2, 2, 1, False), (0, 0, 1, False), (0, 2, 1, False), (2, 0, 1, False),
                                         (3, 1, 2, False), (1, 3, 1, True), (0, 0, 2, True), (10, 10, 1, False)])
def test_ilu_smooth(case, kl, ku, nu, xz):
    name, A, F, S = case
    b = inputs.uniform(0, A.nrows)
    x0 = np.zeros(A.nrows) if xz else inputs.uniform(1, A.nrows)
    x = start(x0, xz)
    S.smooth(dev(b), x, "ilu", nu=nu, k_l=kl, k_u=ku, x_is_zero=xz)
    want = oracle.ilu_apply(A, (A.rowptr, A.col, F), b, x0, kl, ku, nu=nu, x_is_zero=xz)
    agree(host(x), want, f"{name} ilu kl={kl} ku={ku} nu={nu} xz={xz}")


def test_config1_integer_bitwise():
    """C1 with integer b, x = 0: the oracle is exact (pinned against integer
    arithmetic in test_oracle_pins); the GPU must be bit-identical."""
    A = inputs.config_matrix("C1")
    b = inputs.uniform_int(0, A.nrows, 20)
    with nsm.Smoother(A) as S:
        for k in (1, 2, 3):
            x = torch.zeros(A.nrows, dtype=torch.float64, device="cuda")
            S.smooth(dev(b), x, "pgs", k_l=k, x_is_zero=True)
            assert np.array_equal(host(x), oracle.pgs_apply(A, b, np.zeros(A.nrows), k, x_is_zero=True))


def test_edge_sizes():
    # n = 1, diagonal matrix (empty triangles), a row longer than a warp
    for A in [inputs.CSR.from_scipy(sp.csr_matrix(np.array([[4.0]]))),
              inputs.CSR.from_scipy(sp.diags(np.arange(1.0, 40.0)).tocsr()),
              inputs.random_dense(40, seed=2, diag_shift=30.0)]:
        b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
        with nsm.Smoother(A, oracle.ilu0(A)[2]) as S:
            x = dev(x0)
            S.smooth(dev(b), x, "pgs", k_l=3)
            agree(host(x), oracle.pgs_apply(A, b, x0, 3), f"edge n={A.nrows}")
            x = dev(x0)
            S.smooth(dev(b), x, "ilu", k_l=2, k_u=2)
            agree(host(x), oracle.ilu_apply(A, oracle.ilu0(A), b, x0, 2, 2), f"edge ilu n={A.nrows}")


def test_empty_matrix():
    A = inputs.CSR(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    with nsm.Smoother(A) as S:
        e = torch.zeros(0, dtype=torch.float64, device="cuda")
        S.smooth(e, torch.zeros(0, dtype=torch.float64, device="cuda"), "pgs", k_l=2)
        S.check()


def test_divergence_flag():
    """Jacobi on a highly non-normal triangle may diverge: a
    non-finite sweep output is reported by nsm_check with its sweep index."""
    n = 64
    M = sp.diags([np.full(n - 1, -1e300), np.full(n, 1e-10)], [-1, 0]).tocsr()
    A = inputs.CSR.from_scipy(M)
    with nsm.Smoother(A) as S:
        S.lsolve(dev(np.ones(n)), 3)
        with pytest.raises(nsm.NsmError) as e:
            S.check()
        assert e.value.name == "NSM_ERR_NONFINITE"
        S.check()  # flag is cleared


def test_errors_and_determinism():
    A = inputs.laplace(9, 9, 9)
    b = dev(inputs.uniform(0, A.nrows))
    with nsm.Smoother(A) as S:
        with pytest.raises(nsm.NsmError) as e:
            S.smooth(b, dev(np.zeros(A.nrows)), "ilu", k_l=1)
        assert e.value.name == "NSM_ERR_STATE"
        with pytest.raises(nsm.NsmError) as e:
            S.smooth(b, b, "pgs", k_l=1)
        assert e.value.name == "NSM_ERR_ARG"
        x1, x2 = dev(np.zeros(A.nrows)), dev(np.zeros(A.nrows))
        S.smooth(b, x1, "pgs", nu=2, k_l=3)
        S.smooth(b, x2, "pgs", nu=2, k_l=3)
        assert torch.equal(x1, x2)


# ------------------------------------------------------- full BASELINE sizes --
@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C2", "C3", "C4", "C5"])
def test_full_size_parity(cfg):
    """BASELINE.json configs at full size, in the launch configuration bench.py
    times (one nsm_smooth per application, both kernel families); the oracle
    computes the whole vector (a few seconds of CPU)."""
    A = inputs.config_matrix(cfg)
    kind = {"C2": "ilu", "C3": "pgs", "C4": "ilu", "C5": "pgs"}[cfg]
    F = oracle.ilu0(A)[2] if kind == "ilu" else None
    b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    if kind == "ilu":
        want = oracle.ilu_apply(A, (A.rowptr, A.col, F), b, x0, 2, 2)
    else:
        want = oracle.pgs_apply(A, b, x0, 2)
    with nsm.Smoother(A, F) as S:
        for mode in KERNELS:
            set_kernels(S, mode)
            x = dev(x0)
            S.smooth(dev(b), x, kind, nu=1, k_l=2, k_u=2)
            agree(host(x), want, f"{cfg} kernels={mode}")


ORACLE_APPLY = {
    "pgs_backward": lambda A, b, x0, k, nu, xz: oracle.pgs_backward_apply(A, b, x0, k, nu=nu, x_is_zero=xz),
    "pgs_symmetric": lambda A, b, x0, k, nu, xz: oracle.pgs_symmetric_apply(A, b, x0, k, nu=nu, x_is_zero=xz),
    "l1_jacobi": lambda A, b, x0, k, nu, xz: oracle.l1_jacobi_apply(A, b, x0, nu=nu, x_is_zero=xz),
}


@pytest.mark.parametrize("kind,k,nu,xz", [("pgs_backward", 2, 1, False), ("pgs_backward", 0, 2, True),
                                          ("pgs_backward", 3, 2, True), ("pgs_symmetric", 2, 2, False),
                                          ("pgs_symmetric", 1, 1, True), ("l1_jacobi", 0, 3, False),
                                          ("l1_jacobi", 0, 1, True)])
def test_other_smoothers(case, kind, k, nu, xz):
    """Backward / symmetric pGS and l1-Jacobi."""
    name, A, F, S = case
    b = inputs.uniform(0, A.nrows)
    x0 = np.zeros(A.nrows) if xz else inputs.uniform(1, A.nrows)
    x = start(x0, xz)
    S.smooth(dev(b), x, kind, nu=nu, k_l=k, x_is_zero=xz)
    agree(host(x), ORACLE_APPLY[kind](A, b, x0, k, nu, xz), f"{name} {kind} k={k} nu={nu} xz={xz}")


def test_layout_choice_matches_host_mirror(case):
    """The builder's offset-aligned layout choice (nsm_layout) is the one
    bench.py's reference arm assumes when it counts bytes."""
    import bench
    name, A, F, S = case
    lay, want = S.layout(), bench.aligned_parts(A)
    assert lay["L"] == want["L"] and lay["U"] == want["U"], (name, lay, want)


@pytest.mark.parametrize("name", ["var27_aligned_40", "var27_ragged"])
@pytest.mark.parametrize("xz", [False, True])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_onepass_windowed_pgs(name, xz, k):
    """The one-pass windowed pGS (fused_w.cu, NSM_OPT_FUSED = 3) really runs on
    27-point matrices (its producer counters move) and is bit-identical to
    the oracle for k = 1..4, from x = 0 and x != 0, nu = 2, at the default and
    the tightest skew."""
    A = SMALL[name]() if name in SMALL else inputs.var27_grid(130, 20, 6)   # 15,600 rows: a ragged last tile
    b = inputs.uniform(0, A.nrows)
    x0 = np.zeros(A.nrows) if xz else inputs.uniform(1, A.nrows)
    want = oracle.pgs_apply(A, b, x0, k, nu=2, x_is_zero=xz)
    with nsm.Smoother(A) as S:
        for margin in (0, 1):
            set_kernels(S, "onepass" if margin == 0 else "onepassw1")
            c0 = S.fused_counters()
            x = start(x0, xz)
            S.smooth(dev(b), x, "pgs", nu=2, k_l=k, x_is_zero=xz)
            agree(host(x), want, f"{name} onepass k={k} xz={xz} margin={margin}")
            assert S.fused_counters()[4] > c0[4], "the one-pass kernel did not run"
            S.check()


@pytest.mark.parametrize("grid", [(128, 16, 12), (256, 4, 10)])
@pytest.mark.parametrize("xz", [False, True])
@pytest.mark.parametrize("k", [2, 3, 4])
def test_onepass_plane_wavefront(grid, xz, k):
    """The plane-wavefront one-pass pGS (NSM_OPT_PLANE_ROWS + NSM_OPT_FUSED =
    3; one CTA per line, neighbour-only readiness) is bit-identical to the
    oracle for k = 2..4, x = 0 and x != 0, nu = 2; the structure check rejects
    a wrong plane size."""
    nx, ny, nz = grid
    A = inputs.var27_grid(nx, ny, nz)
    b = inputs.uniform(0, A.nrows)
    x0 = np.zeros(A.nrows) if xz else inputs.uniform(1, A.nrows)
    want = oracle.pgs_apply(A, b, x0, k, nu=2, x_is_zero=xz)
    with nsm.Smoother(A) as S:
        S.set_plane_rows(nx * ny)
        set_kernels(S, "onepass")
        c0 = S.fused_counters()
        x = start(x0, xz)
        S.smooth(dev(b), x, "pgs", nu=2, k_l=k, x_is_zero=xz)
        agree(host(x), want, f"plane wavefront {grid} k={k} xz={xz}")
        assert S.fused_counters()[4] > c0[4], "the one-pass kernel did not run"
        S.check()
        with pytest.raises(nsm.NsmError):
            S.set_plane_rows(nx * ny * 2 if (nx * ny) % 256 == 0 and nz % 2 == 1 else nx * ny // 2 * 3)


@pytest.mark.parametrize("name", ["var27_aligned_40", "var27_ragged", "var27_48tiles"])
@pytest.mark.parametrize("lag", [1, 2])
@pytest.mark.parametrize("xz", [False, True])
@pytest.mark.parametrize("k", [2, 3])
def test_coupled_pgs(name, lag, xz, k):
    """The coupled sweeps (coupled.cu, NSM_OPT_COUPLED) really run on 27-point
    matrices (ONE sweep launch per non-fresh application instead of k) and are
    bit-identical to the oracle for k = 2, 3, nu = 2 (the first application
    from x = 0 runs per pass, the second coupled), at the automatic and the
    tightest throttle distance (lag 2 -> 2 tiles: group 0 waits for the last
    group almost every tile); several tiles per CTA, a ragged last tile, and
    fewer tiles than SMs (var27_48tiles)."""
    A = (SMALL[name]() if name in SMALL else
         inputs.var27_grid(64, 16, 12) if name == "var27_48tiles" else inputs.var27_grid(130, 20, 6))
    b = inputs.uniform(0, A.nrows)
    x0 = np.zeros(A.nrows) if xz else inputs.uniform(1, A.nrows)
    want = oracle.pgs_apply(A, b, x0, k, nu=2, x_is_zero=xz)
    with nsm.Smoother(A) as S:
        S.set_coupled(lag)
        S.set_profile(True)
        S.profile()
        x = start(x0, xz)
        S.smooth(dev(b), x, "pgs", nu=2, k_l=k, x_is_zero=xz)
        agree(host(x), want, f"{name} coupled k={k} xz={xz} lag={lag}")
        assert S.profile()["sweep"][1] == (k + 1 if xz else 2), "the coupled kernel did not run"
        S.check()
        for rep in range(3):   # repeated launches: the epoch advances, results stay identical
            x = start(x0, xz)
            S.smooth(dev(b), x, "pgs", nu=2, k_l=k, x_is_zero=xz)
            agree(host(x), want, f"{name} coupled rep {rep}")
        S.check()


def _stencil(nx, ny, nz, offsets, seed=11):
    """Variable-coefficient stencil on an nx x ny x nz grid (x fastest),
    diagonally dominant, rows ordered lexicographically."""
    rng = np.random.default_rng(seed)
    n = nx * ny * nz
    idx = np.arange(n)
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    rows, cols = [], []
    for dx, dy, dz in offsets:
        ok = (x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny) & (z + dz >= 0) & (z + dz < nz)
        rows.append(idx[ok])
        cols.append(idx[ok] + dx + dy * nx + dz * nx * ny)
    r, c = np.concatenate(rows), np.concatenate(cols)
    M = sp.csr_matrix((rng.uniform(-1, 1, len(r)), (r, c)), shape=(n, n))
    M.setdiag(0.0)
    M.eliminate_zeros()
    M = M + sp.diags(np.abs(M).sum(1).A1 + 1.0)
    return inputs.CSR.from_scipy(M.tocsr())


@pytest.mark.parametrize("wide", [False, True])
def test_windowed_register_chunks(wide):
    """The windowed kernels' register-chunk variants: 27-point rows (13 entries
    per triangle: the 14-entry residual chunk, three CTAs per SM, and the sweeps'
    7-entry chunks) and 27-point + (+-2, 0, 0) rows (15 per triangle: the 16-entry
    residual chunk, and three 7-entry sweep chunks, the last partial); bitwise
    against the oracle, with the windows verifiably in use."""
    offs = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    if wide:
        offs += [(2, 0, 0), (-2, 0, 0)]
    A = _stencil(64, 24, 10, offs)
    b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    with nsm.Smoother(A) as S:
        assert S.windows() == {"residual": True, "L": True, "U": True}, S.windows()
        agree(host(S.residual(dev(b), dev(x0))), oracle.residual(A, b, x0), f"wide={wide} residual")
        for k in (1, 2, 3):
            x = dev(x0)
            S.smooth(dev(b), x, "pgs", nu=2, k_l=k)
            agree(host(x), oracle.pgs_apply(A, b, x0, k, nu=2), f"wide={wide} pgs k={k}")
        r = inputs.uniform(3, A.nrows)
        for k in (1, 3):
            agree(host(S.lsolve(dev(r), k)), oracle.tri_jacobi(A, r, k, lower=True), f"wide={wide} lsolve k={k}")
        S.check()
