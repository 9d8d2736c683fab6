"""Distributed solver layer on ONE GPU (-m gpu): the cross-rank all-reduce
(nsm_comm: Algorithm 1's single global reduction per iteration, step 6
P:L485, "one MPI_AllReduce per iteration" P:L299-307) and GMRES + one C-AMG
V-cycle on a row-block partition of the finest level (virtual ranks: one
handle, comm and stream per rank, one host thread per rank because every
GMRES iteration synchronises its stream).  The finest level runs in GLOBAL
mode (exact global sweeps, partition-independent), coarse levels are
replicated, so the iteration counts must equal the oracle's on the global
matrix (the north_star's "iteration counts must be identical")."""
import threading

import numpy as np
import pytest
import torch

import inputs
import oracle
import paper_2112_14681_b200 as nsm
from oracle import amg, krylov

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def make_comms(P, cap):
    cs = [nsm.Comm(r, P, cap, device=0) for r in range(P)]
    nsm.Comm.connect_local(cs)
    return cs


@pytest.mark.parametrize("P", [1, 2, 3, 5])
@pytest.mark.parametrize("m", [1, 37, 5000, 100003])
def test_comm_allreduce_sums_in_rank_order(P, m):
    cs = make_comms(P, 100003)
    streams = [torch.cuda.Stream() for _ in range(P)]
    try:
        for rep in range(5):  # both parity buffers, several times
            vals = [inputs.uniform(10 * rep + r, m) * (1 + r) for r in range(P)]
            want = vals[0].copy()
            for r in range(1, P):
                want = want + vals[r]  # ascending rank order, one rounding per add
            ins = [dev(v) for v in vals]
            outs = [torch.empty_like(x) for x in ins] if rep % 2 == 0 else ins   # in == out allowed
            torch.cuda.synchronize()
            for r in range(P):
                cs[r].allreduce(ins[r], outs[r], stream=streams[r])
            torch.cuda.synchronize()
            for r in range(P):
                cs[r].check(stream=streams[r])
                assert np.array_equal(outs[r].cpu().numpy(), want), (P, m, rep, r)
        assert all(c.stats() == 5 for c in cs)
    finally:
        for c in cs:
            c.close()


def test_comm_errors():
    c = nsm.Comm(0, 2, 16, device=0)
    x = dev(np.ones(4))
    with pytest.raises(nsm.NsmError, match="NSM_ERR_STATE"):
        c.allreduce(x)                              # rank 1 not connected
    c.close()
    cs = make_comms(2, 64)
    with pytest.raises(nsm.NsmError, match="NSM_ERR_ARG"):
        cs[0].allreduce(dev(np.ones(65)))           # above the capacity
    # a rank that never joins: the other one times out (flag, no hang)
    cs[0].set_timeout(200)
    cs[0].allreduce(x)
    with pytest.raises(nsm.NsmError, match="NSM_ERR_DIST"):
        cs[0].check()
    for c in cs:
        c.close()


def rand_fn(level, n):
    return inputs.uniform(1000 + level, n, 0.0, 1.0)


CASES = {
    # name: (matrix, partition fractions, smoother of the finest level)
    "C1_P2": (lambda: inputs.config_matrix("C1"), 2, "pgs"),
    "C3shape_24_P3": (lambda: inputs.var27(24), 3, "pgs"),
    "C4shape_16_P2_hybrid_ilu": (lambda: inputs.convdiff(16), 2, "ilu"),
}


class DistBuilt:
    """The oracle's hierarchy; the finest level split into P row blocks
    (GLOBAL-mode handles, global ILU(0) factor rows), coarse levels
    replicated: every rank gets its own single-rank handles and V-cycle."""

    def __init__(self, name, k, maxit=200):
        Afn, P, finest = CASES[name]
        A = Afn()
        self.A = A.to_scipy()
        self.levels = amg.hierarchy(self.A, rand_fn, min_coarse=200)
        nl = len(self.levels) - 1
        self.kinds = [finest] + ["pgs"] * (nl - 1)
        self.F = [oracle.ilu0(self.levels[l][0])[2] if self.kinds[l] == "ilu" else None for l in range(nl)]
        self.k, self.P, self.nl = k, P, nl
        n = A.nrows
        self.bounds = np.array([n * r // P for r in range(P + 1)], dtype=np.int64)
        self.lu = amg.coarse_lu(self.levels)
        A0 = inputs.CSR.from_scipy(self.levels[0][0])
        P0 = inputs.CSR.from_scipy(self.levels[0][1])
        n1 = self.levels[1][0].shape[0]
        self.comms = make_comms(P, max(n1, 2 * (maxit + 2)))
        self.S0, self.Sc, self.M, self.streams = [], [], [], []
        for r in range(P):
            r0, r1 = int(self.bounds[r]), int(self.bounds[r + 1])
            F = self.F[0][A0.rowptr[r0]:A0.rowptr[r1]] if self.F[0] is not None else None
            S = nsm.Smoother(A0.rows(r0, r1), F, rank=r, nranks=P, row_offsets=self.bounds, mode=nsm.NSM_DIST_GLOBAL)
            self.S0.append(S)
        nsm.Smoother.connect_local(self.S0)
        for r in range(P):
            self.S0[r].set_comm(self.comms[r])
            r0, r1 = int(self.bounds[r]), int(self.bounds[r + 1])
            Sc = [nsm.Smoother(inputs.CSR.from_scipy(self.levels[l][0]), self.F[l]) for l in range(1, nl)]
            Ps = [P0.rows(r0, r1)] + [inputs.CSR.from_scipy(self.levels[l][1]) for l in range(1, nl)]
            for p in Ps:
                p.row_begin = 0
            M = nsm.Amg([self.S0[r]] + Sc, Ps, inputs.CSR.from_scipy(self.levels[-1][0]))
            for l in range(nl):
                M.set_smoother(l, self.kinds[l], 1, 1, k, k)
            self.Sc.append(Sc)
            self.M.append(M)
            self.streams.append(torch.cuda.Stream())

    def smooth_orc(self, lev, Mat, b, x, z):
        if self.kinds[lev] == "ilu":
            Mc = inputs.CSR.from_scipy(Mat)
            return oracle.ilu_apply(Mc, (Mc.rowptr, Mc.col, self.F[lev]), b, x, self.k, self.k, x_is_zero=z)
        return oracle.pgs_apply(Mat, b, x, self.k, x_is_zero=z)

    def vcycle_orc(self, v):
        return amg.vcycle(self.levels, self.smooth_orc, v, lu=self.lu)

    def split(self, v):
        return [dev(v[self.bounds[r]:self.bounds[r + 1]]) for r in range(self.P)]

    def run_ranks(self, fn):
        """fn(r) on one host thread per rank (each GMRES iteration waits for
        the global reduction, which needs every rank's kernels in flight)."""
        out, errs = [None] * self.P, []

        def body(r):
            try:
                torch.cuda.set_device(0)
                out[r] = fn(r)
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        torch.cuda.synchronize()   # inputs made on the default stream; the rank streams do not wait for it
        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.P)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(timeout=300)
        assert not errs, errs
        return out

    def close(self):
        for M in self.M:
            M.close()
        for Sc in self.Sc:
            for S in Sc:
                S.close()
        for S in self.S0:
            S.close()
        for c in self.comms:
            c.close()


@pytest.mark.parametrize("case", list(CASES))
def test_dist_vcycle_matches_oracle(case):
    B = DistBuilt(case, 2)
    try:
        b = inputs.uniform(0, B.A.shape[0])
        bs = B.split(b)
        xs = B.run_ranks(lambda r: B.M[r].vcycle(bs[r], stream=B.streams[r].cuda_stream))
        torch.cuda.synchronize()
        got = np.concatenate([x.cpu().numpy() for x in xs])
        want = B.vcycle_orc(b)
        # restriction sums across ranks in another order than the oracle's rows
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-11
        for S in B.S0:
            S.check()
    finally:
        B.close()


@pytest.mark.parametrize("case", list(CASES))
def test_dist_gmres_iteration_parity(case):
    """Algorithm 1 across ranks: the counts equal the oracle's Algorithm 1 and
    classical MGS-GMRES on the global matrix at 1e-5 and 1e-8, every rank
    stops at the same iteration, and the assembled x solves the system."""
    B = DistBuilt(case, 2)
    try:
        b = inputs.uniform(0, B.A.shape[0])
        bs = B.split(b)
        for tol in (1e-5, 1e-8):
            res = B.run_ranks(lambda r: nsm.gmres(B.S0[r], bs[r], B.M[r], tol=tol,
                                                  stream=B.streams[r].cuda_stream))
            its = [r[1] for r in res]
            _, its_ls, h_ls = krylov.gmres_lowsync(B.A, b, B.vcycle_orc, tol=tol)
            _, its_cl, _ = amg.gmres(B.A, b, B.vcycle_orc, tol=tol)
            assert len(set(its)) == 1 and its[0] == its_ls == its_cl, (case, tol, its, its_ls, its_cl)
            for r in range(B.P):
                np.testing.assert_array_equal(res[r][2], res[0][2])   # identical reduced values on every rank
            np.testing.assert_allclose(res[0][2], h_ls, rtol=1e-6)
            x = np.concatenate([r[0].cpu().numpy() for r in res])
            assert np.linalg.norm(b - B.A @ x) / np.linalg.norm(b) < tol * 10
        for c in B.comms:
            c.check()
    finally:
        B.close()


def test_dist_gmres_without_comm_is_an_error():
    A = inputs.laplace(8, 8, 8)
    bounds = np.array([0, 256, 512], dtype=np.int64)
    S = [nsm.Smoother(A.rows(int(bounds[r]), int(bounds[r + 1])), rank=r, nranks=2, row_offsets=bounds,
                      mode=nsm.NSM_DIST_GLOBAL) for r in range(2)]
    nsm.Smoother.connect_local(S)
    with pytest.raises(nsm.NsmError, match="NSM_ERR_STATE"):
        nsm.gmres(S[0], dev(np.ones(256)))
    for s in S:
        s.close()
