"""Multi-rank CUDA path on ONE GPU (-m gpu): several row-block "ranks", each
its own nsm handle and stream, exchange halos through the peer-memory
mailbox path (same device: plain pointers in one process; CUDA IPC across
two processes).  Results must equal the oracle with the same partition
(HYBRID) or without one (GLOBAL: exact global sweeps), bit for
bit and within the 1e-12 contract."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import inputs
import oracle
import paper_2112_14681_b200 as nsm

pytestmark = pytest.mark.gpu


def agree(got, want, what):
    e = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
    assert e <= 1e-12, f"{what}: relerr {e:.2e}"
    assert np.array_equal(got, want), f"{what}: {int(np.sum(got != want))} entries differ (relerr {e:.1e})"


def random_sparse(n, seed):
    rng = np.random.default_rng(seed)
    M = sp.random(n, n, density=6.0 / n, random_state=rng, format="csr")
    M = M + sp.diags(np.abs(M).sum(1).A1 + 1.0)
    return inputs.CSR.from_scipy(M)


CASES = {
    "lap3d_2": (lambda: inputs.laplace(10, 9, 8), [0, 300, 720]),
    "lap3d_3_uneven": (lambda: inputs.laplace(10, 9, 8), [0, 101, 450, 720]),
    "random_3": (lambda: random_sparse(900, 3), [0, 250, 610, 900]),   # couplings between all ranks
    "cd_rcm_4": (lambda: inputs.convdiff(8), [0, 128, 256, 384, 512]),
    # 27-point z-slabs (offset-aligned, gather windows): the interior slices of
    # each rank start on a tile boundary, so they run the windowed kernels
    "var27_slab_3": (lambda: inputs.var27_grid(64, 40, 12), [0, 10240, 20480, 30720]),
    "var27_slab_uneven": (lambda: inputs.var27_grid(64, 40, 12), [0, 7680, 20480, 30720]),
}


class VirtualRanks:
    def __init__(self, A, bounds, mode, factors=None):
        self.A, self.bounds, self.P = A, np.asarray(bounds, np.int64), len(bounds) - 1
        self.S, self.streams = [], []
        for r in range(self.P):
            blk = A.rows(int(bounds[r]), int(bounds[r + 1]))
            F = None
            if isinstance(factors, str) and factors == "block":
                F = nsm.ilu0(blk, row_begin=int(bounds[r]))
            elif factors is not None:  # global factor values on A's pattern
                F = factors[A.rowptr[bounds[r]]:A.rowptr[bounds[r + 1]]]
            self.S.append(nsm.Smoother(blk, F, rank=r, nranks=self.P, row_offsets=self.bounds, mode=mode))
            self.streams.append(torch.cuda.Stream())
        nsm.Smoother.connect_local(self.S)

    def split(self, v):
        return [torch.from_numpy(v[self.bounds[r]:self.bounds[r + 1]].copy()).cuda() for r in range(self.P)]

    def run(self, fn):
        torch.cuda.synchronize()
        for r in range(self.P):
            with torch.cuda.stream(self.streams[r]):
                fn(r, self.S[r])
        torch.cuda.synchronize()
        for S in self.S:
            S.check()

    def close(self):
        for S in self.S:
            S.close()


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("mode", ["hybrid", "global"])
def test_dist_pgs(case, mode):
    A = CASES[case][0]()
    bounds = CASES[case][1]
    m = nsm.NSM_DIST_HYBRID if mode == "hybrid" else nsm.NSM_DIST_GLOBAL
    V = VirtualRanks(A, bounds, m)
    b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    bs, xs = V.split(b), V.split(x0)
    part = bounds if mode == "hybrid" else None
    try:
        # residual and SpMV (halo exchange of x)
        rs = [torch.empty_like(t) for t in bs]
        V.run(lambda r, S: S.residual(bs[r], xs[r], rs[r]))
        agree(torch.cat(rs).cpu().numpy(), oracle.residual(A, b, x0), f"{case} residual")
        # pGS smoothing, nu = 2, k = 2 (and x = 0 start)
        V.run(lambda r, S: S.smooth(bs[r], xs[r], "pgs", nu=2, k_l=2))
        agree(torch.cat(xs).cpu().numpy(), oracle.pgs_apply(A, b, x0, 2, nu=2, bounds=part), f"{case} {mode} pgs")
        zs = [torch.zeros_like(t) for t in bs]
        V.run(lambda r, S: S.smooth(bs[r], zs[r], "pgs", nu=1, k_l=3, x_is_zero=True))
        agree(torch.cat(zs).cpu().numpy(), oracle.pgs_apply(A, b, np.zeros(A.nrows), 3, x_is_zero=True, bounds=part),
              f"{case} {mode} pgs x0=0")
        # lsolve / usolve
        ls = [torch.empty_like(t) for t in bs]
        V.run(lambda r, S: S.lsolve(bs[r], 3, ls[r]))
        agree(torch.cat(ls).cpu().numpy(), oracle.tri_jacobi(A, b, 3, lower=True, bounds=part), f"{case} lsolve")
        V.run(lambda r, S: S.usolve(bs[r], 2, ls[r]))
        agree(torch.cat(ls).cpu().numpy(), oracle.tri_jacobi(A, b, 2, lower=False, bounds=part), f"{case} usolve")
    finally:
        V.close()


@pytest.mark.parametrize("case", ["lap3d_3_uneven", "cd_rcm_4", "random_3"])
@pytest.mark.parametrize("mode", ["hybrid", "global"])
def test_dist_ilu(case, mode):
    A = CASES[case][0]()
    bounds = CASES[case][1]
    b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    if mode == "hybrid":
        V = VirtualRanks(A, bounds, nsm.NSM_DIST_HYBRID, factors="block")
        Fo = oracle.block_ilu0(A, bounds)
        part = bounds
    else:
        Fg = oracle.ilu0(A)
        V = VirtualRanks(A, bounds, nsm.NSM_DIST_GLOBAL, factors=Fg[2])
        Fo, part = Fg, None
    try:
        bs, xs = V.split(b), V.split(x0)
        V.run(lambda r, S: S.smooth(bs[r], xs[r], "ilu", nu=2, k_l=2, k_u=3))
        want = oracle.ilu_apply(A, Fo, b, x0, 2, 3, nu=2, bounds=part)
        agree(torch.cat(xs).cpu().numpy(), want, f"{case} {mode} ilu")
    finally:
        V.close()


def test_global_mode_partition_invariant():
    """GLOBAL results do not depend on the partition (exact global sweeps)."""
    A = inputs.laplace(12, 10, 6)
    b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    outs = []
    for bounds in ([0, A.nrows], [0, 200, A.nrows], [0, 100, 333, 600, A.nrows]):
        if len(bounds) == 2:
            with nsm.Smoother(A) as S:
                x = torch.from_numpy(x0.copy()).cuda()
                S.smooth(torch.from_numpy(b).cuda(), x, "pgs", nu=1, k_l=4)
                outs.append(x.cpu().numpy())
            continue
        V = VirtualRanks(A, bounds, nsm.NSM_DIST_GLOBAL)
        bs, xs = V.split(b), V.split(x0)
        V.run(lambda r, S: S.smooth(bs[r], xs[r], "pgs", nu=1, k_l=4))
        outs.append(torch.cat(xs).cpu().numpy())
        V.close()
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


# ------------------------------------------------ two processes, CUDA IPC ----
def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        N = 8
        n_loc = N ** 3
        offsets = np.arange(world + 1) * n_loc
        A = inputs.weak_slab(N, world, rank)
        rb = rank * n_loc
        S = nsm.Smoother(A, device=0, rank=rank, nranks=world, row_offsets=offsets)
        S.connect(dist)
        b = torch.from_numpy(inputs.uniform(0, n_loc, idx0=rb)).cuda()
        x = torch.from_numpy(inputs.uniform(1, n_loc, idx0=rb)).cuda()
        S.smooth(b, x, "pgs", nu=2, k_l=2)
        S.check()
        out = [torch.empty(n_loc, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, x.cpu())
        if rank == 0:
            Ag = inputs.laplace(N, N, N * world)
            want = oracle.pgs_apply(Ag, inputs.uniform(0, Ag.nrows), inputs.uniform(1, Ag.nrows), 2, nu=2,
                                    bounds=offsets)
            q.put(bool(np.array_equal(torch.cat(out).numpy(), want)))
        dist.barrier()
        S.close()
        dist.destroy_process_group()
    except Exception as e:
        q.put(repr(e))
        raise


def test_two_process_ipc_same_device():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert res is True, res


@pytest.mark.parametrize("mode", ["hybrid", "global"])
@pytest.mark.parametrize("kind", ["pgs_backward", "pgs_symmetric", "l1_jacobi"])
def test_dist_other_smoothers(mode, kind):
    A = CASES["random_3"][0]()
    bounds = CASES["random_3"][1]
    m = nsm.NSM_DIST_HYBRID if mode == "hybrid" else nsm.NSM_DIST_GLOBAL
    part = bounds if mode == "hybrid" else None
    V = VirtualRanks(A, bounds, m)
    b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    try:
        bs, xs = V.split(b), V.split(x0)
        V.run(lambda r, S: S.smooth(bs[r], xs[r], kind, nu=2, k_l=2))
        if kind == "pgs_backward":
            want = oracle.pgs_backward_apply(A, b, x0, 2, nu=2, bounds=part)
        elif kind == "pgs_symmetric":
            want = oracle.pgs_symmetric_apply(A, b, x0, 2, nu=2, bounds=part)
        else:
            want = oracle.l1_jacobi_apply(A, b, x0, nu=2)
        agree(torch.cat(xs).cpu().numpy(), want, f"{mode} {kind}")
    finally:
        V.close()


@pytest.mark.parametrize("mode", ["hybrid", "global"])
def test_eight_rank_slabs(mode):
    """C5 shape: 8 z-slabs of a 7-point grid (each rank 20 x 20 x 6 rows),
    pGS k = 2 and ILU(0) k = 2, nu = 2, all ranks exchanging over the
    mailbox path at once."""
    P, N = 8, 20
    A = inputs.laplace(N, N, 6 * P)
    n_loc = N * N * 6
    bounds = list(range(0, P * n_loc + 1, n_loc))
    b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
    m = nsm.NSM_DIST_HYBRID if mode == "hybrid" else nsm.NSM_DIST_GLOBAL
    part = bounds if mode == "hybrid" else None
    V = VirtualRanks(A, bounds, m)
    try:
        bs, xs = V.split(b), V.split(x0)
        V.run(lambda r, S: S.smooth(bs[r], xs[r], "pgs", nu=2, k_l=2))
        agree(torch.cat(xs).cpu().numpy(), oracle.pgs_apply(A, b, x0, 2, nu=2, bounds=part), f"8 ranks {mode} pgs")
    finally:
        V.close()
    if mode == "hybrid":
        V = VirtualRanks(A, bounds, m, factors="block")
        Fo = oracle.block_ilu0(A, bounds)
    else:
        Fg = oracle.ilu0(A)
        V = VirtualRanks(A, bounds, m, factors=Fg[2])
        Fo = Fg
    try:
        bs, xs = V.split(b), V.split(x0)
        V.run(lambda r, S: S.smooth(bs[r], xs[r], "ilu", nu=2, k_l=2, k_u=2))
        agree(torch.cat(xs).cpu().numpy(), oracle.ilu_apply(A, Fo, b, x0, 2, 2, nu=2, bounds=part),
              f"8 ranks {mode} ilu")
    finally:
        V.close()


def _xdev_worker(rank, world, port, q, same_device):
    """One rank per process (CUDA IPC mailboxes, gloo plumbing): HYBRID and
    GLOBAL pGS, the device all-reduce and Algorithm 1 across the ranks."""
    import torch.distributed as dist
    from oracle import krylov
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = 0 if same_device else rank
        torch.cuda.set_device(dev)
        N = 8
        n_loc = N ** 3
        offsets = np.arange(world + 1) * n_loc
        A = inputs.weak_slab(N, world, rank)
        rb = rank * n_loc
        Ag = inputs.laplace(N, N, N * world)
        bg, xg = inputs.uniform(0, Ag.nrows), inputs.uniform(1, Ag.nrows)
        ok = True
        for mode, bounds in ((nsm.NSM_DIST_HYBRID, offsets), (nsm.NSM_DIST_GLOBAL, None)):
            S = nsm.Smoother(A, device=dev, rank=rank, nranks=world, row_offsets=offsets, mode=mode)
            S.connect(dist)
            b = torch.from_numpy(bg[rb:rb + n_loc].copy()).cuda(dev)
            x = torch.from_numpy(xg[rb:rb + n_loc].copy()).cuda(dev)
            S.smooth(b, x, "pgs", nu=2, k_l=2)
            S.check()
            out = [torch.empty(n_loc, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(out, x.cpu())
            want = oracle.pgs_apply(Ag, bg, xg, 2, nu=2, bounds=bounds)
            ok = ok and bool(np.array_equal(torch.cat(out).numpy(), want))
            if mode == nsm.NSM_DIST_GLOBAL:
                C = nsm.Comm(rank, world, 1024, device=dev)
                C.connect(dist)
                v = torch.full((37,), float(rank + 1), dtype=torch.float64, device=f"cuda:{dev}")
                s = C.allreduce(v)
                C.check()
                ok = ok and bool(torch.all(s.cpu() == world * (world + 1) / 2))
                S.set_comm(C)
                xs, its, hist = nsm.gmres(S, b, None, tol=1e-8, maxit=200)
                _, its_o, _ = krylov.gmres_lowsync(Ag.to_scipy(), bg, lambda v_: v_, tol=1e-8)
                ok = ok and its == its_o
                C.check()
                dist.barrier()
                S.set_comm(None)
                C.close()
            dist.barrier()
            S.close()
        res = [None] * world
        dist.all_gather_object(res, ok)
        if rank == 0:
            q.put(all(res))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        q.put(repr(e))
        raise


@pytest.mark.parametrize("same_device", [True, False])
def test_two_process_halo_comm_gmres(same_device):
    """Two processes exchange halos and reduce through CUDA IPC mappings: on
    one device (always runnable) and on two distinct devices over NVLink
    (skipped unless two GPUs are visible)."""
    if not same_device and torch.cuda.device_count() < 2:
        pytest.skip("needs two visible GPUs (peer stores over NVLink)")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_xdev_worker, args=(r, 2, port, q, same_device)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert res is True, res
