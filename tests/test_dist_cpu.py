"""Multi-rank host logic on CPU (-m "not gpu"): the halo plan of the C-ABI
(nsm_halo_plan, host-only), the plan exchange over a world_size-2 gloo
process group, and the HYBRID semantics of the distributed smoother
(exchange the boundary x, then relax locally) emulated rank by
rank with the oracle and compared with the single-process oracle on the same
partition."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle
import paper_2112_14681_b200 as nsm


def test_halo_plan_slabs():
    N, P = 4, 3
    n_loc = N ** 3
    offsets = np.arange(P + 1) * n_loc
    A1 = inputs.weak_slab(N, P, 1)
    plan = nsm.halo_plan(A1, offsets, 1)
    assert sorted(plan) == [0, 2]
    np.testing.assert_array_equal(plan[0], np.arange(n_loc - N * N, n_loc))        # last plane of rank 0
    np.testing.assert_array_equal(plan[2], np.arange(2 * n_loc, 2 * n_loc + N * N))  # first plane of rank 2
    A0 = inputs.weak_slab(N, P, 0)
    assert sorted(nsm.halo_plan(A0, offsets, 0)) == [1]


def test_exchange_plan_local():
    """exchange_plan inverts the request lists (emulated collective)."""
    reqs = [{1: np.array([5, 6])}, {0: np.array([1]), 2: np.array([9])}, {1: np.array([4, 7])}]

    def ago_for(r):
        def ago(out, obj):
            for q in range(3):
                out[q] = reqs[q]
        return ago
    s0 = nsm.exchange_plan(reqs[0], 0, 3, ago_for(0))
    s1 = nsm.exchange_plan(reqs[1], 1, 3, ago_for(1))
    assert list(s0) == [1] and s0[1].tolist() == [1]
    assert sorted(s1) == [0, 2] and s1[0].tolist() == [5, 6] and s1[2].tolist() == [4, 7]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _relabel(A, row_begin, ghosts):
    """Local CSR with columns [0, n) owned and [n, n + ng) ghosts (stored
    order unchanged, so ascending-order sums are preserved)."""
    n = A.nrows
    col = A.col.copy()
    own = (col >= row_begin) & (col < row_begin + n)
    col[own] -= row_begin
    col[~own] = n + np.searchsorted(ghosts, col[~own])
    return inputs.CSR(n, n + len(ghosts), A.rowptr, col, A.val)


def _diag_block(A, row_begin):
    n = A.nrows
    rows = np.repeat(np.arange(n), np.diff(A.rowptr))
    keep = (A.col >= row_begin) & (A.col < row_begin + n)
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows[keep], minlength=n))]).astype(np.int64)
    return inputs.CSR(n, n, rp, A.col[keep] - row_begin, A.val[keep])


def _worker(rank, world, port, cfg, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        N = 6
        n_loc = N ** 3
        offsets = np.arange(world + 1) * n_loc
        A = inputs.weak_slab(N, world, rank)
        rb = rank * n_loc
        b = inputs.uniform(inputs.SEED_B, n_loc, idx0=rb)
        x = inputs.uniform(inputs.SEED_X0, n_loc, idx0=rb)
        # 1. plan + plan exchange (the code path Smoother.connect uses)
        req = nsm.halo_plan(A, offsets, rank)
        sends = nsm.exchange_plan(req, rank, world, dist.all_gather_object)
        # 2. exchange the boundary x over gloo along the plan
        ops = []
        recv = {qq: torch.empty(len(v), dtype=torch.float64) for qq, v in req.items()}
        for qq, rows in sends.items():
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(x[rows - rb].copy()), qq))
        for qq, t in recv.items():
            ops.append(dist.P2POp(dist.irecv, t, qq))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        ghosts_id = np.concatenate([req[qq] for qq in sorted(req)])
        ghosts = np.concatenate([recv[qq].numpy() for qq in sorted(recv)])
        np.testing.assert_array_equal(ghosts, np.concatenate(
            [inputs.uniform(inputs.SEED_X0, 1, idx0=int(g)) for g in ghosts_id]))
        # 3. HYBRID pGS on this rank: full residual with the halo, local sweeps
        k = 2
        Al = _relabel(A, rb, ghosts_id)
        r = oracle.residual(Al, b, np.concatenate([x, ghosts]))
        g = oracle.tri_jacobi(_diag_block(A, rb), r, k, lower=True)
        xn = x + g
        out = [torch.empty(n_loc, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(xn))
        if rank == 0:
            Ag = inputs.laplace(N, N, N * world)
            bg = inputs.uniform(inputs.SEED_B, Ag.nrows)
            xg = inputs.uniform(inputs.SEED_X0, Ag.nrows)
            want = oracle.pgs_apply(Ag, bg, xg, k, bounds=offsets)
            got = torch.cat(out).numpy()
            q.put(bool(np.array_equal(got, want)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # report to the parent
        q.put(repr(e))
        raise


def test_gloo_world2_plan_and_hybrid_semantics():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, None, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert res is True, res
    assert all(p.exitcode == 0 for p in procs)
