"""Debug the in-process halo exchange between virtual ranks on one GPU."""
import ctypes
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_2112_14681_b200 as nsm  # noqa: E402

A = inputs.laplace(10, 9, 8)
bounds = np.array([0, 300, 720], dtype=np.int64)
P = 2
S = [nsm.Smoother(A.rows(int(bounds[r]), int(bounds[r + 1])), rank=r, nranks=P, row_offsets=bounds) for r in range(P)]
for s in S:
    s.set_halo_timeout(2000)
nsm.Smoother.connect_local(S)
streams = [torch.cuda.Stream() for _ in range(P)]
b = inputs.uniform(0, A.nrows)
x = inputs.uniform(1, A.nrows)
bs = [torch.from_numpy(b[bounds[r]:bounds[r + 1]].copy()).cuda() for r in range(P)]
xs = [torch.from_numpy(x[bounds[r]:bounds[r + 1]].copy()).cuda() for r in range(P)]
rs = [torch.empty_like(t) for t in bs]
want = oracle.residual(A, b, x)

from cuda.bindings import runtime as cudart  # noqa: E402


def flags(r):
    base, _, _ = S[r]._mailbox()
    out = np.zeros(P, dtype=np.uint64)
    err, = cudart.cudaMemcpy(out.ctypes.data, base, 8 * P, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    return out


def check(tag):
    torch.cuda.synchronize()
    res = []
    for s in S:
        try:
            s.check()
            res.append("ok")
        except nsm.NsmError as e:
            res.append(e.name)
    got = torch.cat(rs).cpu().numpy()
    print(tag, res, "equal" if np.array_equal(got, want) else "DIFF", "flags", [flags(r).tolist() for r in range(P)],
          flush=True)


print("peers", [s.requests and {int(k): len(v) for k, v in s.requests.items()} for s in S], "n_ghost",
      [s.n_ghost for s in S])
t = time.time()
for r in range(P):
    with torch.cuda.stream(streams[r]):
        S[r].residual(bs[r], xs[r], rs[r])
check(f"A in-order streams {time.time() - t:.2f}s")
t = time.time()
for r in reversed(range(P)):
    with torch.cuda.stream(streams[r]):
        S[r].residual(bs[r], xs[r], rs[r])
check(f"B reversed streams {time.time() - t:.2f}s")
t = time.time()


def work(r):
    with torch.cuda.stream(streams[r]):
        S[r].residual(bs[r], xs[r], rs[r])


th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
for h in th:
    h.start()
for h in th:
    h.join()
check(f"C threads {time.time() - t:.2f}s")
