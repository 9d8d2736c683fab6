"""Where does the end-to-end time go?  C5-sized pGS: (a) torch pinned copies +
device smooth, (b) nsm_smooth_host, (c) the copies alone, each timed with
events over 10 steps (no L2 flush)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs
import paper_2112_14681_b200 as nsm

A = inputs.laplace(256, 256, 256)
n = A.nrows
b = torch.from_numpy(inputs.uniform(0, n)).cuda(); x0 = torch.from_numpy(inputs.uniform(1, n)).cuda()
bh, xh = b.cpu().pin_memory(), x0.cpu().pin_memory()
xw, xo = torch.empty_like(xh).pin_memory(), torch.empty_like(xh).pin_memory()
bd, xd = torch.empty_like(b), torch.empty_like(b)
st = torch.cuda.current_stream()
print("pinned:", bh.is_pinned(), xw.is_pinned())
with nsm.Smoother(A, None, device=0) as S:
    def run(name, f, reps=10):
        f(); torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            xw.copy_(xh)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(st); f(); e1.record(st); torch.cuda.synchronize()
            ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
        a = np.array(ts).mean(0)
        print(f"{name:28s} events {a[0]:8.3f} ms   wall {a[1]:8.3f} ms")
    def torch_path():
        bd.copy_(bh, non_blocking=True); xd.copy_(xh, non_blocking=True)
        S.smooth(bd, xd, "pgs", nu=1, k_l=2); xo.copy_(xd, non_blocking=True)
    run("torch copies + smooth", torch_path)
    run("nsm_smooth_host in place", lambda: S.smooth_host(bh, xw, "pgs", nu=1, k_l=2))
    run("nsm_smooth_host out=", lambda: S.smooth_host(bh, xh, "pgs", nu=1, k_l=2, out=xo))
    run("copies only (torch)", lambda: (bd.copy_(bh, non_blocking=True), xd.copy_(xh, non_blocking=True), xo.copy_(xd, non_blocking=True)))
    run("smooth only", lambda: S.smooth(bd, xd, "pgs", nu=1, k_l=2))
