"""Host<->device copy bandwidth on this box (the floor of bench.py's e2e):
pinned 256 MB host-to-device, 128 MB device-to-host, and both at once on two
streams (C3's per-step copies: b and x in, x out), CUDA events, best of 5."""
import torch

n_in, n_out = 32 * 1024 * 1024, 16 * 1024 * 1024          # doubles: 256 MB, 128 MB
hi = torch.empty(n_in, dtype=torch.float64).pin_memory()
ho = torch.empty(n_out, dtype=torch.float64).pin_memory()
di = torch.empty(n_in, dtype=torch.float64, device="cuda")
do = torch.zeros(n_out, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(f):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def both():
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)


t_in = timed(lambda: di.copy_(hi, non_blocking=True))
t_out = timed(lambda: ho.copy_(do, non_blocking=True))
t_both = timed(both)
print(f"H2D 256 MB: {t_in:.3f} ms = {256 * 1.048576 / t_in:.1f} GB/s")
print(f"D2H 128 MB: {t_out:.3f} ms = {128 * 1.048576 / t_out:.1f} GB/s")
print(f"both at once: {t_both:.3f} ms (the copy floor of one C3 e2e step)")
