"""Set-up cost per config: the host builder (nsm_setup: split + SELL build +
upload from a host CSR) and the device builder (nsm_setup_device from a
device-resident CSR; the H2D copy of the CSR is reported separately), plus
the GPU Chow-Patel ILU(0) and the host ILU(0) where the config uses factors.
Writes one JSON line per config (median of `reps` timings)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2112_14681_b200 as nsm  # noqa: E402


def timed(fn, reps=3):
    ts, out = [], None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        if hasattr(out, "close") and _ < reps - 1:
            out.close()
    return float(np.median(ts)), out


for cfg in sys.argv[1:] or ["C2", "C3", "C4", "C5"]:
    A = inputs.config_matrix(cfg)
    F = nsm.ilu0(A) if cfg in ("C2", "C4") else None
    t_h2d, dev = timed(lambda: (torch.from_numpy(A.rowptr).cuda(), torch.from_numpy(A.col).cuda(),
                                torch.from_numpy(A.val).cuda(),
                                torch.from_numpy(F).cuda() if F is not None else None), 1)
    t_host, Sh = timed(lambda: nsm.Smoother(A, F))
    t_dev, Sd = timed(lambda: nsm.Smoother.from_device_csr(*dev))
    same = all(np.array_equal(Sh.part(p)[k], Sd.part(p)[k]) for p in range(8 if F is not None else 4)
               for k in ("ptr", "col", "val", "off"))
    Sh.close()
    Sd.close()
    line = {"cfg": cfg, "n": A.nrows, "nnz": A.nnz, "host_setup_s": round(t_host, 3),
            "device_setup_s": round(t_dev, 3), "csr_h2d_s": round(t_h2d, 3), "identical_arrays": bool(same)}
    print(json.dumps(line), flush=True)
