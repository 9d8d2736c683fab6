"""The reference arm of bench.py (the CPU oracle timed as the base contract's
reference) runs on the host: check its JSON line end to end."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["unit"] == "GB/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == len(os.sched_getaffinity(0))
    assert cb["single_core"]["cores"] == 1 and cb["single_core"]["value"] > 0
    # default workload = C3 (the largest single-GPU config); the config object
    # carries the workload only, the same keys as the nsm arm's
    assert line["config"]["name"] == "C3" and "27-point" in line["config"]["workload"]
    assert set(line["config"]) == {"workload", "name", "grid_per_gpu", "n_per_gpu", "kind", "k_l", "k_u", "nu",
                                   "partition", "l2"}
    assert line["config"]["n_per_gpu"] == 256 ** 3 and line["detail"]["nnz"] == 449455096


def test_byte_models():
    """Per-pass algorithmic bytes exceed the one-pass floor (the sweeps re-read
    the triangle); closed forms for a 7-point Laplacian."""
    sys.path.insert(0, ROOT)
    import bench
    import inputs
    A = inputs.laplace(16, 16, 16)
    nl, nu, noff = bench.split_counts(A)
    n = A.nrows
    for kind, kl, ku in (("pgs", 2, 0), ("ilu", 2, 2), ("pgs", 1, 0), ("ilu", 3, 1)):
        pp = bench.algorithmic_bytes(kind, n, noff, nl, nu, kl, ku)
        fl = bench.floor_bytes(kind, n, noff, nl, nu, kl, ku)
        assert fl["total"] < pp["total"]
    pp = bench.algorithmic_bytes("pgs", n, noff, nl, nu, 2, 0)
    assert pp["residual"] == 12 * noff + 40 * n                      # OUT_RG: r and g0 written
    assert pp["sweeps"] == [12 * nl + 32 * n, 12 * nl + 40 * n]      # last sweep: x read + write
    assert bench.floor_bytes("pgs", n, noff, nl, nu, 2, 0)["total"] == 12 * noff + 32 * n
    # the coupled sweeps (one kernel, L streamed once): the per-pass sweeps'
    # vectors, L's entries once; k = 1 has nothing to couple
    cp = bench.algorithmic_bytes("pgs", n, noff, nl, nu, 2, 0, coupled=True)
    assert cp["residual"] == pp["residual"]
    assert cp["sweeps"] == [12 * nl + 32 * n + 8 * n + 32 * n]      # L once; r, d, g0 | r, d, g1, x rd+wr; g1 written
    k3 = bench.algorithmic_bytes("pgs", n, noff, nl, nu, 3, 0, coupled=True)
    assert k3["sweeps"] == [sum(bench.algorithmic_bytes("pgs", n, noff, nl, nu, 3, 0)["sweeps"]) - 2 * 12 * nl]
    assert bench.algorithmic_bytes("pgs", n, noff, nl, nu, 1, 0, coupled=True) == \
        bench.algorithmic_bytes("pgs", n, noff, nl, nu, 1, 0)
