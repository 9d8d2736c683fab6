"""Builds libnsm.so in-tree with nvcc for sm_100a (no JIT, no torch extension
machinery): the .so travels with the repository snapshot to the GPU box."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnsm.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-shared",
    "-fmad=false",                       # no FMA contraction (reading R10)
    "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps() -> list[str]:
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "nsm.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, variant: str = "", extra: list[str] | None = None) -> str:
    """variant / extra: an alternative build (libnsm_<variant>.so, extra nvcc
    flags, e.g. -DNSM_EXPERIMENTS for the environment knobs) for A/B
    experiments, loaded with paper_2112_14681_b200.load(variant=<variant>).
    Each source is compiled to an object in parallel, then linked."""
    lib = LIB if not variant else os.path.join(HERE, f"libnsm_{variant}.so")
    if not variant and not force and not stale():
        return LIB
    import concurrent.futures as cf
    import tempfile
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + list(extra or []) + ["-I", os.path.join(ROOT, "include")]
    tmpd = tempfile.mkdtemp(prefix="nsm_build_")
    objs = [os.path.join(tmpd, os.path.basename(src) + ".o") for src in sources()]

    def compile_one(src_obj):
        src, obj = src_obj
        return subprocess.run([nvcc, *flags, "-c", "-o", obj, src], capture_output=True, text=True)

    with cf.ThreadPoolExecutor(max_workers=min(len(objs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, zip(sources(), objs)))
    log = "".join(r.stdout + r.stderr for r in results)
    if any(r.returncode != 0 for r in results):
        raise RuntimeError("nvcc failed:\n" + log)
    tmp = lib + f".tmp{os.getpid()}"
    res = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
                          "-Xcompiler", "-fopenmp", "-lgomp"], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(log)
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    os.rmdir(tmpd)
    return lib


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":
        print(build(variant=sys.argv[2], extra=sys.argv[3:]))
    else:
        print(build(force=True, verbose=True))
