"""paper_2112_14681_b200 — Neumann-series smoothers (arXiv 2112.14681) for B200.

Thin Python binding over the C-ABI library libnsm.so (include/nsm.h).  Every
step of the smoother runs in the library's sm_100a kernels; this module only
marshals arguments (host CSR arrays at setup, device pointers and the
current CUDA stream at call time).  There is no CPU fallback: if libnsm.so
is missing or no CUDA device is present the calls raise.
"""
from __future__ import annotations

from ._lib import (NSM_DIST_GLOBAL, NSM_DIST_HYBRID, NSM_ILU0, NSM_PGS, Amg, Comm, FactorCSR, NsmError, Smoother, SpMat,
                   dep, exchange_plan, exported_symbols, gmres, halo_plan, ilu0, ilu0_fixed_point, ilut, lib_path, load,
                   ruiz)

__all__ = ["Smoother", "SpMat", "Amg", "Comm", "gmres", "ilut", "ruiz", "dep", "FactorCSR", "NsmError", "ilu0", "ilu0_fixed_point", "halo_plan", "exchange_plan", "load", "lib_path", "exported_symbols", "NSM_PGS", "NSM_ILU0",
           "NSM_DIST_HYBRID", "NSM_DIST_GLOBAL"]
