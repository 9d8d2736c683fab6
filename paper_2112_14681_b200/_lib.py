"""ctypes binding of libnsm.so — argument marshalling only (include/nsm.h)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, "libnsm.so")
_lib = None

NSM_PGS, NSM_ILU0, NSM_PGS_BACKWARD, NSM_PGS_SYMMETRIC, NSM_L1_JACOBI = 0, 1, 2, 3, 4
KINDS = {"pgs": NSM_PGS, "ilu": NSM_ILU0, "ilu0": NSM_ILU0, "pgs_backward": NSM_PGS_BACKWARD,
         "pgs_symmetric": NSM_PGS_SYMMETRIC, "l1_jacobi": NSM_L1_JACOBI}
NSM_DIST_HYBRID, NSM_DIST_GLOBAL = 0, 1
_STATUS = {0: "NSM_OK", 1: "NSM_ERR_ARG", 2: "NSM_ERR_PATTERN", 3: "NSM_ERR_ZERO_DIAG", 4: "NSM_ERR_NONFINITE",
           5: "NSM_ERR_CUDA", 6: "NSM_ERR_OOM", 7: "NSM_ERR_STATE", 8: "NSM_ERR_DIST"}

# every symbol include/nsm.h declares (tests check the .so exports them)
SYMBOLS = sorted(["nsm_setup", "nsm_ilu0", "nsm_ilu0_fixed_point", "nsm_residual", "nsm_lsolve", "nsm_usolve", "nsm_smooth", "nsm_smooth_host", "nsm_spmv",
                  "nsm_check", "nsm_info", "nsm_stats", "nsm_last_error", "nsm_destroy", "nsm_halo_plan",
                  "nsm_halo_set_send", "nsm_halo_mailbox", "nsm_halo_connect_ipc", "nsm_halo_connect",
                  "nsm_halo_commit", "nsm_set_option", "nsm_spmat_setup", "nsm_spmat_apply",
                  "nsm_spmat_destroy", "nsm_amg_setup", "nsm_amg_set_smoother", "nsm_amg_vcycle", "nsm_amg_destroy",
                  "nsm_solver_last_error", "nsm_gmres", "nsm_profile", "nsm_ilut", "nsm_ruiz", "nsm_set_ruiz",
                  "nsm_fused_stats", "nsm_layout", "nsm_comm_create", "nsm_comm_mailbox", "nsm_comm_connect",
                  "nsm_comm_connect_ipc", "nsm_comm_allreduce", "nsm_comm_check", "nsm_comm_set_timeout",
                  "nsm_comm_stats", "nsm_comm_last_error", "nsm_comm_destroy", "nsm_set_comm", "nsm_ruiz_dep",
                  "nsm_dep", "nsm_setup_device", "nsm_part_info", "nsm_part_copy", "nsm_diag_copy",
                  "nsm_fused_counters", "nsm_coupled_counters"])


class NsmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = _STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {msg}")


class _Csr(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64), ("rowptr", ctypes.c_void_p),
                ("colind", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class _Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("row_offsets", ctypes.c_void_p),
                ("mode", ctypes.c_int)]


def lib_path() -> str:
    return _LIBPATH


def load(variant: str = ""):
    """Load libnsm.so; raises if it has not been built (no fallback).
    variant: an alternative in-tree build for A/B experiments
    (build.py --variant NAME -> libnsm_NAME.so), chosen explicitly before the
    first handle is created."""
    global _lib, _LIBPATH
    if _lib is not None:
        if variant and not _LIBPATH.endswith(f"libnsm_{variant}.so"):
            raise RuntimeError("load(variant) after the library was loaded")
        return _lib
    if variant:
        _LIBPATH = os.path.join(_HERE, f"libnsm_{variant}.so")
    if not os.path.exists(_LIBPATH):
        raise ImportError(f"{_LIBPATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
    L = ctypes.CDLL(_LIBPATH)
    vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    P = ctypes.POINTER
    L.nsm_setup.argtypes = [P(vp), P(_Csr), P(_Csr), P(_Dist), ci]
    L.nsm_ilu0.argtypes = [P(_Csr), i64, vp]
    L.nsm_ilu0_fixed_point.argtypes = [P(_Csr), i64, ci, vp, ci]
    L.nsm_residual.argtypes = [vp, vp, vp, vp, vp]
    L.nsm_spmv.argtypes = [vp, vp, vp, vp]
    L.nsm_lsolve.argtypes = [vp, vp, vp, ci, vp]
    L.nsm_usolve.argtypes = [vp, vp, vp, ci, vp]
    L.nsm_smooth.argtypes = [vp, ci, vp, vp, ci, ci, ci, ci, vp]
    L.nsm_smooth_host.argtypes = [vp, ci, vp, vp, vp, ci, ci, ci, ci, vp]
    L.nsm_check.argtypes = [vp, P(i64), vp]
    L.nsm_info.argtypes = [vp, P(i64), P(i64), P(i64), P(i64)]
    L.nsm_stats.argtypes = [vp, P(i64), P(i64)]
    L.nsm_halo_plan.argtypes = [P(_Csr), P(_Dist), vp, vp, P(i64)]
    L.nsm_halo_set_send.argtypes = [vp, ci, vp, i64]
    L.nsm_halo_mailbox.argtypes = [vp, P(vp), vp, vp]
    L.nsm_halo_connect_ipc.argtypes = [vp, ci, vp, i64, i64]
    L.nsm_halo_connect.argtypes = [vp, ci, vp, i64, i64]
    L.nsm_halo_commit.argtypes = [vp]
    L.nsm_set_option.argtypes = [vp, ci, i64]
    L.nsm_spmat_setup.argtypes = [P(vp), P(_Csr), ci]
    L.nsm_spmat_apply.argtypes = [vp, vp, vp, ctypes.c_double, ctypes.c_double, vp]
    L.nsm_spmat_destroy.argtypes = [vp]
    L.nsm_spmat_destroy.restype = None
    L.nsm_amg_setup.argtypes = [P(vp), ci, vp, vp, P(_Csr), ci]
    L.nsm_amg_set_smoother.argtypes = [vp, ci, ci, ci, ci, ci, ci]
    L.nsm_amg_vcycle.argtypes = [vp, vp, vp, vp]
    L.nsm_amg_destroy.argtypes = [vp]
    L.nsm_amg_destroy.restype = None
    L.nsm_solver_last_error.argtypes = [vp]
    L.nsm_solver_last_error.restype = ctypes.c_char_p
    L.nsm_gmres.argtypes = [vp, vp, vp, vp, ci, ctypes.c_double, ci, P(ci), vp, vp]
    L.nsm_profile.argtypes = [vp, vp, vp]
    L.nsm_fused_stats.argtypes = [vp, P(i64), P(i64)]
    L.nsm_layout.argtypes = [vp, P(ci)]
    L.nsm_ilut.argtypes = [P(_Csr), ctypes.c_double, ci, vp, P(i64), vp, vp]
    L.nsm_ruiz.argtypes = [P(_Csr), ci, vp, vp, vp]
    L.nsm_set_ruiz.argtypes = [vp, vp, vp]
    L.nsm_last_error.argtypes = [vp]
    L.nsm_last_error.restype = ctypes.c_char_p
    L.nsm_destroy.argtypes = [vp]
    L.nsm_destroy.restype = None
    L.nsm_comm_create.argtypes = [P(vp), ci, ci, i64, ci]
    L.nsm_comm_mailbox.argtypes = [vp, P(vp), vp]
    L.nsm_comm_connect.argtypes = [vp, ci, vp]
    L.nsm_comm_connect_ipc.argtypes = [vp, ci, vp]
    L.nsm_comm_allreduce.argtypes = [vp, vp, vp, i64, vp]
    L.nsm_comm_check.argtypes = [vp, vp]
    L.nsm_comm_set_timeout.argtypes = [vp, i64]
    L.nsm_comm_stats.argtypes = [vp, P(i64)]
    L.nsm_comm_last_error.argtypes = [vp]
    L.nsm_comm_last_error.restype = ctypes.c_char_p
    L.nsm_comm_destroy.argtypes = [vp]
    L.nsm_comm_destroy.restype = None
    L.nsm_set_comm.argtypes = [vp, vp]
    L.nsm_ruiz_dep.argtypes = [P(_Csr), ci, ctypes.c_double, vp, vp, vp, P(ci), vp]
    L.nsm_dep.argtypes = [P(_Csr), vp, ci, vp]
    L.nsm_setup_device.argtypes = [P(vp), P(_Csr), P(_Csr), ci]
    L.nsm_part_info.argtypes = [vp, ci, P(i64), P(i64), P(ci), P(ci)]
    L.nsm_part_copy.argtypes = [vp, ci, vp, vp, vp, vp]
    L.nsm_diag_copy.argtypes = [vp, ci, vp]
    L.nsm_fused_counters.argtypes = [vp, vp]
    L.nsm_coupled_counters.argtypes = [vp, vp]
    for name in ["nsm_setup", "nsm_ilu0", "nsm_ilu0_fixed_point", "nsm_residual", "nsm_spmv", "nsm_lsolve", "nsm_usolve", "nsm_smooth",
                 "nsm_smooth_host", "nsm_check", "nsm_info", "nsm_stats", "nsm_halo_plan", "nsm_halo_set_send", "nsm_halo_mailbox",
                 "nsm_halo_connect_ipc", "nsm_halo_connect", "nsm_halo_commit", "nsm_set_option",
                 "nsm_spmat_setup", "nsm_spmat_apply", "nsm_amg_setup", "nsm_amg_set_smoother", "nsm_amg_vcycle",
                 "nsm_gmres", "nsm_profile", "nsm_ilut", "nsm_ruiz", "nsm_set_ruiz", "nsm_fused_stats", "nsm_layout",
                 "nsm_comm_create", "nsm_comm_mailbox", "nsm_comm_connect", "nsm_comm_connect_ipc",
                 "nsm_comm_allreduce", "nsm_comm_check", "nsm_comm_set_timeout", "nsm_comm_stats", "nsm_set_comm",
                 "nsm_ruiz_dep", "nsm_dep", "nsm_setup_device", "nsm_part_info", "nsm_part_copy", "nsm_diag_copy",
                 "nsm_fused_counters", "nsm_coupled_counters"]:
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def exported_symbols() -> list[str]:
    L = load()
    return [s for s in SYMBOLS if hasattr(L, s)]


def _err(handle) -> str:
    m = load().nsm_last_error(handle)
    return m.decode() if m else ""


def _csr_struct(A, keep: list):
    """A: object with nrows, ncols, rowptr, col, val (numpy)."""
    rp = np.ascontiguousarray(A.rowptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col, dtype=np.int64)
    va = np.ascontiguousarray(A.val, dtype=np.float64)
    keep += [rp, ci, va]
    return _Csr(int(A.nrows), int(A.ncols), rp.ctypes.data, ci.ctypes.data, va.ctypes.data)


class _FactorView:
    def __init__(self, A, fval):
        self.nrows, self.ncols, self.rowptr, self.col = A.nrows, A.ncols, A.rowptr, A.col
        self.val = np.ascontiguousarray(fval, dtype=np.float64)


def ilu0(A, row_begin: int = 0) -> np.ndarray:
    """Host ILU(0) values on A's pattern (nsm_ilu0; strict lower = L_s,
    upper incl. diagonal = U)."""
    L = load()
    keep: list = []
    cs = _csr_struct(A, keep)
    out = np.empty(int(A.rowptr[-1]), dtype=np.float64)
    st = L.nsm_ilu0(ctypes.byref(cs), int(row_begin), out.ctypes.data)
    if st != 0:
        raise NsmError(st, _err(None))
    return out


def ilu0_fixed_point(A, sweeps: int, row_begin: int = 0, device: int = 0) -> np.ndarray:
    """ILU(0) values computed on the GPU by `sweeps` Chow-Patel fixed-point
    sweeps (nsm_ilu0_fixed_point; nsm_ilu0's layout)."""
    L = load()
    keep: list = []
    cs = _csr_struct(A, keep)
    out = np.empty(int(A.rowptr[-1]), dtype=np.float64)
    st = L.nsm_ilu0_fixed_point(ctypes.byref(cs), int(row_begin), int(sweeps), out.ctypes.data, int(device))
    if st != 0:
        raise NsmError(st, _err(None))
    return out


def halo_plan(A, row_offsets, rank: int):
    """Host-only (no device): the ghost columns of this rank's row block,
    grouped by owner.  Returns {q: int64 array of global rows needed from q}."""
    L = load()
    keep: list = []
    cs = _csr_struct(A, keep)
    ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
    nranks = len(ro) - 1
    dist = _Dist(int(rank), int(nranks), ro.ctypes.data, NSM_DIST_HYBRID)
    counts = np.zeros(nranks, dtype=np.int64)
    ng = ctypes.c_int64()
    st = L.nsm_halo_plan(ctypes.byref(cs), ctypes.byref(dist), counts.ctypes.data, None, ctypes.byref(ng))
    if st != 0:
        raise NsmError(st, _err(None))
    rows = np.zeros(ng.value, dtype=np.int64)
    st = L.nsm_halo_plan(ctypes.byref(cs), ctypes.byref(dist), counts.ctypes.data, rows.ctypes.data, ctypes.byref(ng))
    if st != 0:
        raise NsmError(st, _err(None))
    off = np.concatenate([[0], np.cumsum(counts)])
    return {q: rows[off[q]:off[q + 1]] for q in range(nranks) if counts[q] > 0}


def exchange_plan(requests: dict, rank: int, nranks: int, all_gather_object) -> dict:
    """Given this rank's {q: rows needed from q}, return {q: rows q needs from
    this rank}, using a collective `all_gather_object(list_out, obj)` (the
    torch.distributed signature: plumbing only)."""
    allreq = [None] * nranks
    all_gather_object(allreq, {int(q): np.asarray(v, dtype=np.int64) for q, v in requests.items()})
    return {q: allreq[q][rank] for q in range(nranks) if q != rank and rank in allreq[q]}


class FactorCSR:
    """Host factor CSR (strict lower = L_s, upper incl. diagonal = U)."""

    def __init__(self, nrows, rowptr, col, val):
        self.nrows = self.ncols = int(nrows)
        self.rowptr, self.col, self.val = rowptr, col, val


def ilut(A, droptol: float, lfil: int) -> FactorCSR:
    """Host ILUT(droptol, lfil) factors (nsm_ilut)."""
    L = load()
    keep: list = []
    cs = _csr_struct(A, keep)
    n = int(A.nrows)
    rp = np.zeros(n + 1, dtype=np.int64)
    nnz = ctypes.c_int64()
    st = L.nsm_ilut(ctypes.byref(cs), float(droptol), int(lfil), rp.ctypes.data, ctypes.byref(nnz), None, None)
    if st != 0:
        raise NsmError(st, _err(None))
    col = np.zeros(nnz.value, dtype=np.int64)
    val = np.zeros(nnz.value, dtype=np.float64)
    st = L.nsm_ilut(ctypes.byref(cs), float(droptol), int(lfil), rp.ctypes.data, ctypes.byref(nnz),
                    col.ctypes.data, val.ctypes.data)
    if st != 0:
        raise NsmError(st, _err(None))
    return FactorCSR(n, rp, col, val)


def ruiz(F, max_iters: int = 5, dep_tol: float = 0.0, history: bool = False):
    """Ruiz scaling of the U part of a factor CSR (nsm_ruiz; with dep_tol > 0
    or history, nsm_ruiz_dep: early termination on dep(U)).
    Returns (FactorCSR with U~, s_r, s_c) [+ (rounds done, dep history)]."""
    L = load()
    keep: list = []
    cs = _csr_struct(F, keep)
    n = int(F.nrows)
    val = np.zeros(int(F.rowptr[-1]), dtype=np.float64)
    sr, sc = np.zeros(n), np.zeros(n)
    if dep_tol > 0.0 or history:
        its = ctypes.c_int()
        hist = np.zeros(max_iters + 1)
        st = L.nsm_ruiz_dep(ctypes.byref(cs), int(max_iters), float(dep_tol), val.ctypes.data, sr.ctypes.data,
                            sc.ctypes.data, ctypes.byref(its), hist.ctypes.data)
    else:
        st = L.nsm_ruiz(ctypes.byref(cs), int(max_iters), val.ctypes.data, sr.ctypes.data, sc.ctypes.data)
    if st != 0:
        raise NsmError(st, _err(None))
    out = (FactorCSR(n, np.asarray(F.rowptr, np.int64), np.asarray(F.col, np.int64), val), sr, sc)
    if dep_tol > 0.0 or history:
        return out + ((its.value, hist[:its.value + 1]),)
    return out


class _DepInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("dep", ctypes.c_double), ("fro", ctypes.c_double),
                ("fro_strict", ctypes.c_double), ("delta", ctypes.c_double), ("bound_thm3", ctypes.c_double),
                ("bound_table5", ctypes.c_double), ("bound_thm4", ctypes.c_double)]


def dep(F, val=None, upper: bool = True) -> dict:
    """nsm_dep: departure-from-normality diagnostics (Henrici dep, Theorem 3
    and 4 bounds, near diagonal dominance delta) of the U (upper) or unit-L
    part of a factor CSR; val = values on F's pattern (default F.val)."""
    keep: list = []
    cs = _csr_struct(F, keep)
    v = None if val is None else np.ascontiguousarray(val, dtype=np.float64)
    out = _DepInfo()
    st = load().nsm_dep(ctypes.byref(cs), v.ctypes.data if v is not None else None, int(bool(upper)),
                        ctypes.byref(out))
    if st != 0:
        raise NsmError(st, _err(None))
    return {k: getattr(out, k) for k, _ in _DepInfo._fields_}


class Smoother:
    """One nsm handle: the split storage of A (and optionally its ILU(0)
    factors) resident on a CUDA device.  Vectors are float64 CUDA tensors of
    length n_local; calls run on the current torch stream (or `stream`)."""

    def __init__(self, A, F=None, *, device: int | None = None, rank: int = 0, nranks: int = 1,
                 row_offsets=None, mode: int = NSM_DIST_HYBRID):
        import torch  # plumbing: device selection and streams only
        self._torch = torch
        L = load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        keep: list = []
        ca = _csr_struct(A, keep)
        cf = None
        if F is not None:
            Fv = F if hasattr(F, "rowptr") else _FactorView(A, F)
            cf = _csr_struct(Fv, keep)
        dist = None
        if nranks > 1:
            ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
            keep.append(ro)
            dist = _Dist(int(rank), int(nranks), ro.ctypes.data, int(mode))
        h = ctypes.c_void_p()
        st = L.nsm_setup(ctypes.byref(h), ctypes.byref(ca), ctypes.byref(cf) if cf is not None else None,
                         ctypes.byref(dist) if dist is not None else None, self.device)
        if st != 0:
            raise NsmError(st, _err(None))
        self._h = h
        self.has_ilu = F is not None
        self.rank, self.nranks = int(rank), int(nranks)
        self.requests = halo_plan(A, row_offsets, rank) if nranks > 1 else {}
        n, ng, nnz, db = (ctypes.c_int64() for _ in range(4))
        L.nsm_info(h, ctypes.byref(n), ctypes.byref(ng), ctypes.byref(nnz), ctypes.byref(db))
        self.n, self.n_ghost, self.nnz_offdiag, self.device_bytes = n.value, ng.value, nnz.value, db.value

    @classmethod
    def from_device_csr(cls, rowptr, col, val, fval=None, device: int | None = None):
        """nsm_setup_device: a single-rank handle built ON THE GPU from a device
        CSR (torch CUDA tensors: int64 rowptr, int64 col, float64 val; fval =
        the ILU factor values on the same pattern, or None)."""
        import torch
        self = cls.__new__(cls)
        self._torch = torch
        L = load()
        self.device = rowptr.device.index if device is None else int(device)
        for t, dt in ((rowptr, torch.int64), (col, torch.int64), (val, torch.float64)):
            if not (t.is_cuda and t.dtype == dt and t.is_contiguous() and t.device.index == self.device):
                raise TypeError("from_device_csr: contiguous CUDA tensors (int64 rowptr, int64 col, float64 val)")
        n = rowptr.numel() - 1
        ca = _Csr(n, n, rowptr.data_ptr(), col.data_ptr(), val.data_ptr())
        cf = _Csr(n, n, rowptr.data_ptr(), col.data_ptr(), fval.data_ptr()) if fval is not None else None
        h = ctypes.c_void_p()
        st = L.nsm_setup_device(ctypes.byref(h), ctypes.byref(ca), ctypes.byref(cf) if cf is not None else None,
                                self.device)
        if st != 0:
            raise NsmError(st, _err(None))
        self._h = h
        self.has_ilu = fval is not None
        self.rank, self.nranks = 0, 1
        self.requests = {}
        nn, ng, nnz, db = (ctypes.c_int64() for _ in range(4))
        L.nsm_info(h, ctypes.byref(nn), ctypes.byref(ng), ctypes.byref(nnz), ctypes.byref(db))
        self.n, self.n_ghost, self.nnz_offdiag, self.device_bytes = nn.value, ng.value, nnz.value, db.value
        return self

    def part(self, p: int) -> dict:
        """Host copy of device part p (0..7 = L, U, LG, UG, Ls, Us, LsG, UsG)."""
        L = load()
        padded, nnz = ctypes.c_int64(), ctypes.c_int64()
        maxw, al = ctypes.c_int(), ctypes.c_int()
        self._call(L.nsm_part_info(self._h, int(p), ctypes.byref(padded), ctypes.byref(nnz), ctypes.byref(maxw),
                                   ctypes.byref(al)))
        ns = (self.n + 31) // 32
        ptr = np.zeros(ns + 1, dtype=np.int64)
        col = np.zeros(padded.value, dtype=np.int32)
        val = np.zeros(padded.value, dtype=np.float64)
        off = np.zeros(padded.value // 32 if al.value else 0, dtype=np.int32)
        self._call(L.nsm_part_copy(self._h, int(p), ptr.ctypes.data, col.ctypes.data if len(col) else None,
                                   val.ctypes.data if len(val) else None, off.ctypes.data if len(off) else None))
        return {"ptr": ptr, "col": col, "val": val, "off": off, "nnz": nnz.value, "maxw": maxw.value,
                "aligned": bool(al.value)}

    def diag(self, which: int = 0) -> np.ndarray:
        """Host copy of d (0), the l1 diagonal (1) or d_U (2)."""
        out = np.zeros(self.n, dtype=np.float64)
        self._call(load().nsm_diag_copy(self._h, int(which), out.ctypes.data if self.n else None))
        return out

    # -- marshalling helpers ------------------------------------------------
    def _stream(self, stream):
        if stream is None:
            return self._torch.cuda.current_stream(self.device).cuda_stream
        return getattr(stream, "cuda_stream", stream)

    def _vec(self, t, name):
        torch = self._torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                and t.numel() == self.n and t.device.index == self.device):
            raise TypeError(f"{name}: expected a contiguous float64 CUDA tensor of length {self.n} on cuda:{self.device}")
        return t.data_ptr()

    def _new(self):
        return self._torch.empty(self.n, dtype=self._torch.float64, device=f"cuda:{self.device}")

    def _call(self, st):
        if st != 0:
            raise NsmError(st, _err(self._h))

    # -- the C-ABI entry points ----------------------------------------------
    def residual(self, b, x, r=None, stream=None):
        r = self._new() if r is None else r
        self._call(load().nsm_residual(self._h, self._vec(b, "b"), self._vec(x, "x"), self._vec(r, "r"),
                                       self._stream(stream)))
        return r

    def spmv(self, x, y=None, stream=None):
        y = self._new() if y is None else y
        self._call(load().nsm_spmv(self._h, self._vec(x, "x"), self._vec(y, "y"), self._stream(stream)))
        return y

    def lsolve(self, r, k, x=None, stream=None):
        x = self._new() if x is None else x
        self._call(load().nsm_lsolve(self._h, self._vec(r, "r"), self._vec(x, "x"), int(k), self._stream(stream)))
        return x

    def usolve(self, r, k, x=None, stream=None):
        x = self._new() if x is None else x
        self._call(load().nsm_usolve(self._h, self._vec(r, "r"), self._vec(x, "x"), int(k), self._stream(stream)))
        return x

    def smooth(self, b, x, kind="pgs", nu=1, k_l=2, k_u=None, x_is_zero=False, stream=None):
        kd = KINDS[kind] if isinstance(kind, str) else int(kind)
        k_u = k_l if k_u is None else k_u
        self._call(load().nsm_smooth(self._h, kd, self._vec(b, "b"), self._vec(x, "x"), int(nu), int(k_l), int(k_u),
                                     int(bool(x_is_zero)), self._stream(stream)))
        return x

    def smooth_host(self, b, x, kind="pgs", nu=1, k_l=2, k_u=None, x_is_zero=False, stream=None, out=None):
        """nsm_smooth_host: b, x (and out) are host vectors (float64, contiguous,
        length n: numpy arrays or CPU tensors, pinned for full bandwidth).  The
        result goes to `out`, or to x in place when out is None.  Synchronous."""
        kd = KINDS[kind] if isinstance(kind, str) else int(kind)
        k_u = k_l if k_u is None else k_u
        dst = x if out is None else out
        self._call(load().nsm_smooth_host(self._h, kd, self._hvec(b, "b"), self._hvec(x, "x"), self._hvec(dst, "out"),
                                          int(nu), int(k_l), int(k_u), int(bool(x_is_zero)), self._stream(stream)))
        return dst

    def _hvec(self, t, name):
        torch = self._torch
        if isinstance(t, torch.Tensor):
            ok = not t.is_cuda and t.dtype == torch.float64 and t.is_contiguous() and t.numel() == self.n
            ptr = t.data_ptr()
        else:
            import numpy as np
            ok = isinstance(t, np.ndarray) and t.dtype == np.float64 and t.flags.c_contiguous and t.size == self.n
            ptr = t.ctypes.data if ok else 0
        if not ok:
            raise TypeError(f"{name}: expected a contiguous float64 host vector (numpy or CPU tensor) of length {self.n}")
        return ptr

    def check(self, stream=None):
        """Synchronises; returns None, or raises NsmError(NSM_ERR_NONFINITE)."""
        bad = ctypes.c_int64()
        self._call(load().nsm_check(self._h, ctypes.byref(bad), self._stream(stream)))
        return None

    # -- multi-GPU wiring (plumbing around the nsm_halo_* calls) ---------------
    def _neighbours(self, sends):
        return sorted(set(self.requests) | {q for q, v in sends.items() if len(v) > 0})

    def _set_sends(self, sends):
        L = load()
        for q, rows in sends.items():
            rows = np.ascontiguousarray(rows, dtype=np.int64)
            self._call(L.nsm_halo_set_send(self._h, int(q), rows.ctypes.data if len(rows) else None, len(rows)))

    def _mailbox(self):
        base = ctypes.c_void_p()
        ipc = ctypes.create_string_buffer(64)
        offs = np.zeros(self.nranks, dtype=np.int64)
        self._call(load().nsm_halo_mailbox(self._h, ctypes.byref(base), ipc, offs.ctypes.data))
        return base.value, ipc.raw, offs

    def connect(self, dist=None, group=None):
        """Wire the halo exchange across processes (one rank per GPU): the plan
        and the CUDA IPC mailbox handles travel over torch.distributed."""
        if self.nranks == 1:
            return
        if dist is None:
            import torch.distributed as dist
        ago = lambda out, obj: dist.all_gather_object(out, obj, group=group)
        sends = exchange_plan(self.requests, self.rank, self.nranks, ago)
        self._set_sends(sends)
        base, ipc, offs = self._mailbox()
        info = [None] * self.nranks
        ago(info, (ipc, offs, self.n_ghost))
        L = load()
        for q in self._neighbours(sends):
            qipc, qoffs, qng = info[q]
            buf = ctypes.create_string_buffer(qipc, 64)
            self._call(L.nsm_halo_connect_ipc(self._h, int(q), buf, int(qng), int(qoffs[self.rank])))
        self._call(L.nsm_halo_commit(self._h))

    @staticmethod
    def connect_local(ranks):
        """Wire the halo exchange between handles of ONE process on ONE device
        (virtual ranks: tests and single-GPU emulation of a partition)."""
        nranks = len(ranks)
        allreq = [S.requests for S in ranks]
        L = load()
        sends = []
        for S in ranks:
            sd = {q: allreq[q][S.rank] for q in range(nranks) if q != S.rank and S.rank in allreq[q]}
            S._set_sends(sd)
            sends.append(sd)
        boxes = [S._mailbox() for S in ranks]
        for S, sd in zip(ranks, sends):
            for q in S._neighbours(sd):
                qbase, _, qoffs = boxes[q]
                S._call(L.nsm_halo_connect(S._h, int(q), qbase, int(ranks[q].n_ghost), int(qoffs[S.rank])))
        for S in ranks:
            S._call(L.nsm_halo_commit(S._h))

    def set_comm(self, comm: "Comm | None"):
        """Attach the cross-rank reduction used by gmres / Amg on this
        distributed handle (nsm_set_comm; the comm is borrowed: keep it alive)."""
        self._comm = comm
        self._call(load().nsm_set_comm(self._h, comm._h if comm is not None else None))

    def set_ruiz(self, s_r, s_c):
        """Ruiz form of the ILU U solve (the factor must hold U~); None, None = off."""
        if s_r is None:
            self._call(load().nsm_set_ruiz(self._h, None, None))
            return
        sr = np.ascontiguousarray(s_r, dtype=np.float64)
        sc = np.ascontiguousarray(s_c, dtype=np.float64)
        self._call(load().nsm_set_ruiz(self._h, sr.ctypes.data, sc.ctypes.data))

    def set_pipeline(self, enable: bool):
        """Bulk-copy pipelined kernels (default) or the plain ones."""
        self._call(load().nsm_set_option(self._h, 0, int(bool(enable))))

    def set_fused(self, mode):
        """Phase-skewed fused passes: False/0 off (the default), True/1 whenever
        possible, 2 = automatic (large problems), 3 = as 1 plus the one-pass
        windowed pGS on stencil-like matrices (experimental)."""
        self._call(load().nsm_set_option(self._h, 2, int(mode)))

    def set_fused_window(self, items: int):
        """Wait distance of the fused passes in work items (0 = automatic)."""
        self._call(load().nsm_set_option(self._h, 5, int(items)))

    def set_window(self, enable: bool):
        """NSM_OPT_WINDOW: shared-memory gather windows in the pipelined kernels."""
        self._call(load().nsm_set_option(self._h, 6, int(bool(enable))))

    def set_plane_rows(self, rows: int):
        """NSM_OPT_PLANE_ROWS: declare planes of `rows` rows (a multiple of 256)
        for the plane-wavefront one-pass pGS (checked; NsmError if the matrix
        lacks the structure)."""
        self._call(load().nsm_set_option(self._h, 7, int(rows)))

    def set_host_chunks(self, enable: bool):
        """NSM_OPT_HOST_CHUNKS: nsm_smooth_host overlaps copies and passes in row chunks."""
        self._call(load().nsm_set_option(self._h, 8, int(bool(enable))))

    def set_coupled(self, mode):
        """NSM_OPT_COUPLED: the k = 2, 3 sweeps of a forward pGS application on
        windowed stencil matrices as concurrent CTA groups of one kernel (True/1,
        experimental), the per-pass kernels (False/0, the default), or on with a
        throttle distance of `mode` tiles (> 1)."""
        self._call(load().nsm_set_option(self._h, 9, int(mode)))

    def set_pdl(self, enable: bool):
        """Programmatic dependent launch between consecutive pipelined kernels."""
        self._call(load().nsm_set_option(self._h, 3, int(bool(enable))))

    def set_profile(self, enable: bool):
        """Record an event pair around every residual / sweep pass."""
        self._call(load().nsm_set_option(self._h, 4, int(bool(enable))))

    def profile(self):
        """{'residual' | 'sweep' | 'fused': (ms, count)} since the last call."""
        ms = np.zeros(3)
        cnt = np.zeros(3, dtype=np.int64)
        self._call(load().nsm_profile(self._h, ms.ctypes.data, cnt.ctypes.data))
        return {"residual": (float(ms[0]), int(cnt[0])), "sweep": (float(ms[1]), int(cnt[1])),
                "fused": (float(ms[2]), int(cnt[2]))}

    def layout(self):
        """{'L', 'U', 'Ls', 'Us'}: which strict parts use the offset-aligned layout."""
        v = ctypes.c_int(0)
        self._call(load().nsm_layout(self._h, ctypes.byref(v)))
        return {k: bool(v.value & b) for k, b in (("L", 1), ("U", 2), ("Ls", 4), ("Us", 8))}

    def windows(self):
        """{'residual', 'L', 'U'}: which gather windows exist (the windowed kernels run)."""
        v = ctypes.c_int(0)
        self._call(load().nsm_layout(self._h, ctypes.byref(v)))
        return {k: bool(v.value & b) for k, b in (("residual", 16), ("L", 32), ("U", 64))}

    def fused_stats(self):
        """(waits that had to spin, total spin ns) of the fused passes since setup."""
        w, t = ctypes.c_int64(0), ctypes.c_int64(0)
        self._call(load().nsm_fused_stats(self._h, ctypes.byref(w), ctypes.byref(t)))
        return int(w.value), int(t.value)

    def fused_counters(self) -> np.ndarray:
        """nsm_fused_counters: polls, poll ns, stage-wait ns, readiness ns, unit ns, fences."""
        out = np.zeros(6, dtype=np.int64)
        self._call(load().nsm_fused_counters(self._h, out.ctypes.data))
        return out

    def coupled_counters(self) -> np.ndarray:
        """nsm_coupled_counters: per sweep group g, [4g..4g+3] = producer cycles in
        dependency waits, producer cycles waiting for a stage, producer cycles in
        total, consumer (warp 0) cycles waiting for staged data (NSM_OPT_PROFILE on)."""
        out = np.zeros(16, dtype=np.int64)
        self._call(load().nsm_coupled_counters(self._h, out.ctypes.data))
        return out

    def set_halo_timeout(self, ms: int):
        """How long a halo wait spins before reporting NSM_ERR_DIST."""
        self._call(load().nsm_set_option(self._h, 1, int(ms)))

    def stats(self):
        """(kernel launches, halo exchanges) since setup."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._call(load().nsm_stats(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def close(self):
        if getattr(self, "_h", None):
            load().nsm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


# ----------------------------------------------------------- solver layer --
def _solver_err(h=None) -> str:
    m = load().nsm_solver_last_error(h)
    return m.decode() if m else ""


class Comm:
    """Device-side all-reduce across the ranks of a row-block partition
    (nsm_comm: Algorithm 1's one global reduction per iteration, over
    NVLink / NVSwitch peer memory; sums in ascending rank order)."""

    def __init__(self, rank: int, nranks: int, capacity: int, device: int | None = None):
        import torch
        self._torch = torch
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.rank, self.nranks, self.capacity = int(rank), int(nranks), int(capacity)
        h = ctypes.c_void_p()
        st = load().nsm_comm_create(ctypes.byref(h), self.rank, self.nranks, self.capacity, self.device)
        if st != 0:
            raise NsmError(st, load().nsm_comm_last_error(None).decode())
        self._h = h

    def _call(self, st):
        if st != 0:
            raise NsmError(st, load().nsm_comm_last_error(self._h).decode())

    def _mailbox(self):
        base = ctypes.c_void_p()
        ipc = ctypes.create_string_buffer(64)
        self._call(load().nsm_comm_mailbox(self._h, ctypes.byref(base), ipc))
        return base.value, ipc.raw

    def connect(self, dist=None, group=None):
        """Across processes (one rank per GPU): the IPC handles travel over
        torch.distributed (plumbing)."""
        if self.nranks == 1:
            return
        if dist is None:
            import torch.distributed as dist
        _, ipc = self._mailbox()
        info = [None] * self.nranks
        dist.all_gather_object(info, ipc, group=group)
        for q in range(self.nranks):
            if q != self.rank:
                self._call(load().nsm_comm_connect_ipc(self._h, q, ctypes.create_string_buffer(info[q], 64)))

    @staticmethod
    def connect_local(comms):
        """Ranks of ONE process (virtual ranks): plain device pointers."""
        boxes = [c._mailbox()[0] for c in comms]
        for c in comms:
            for q, b in enumerate(boxes):
                if q != c.rank:
                    c._call(load().nsm_comm_connect(c._h, q, b))

    def allreduce(self, x, out=None, stream=None):
        torch = self._torch
        out = torch.empty_like(x) if out is None else out
        s = torch.cuda.current_stream(self.device).cuda_stream if stream is None else getattr(stream, "cuda_stream", stream)
        self._call(load().nsm_comm_allreduce(self._h, x.data_ptr(), out.data_ptr(), x.numel(), s))
        return out

    def check(self, stream=None):
        torch = self._torch
        s = torch.cuda.current_stream(self.device).cuda_stream if stream is None else getattr(stream, "cuda_stream", stream)
        self._call(load().nsm_comm_check(self._h, s))

    def set_timeout(self, ms: int):
        self._call(load().nsm_comm_set_timeout(self._h, int(ms)))

    def stats(self) -> int:
        v = ctypes.c_int64()
        self._call(load().nsm_comm_stats(self._h, ctypes.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "_h", None):
            load().nsm_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SpMat:
    """Device CSR (rectangular allowed): y = alpha * M x + beta * y."""

    def __init__(self, M, device: int | None = None):
        import torch
        self._torch = torch
        self.device = torch.cuda.current_device() if device is None else int(device)
        keep: list = []
        cs = _csr_struct(M, keep)
        h = ctypes.c_void_p()
        st = load().nsm_spmat_setup(ctypes.byref(h), ctypes.byref(cs), self.device)
        if st != 0:
            raise NsmError(st, _solver_err())
        self._h, self.shape = h, (int(M.nrows), int(M.ncols))

    def apply(self, x, y=None, alpha=1.0, beta=0.0, stream=None):
        torch = self._torch
        if y is None:
            y = torch.zeros(self.shape[0], dtype=torch.float64, device=f"cuda:{self.device}")
        st = load().nsm_spmat_apply(self._h, x.data_ptr(), y.data_ptr(), float(alpha), float(beta),
                                    torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream)
        if st != 0:
            raise NsmError(st, "nsm_spmat_apply")
        return y

    def close(self):
        if getattr(self, "_h", None):
            load().nsm_spmat_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Amg:
    """GPU V-cycle over a caller-built hierarchy: smoothers = [Smoother of A_l],
    P = [host CSR A_l -> A_{l+1}], coarse = host CSR of the coarsest matrix."""

    def __init__(self, smoothers, P, coarse, device: int | None = None):
        import torch
        self._torch = torch
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.smoothers = list(smoothers)  # keep the borrowed handles alive
        keep: list = []
        nl = len(self.smoothers)
        hs = (ctypes.c_void_p * max(nl, 1))(*[S._h for S in self.smoothers])
        ps = [_csr_struct(p, keep) for p in P]
        parr = (ctypes.POINTER(_Csr) * max(nl, 1))(*[ctypes.pointer(p) for p in ps])
        cc = _csr_struct(coarse, keep)
        h = ctypes.c_void_p()
        st = load().nsm_amg_setup(ctypes.byref(h), nl, ctypes.cast(hs, ctypes.c_void_p),
                                  ctypes.cast(parr, ctypes.c_void_p), ctypes.byref(cc), self.device)
        if st != 0:
            raise NsmError(st, _solver_err())
        self._h = h
        self.n = self.smoothers[0].n if nl else int(coarse.nrows)

    def set_smoother(self, level, kind="pgs", nu_pre=1, nu_post=1, k_l=2, k_u=2):
        kd = KINDS[kind] if isinstance(kind, str) else int(kind)
        st = load().nsm_amg_set_smoother(self._h, int(level), kd, int(nu_pre), int(nu_post), int(k_l), int(k_u))
        if st != 0:
            raise NsmError(st, "nsm_amg_set_smoother")

    def vcycle(self, b, x=None, stream=None):
        torch = self._torch
        x = torch.empty_like(b) if x is None else x
        st = load().nsm_amg_vcycle(self._h, b.data_ptr(), x.data_ptr(),
                                   torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream)
        if st != 0:
            raise NsmError(st, _solver_err(self._h))
        return x

    def close(self):
        if getattr(self, "_h", None):
            load().nsm_amg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gmres(A: "Smoother", b, amg: "Amg | None" = None, tol: float = 1e-5, maxit: int = 200, t_mode: str = "neumann",
          stream=None):
    """Algorithm 1 on the device.  Returns (x, iterations, implicit relres history)."""
    import torch
    x = torch.empty_like(b)
    hist = np.zeros(maxit + 1)
    its = ctypes.c_int()
    tm = {"neumann": 0, "inverse": 1}[t_mode]
    st = load().nsm_gmres(A._h, amg._h if amg is not None else None, b.data_ptr(), x.data_ptr(), int(maxit),
                          float(tol), tm, ctypes.byref(its), hist.ctypes.data,
                          torch.cuda.current_stream(A.device).cuda_stream if stream is None else stream)
    if st != 0:
        raise NsmError(st, _solver_err())
    return x, its.value, hist[:its.value + 1]
