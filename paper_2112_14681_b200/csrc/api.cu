// api.cu — the C-ABI of libnsm.so (include/nsm.h).
//
// Owns the handle (device copies of the split storage + workspace) and
// turns each nsm_* call into a fixed sequence of kernel launches on the
// caller's stream (no allocation, no host synchronisation on hot calls).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>

#include "nsm_internal.h"

using namespace nsm;

struct nsm_handle {
    int device = 0;
    int64_t n = 0, row_begin = 0, n_ghost = 0, nnz_off = 0, device_bytes = 0;
    int nslices = 0;
    int rank = 0, nranks = 1;
    nsm_dist_mode mode = NSM_DIST_HYBRID;
    // A = L + D + U (+ ghost couplings LG / UG)
    double *d = nullptr;
    Sell L, U, LG, UG;
    // ILU(0) factors: unit-lower L = I + Ls, U = D_U (I + D_U^{-1} Us)
    bool has_ilu = false;
    double *dU = nullptr;
    Sell Ls, Us, LsG, UsG;
    // workspace: three n-vectors, ghost values, divergence flag
    double *w[3] = {nullptr, nullptr, nullptr};
    double *ghost = nullptr;
    unsigned long long *flag = nullptr;
    int64_t sweep_counter = 0;
    int64_t launches = 0, exchanges = 0;
    std::string err;
};

namespace {

thread_local std::string g_setup_err;

struct DevAlloc {
    nsm_handle *h;
    template <class T>
    bool get(T **p, int64_t count) {
        *p = nullptr;
        if (count <= 0) return true;
        size_t bytes = (size_t)count * sizeof(T);
        if (cudaMalloc((void **)p, bytes) != cudaSuccess) { *p = nullptr; return false; }
        h->device_bytes += (int64_t)bytes;
        return true;
    }
};

template <class T>
bool upload(T *dst, const T *src, int64_t count) {
    if (count <= 0) return true;
    return cudaMemcpy(dst, src, (size_t)count * sizeof(T), cudaMemcpyHostToDevice) == cudaSuccess;
}

bool upload_sell(DevAlloc &a, const SellHost &hs, Sell *s) {
    s->padded = (int64_t)hs.col.size();
    s->nnz = hs.nnz;
    s->maxw = hs.maxw;
    if (!a.get(&s->ptr, (int64_t)hs.ptr.size())) return false;
    if (!upload(s->ptr, hs.ptr.data(), (int64_t)hs.ptr.size())) return false;
    if (!a.get(&s->col, s->padded) || !a.get(&s->val, s->padded)) return false;
    return upload(s->col, hs.col.data(), s->padded) && upload(s->val, hs.val.data(), s->padded);
}

void free_sell(Sell &s) {
    cudaFree(s.ptr);
    cudaFree(s.col);
    cudaFree(s.val);
    s = Sell();
}

void free_handle(nsm_handle *h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    for (Sell *s : {&h->L, &h->U, &h->LG, &h->UG, &h->Ls, &h->Us, &h->LsG, &h->UsG}) free_sell(*s);
    cudaFree(h->d);
    cudaFree(h->dU);
    for (double *&p : h->w) cudaFree(p);
    cudaFree(h->ghost);
    cudaFree(h->flag);
    delete h;
}

nsm_status cuda_fail(nsm_handle *h, cudaError_t e, const char *where) {
    h->err = std::string(where) + ": " + cudaGetErrorString(e);
    return NSM_ERR_CUDA;
}

inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

bool overlap(const double *a, const double *b, int64_t n) {
    return a && b && a < b + n && b < a + n;
}

// One stage of the Jacobi-iterated solve: k sweeps on T from g^(0) = rhs / dT
// (gin_scaled first sweep), writing the final iterate with epilogue `epi`.
// bufs: two scratch vectors for the ping-pong, distinct from rhs.
struct Stage {
    const Sell *T;
    const double *dT;    // nullptr = unit diagonal
    const double *rhs;
    int k;
};

nsm_status run_sweeps(nsm_handle *h, const Stage &st, double *bufA, double *bufB, int last_epi, double *last_out,
                      double *x, const double *dnext, double *gout2, cudaStream_t s) {
    // k >= 1 required here; k == 0 is handled by the caller (scale kernels).
    const double *gin = nullptr;
    for (int j = 1; j <= st.k; ++j) {
        const bool last = j == st.k;
        SweepArgs a{};
        a.n = h->n;
        a.nslices = h->nslices;
        a.list = nullptr;
        a.T = st.T;
        a.TG = nullptr;
        a.has_ghost = false;
        a.unit = st.dT == nullptr;
        a.epi = last ? last_epi : EPI_STORE;
        a.gin_scaled = j == 1;
        a.dT = st.dT;
        a.rhs = st.rhs;
        a.gin = gin;
        a.ghost = h->ghost;
        double *out = last ? last_out : ((j & 1) ? bufA : bufB);
        a.gout = out;
        a.x = x;
        a.dnext = dnext;
        a.gout2 = gout2;
        a.flag = h->flag;
        a.sweep_id = ++h->sweep_counter;
        cudaError_t e = launch_sweep(a, s);
        if (e != cudaSuccess) return cuda_fail(h, e, "sweep launch");
        ++h->launches;
        gin = out;
    }
    return NSM_OK;
}

nsm_status residual_into(nsm_handle *h, const double *b, const double *x, double *out, bool spmv, cudaStream_t s) {
    cudaError_t e = launch_residual(spmv, h->n, h->nslices, nullptr, h->LG, h->L, h->U, h->UG, h->n_ghost > 0,
                                    h->d, b, x, h->ghost, out, s);
    if (h->n > 0) ++h->launches;
    return e == cudaSuccess ? NSM_OK : cuda_fail(h, e, "residual launch");
}

}  // namespace

extern "C" {

const char *nsm_last_error(const nsm_handle *h) { return h ? h->err.c_str() : g_setup_err.c_str(); }

nsm_status nsm_ilu0(const nsm_csr *A, int64_t row_begin, double *fval) {
    if (!A || !fval) { g_setup_err = "nsm_ilu0: NULL argument"; return NSM_ERR_ARG; }
    return ilu0_host(A, row_begin, fval, &g_setup_err);
}

nsm_status nsm_setup(nsm_handle **out, const nsm_csr *A, const nsm_csr *F, const nsm_dist *dist, int device) {
    if (!out || !A) { g_setup_err = "nsm_setup: NULL argument"; return NSM_ERR_ARG; }
    *out = nullptr;
    int64_t rb = 0, re = A->nrows;
    if (dist && dist->nranks > 1) {
        g_setup_err = "nsm_setup: multi-rank handles are not built by this entry point yet";
        return NSM_ERR_DIST;
    }
    if (A->ncols != A->nrows) { g_setup_err = "nsm_setup: A must be square on one rank"; return NSM_ERR_ARG; }
    Split sa, sf;
    nsm_status st = build_split(A, rb, re, &sa, &g_setup_err);
    if (st != NSM_OK) return st;
    if (F) {
        if (F->nrows != A->nrows || F->ncols != A->ncols) { g_setup_err = "nsm_setup: F shape differs from A"; return NSM_ERR_ARG; }
        st = build_split(F, rb, re, &sf, &g_setup_err);
        if (st != NSM_OK) { g_setup_err = "factor: " + g_setup_err; return st; }
    }
    if (cudaSetDevice(device) != cudaSuccess) { g_setup_err = "nsm_setup: cudaSetDevice failed"; return NSM_ERR_CUDA; }
    nsm_handle *h = new nsm_handle();
    h->device = device;
    h->n = sa.n;
    h->row_begin = rb;
    h->n_ghost = sa.n_ghost;
    h->nnz_off = sa.nnz_off;
    h->nslices = (int)((sa.n + kSlice - 1) / kSlice);
    DevAlloc a{h};
    bool ok = a.get(&h->d, h->n) && upload(h->d, sa.d.data(), h->n) && upload_sell(a, sa.L, &h->L) &&
              upload_sell(a, sa.U, &h->U) && upload_sell(a, sa.LG, &h->LG) && upload_sell(a, sa.UG, &h->UG);
    if (ok && F) {
        h->has_ilu = true;
        ok = a.get(&h->dU, h->n) && upload(h->dU, sf.d.data(), h->n) && upload_sell(a, sf.L, &h->Ls) &&
             upload_sell(a, sf.U, &h->Us) && upload_sell(a, sf.LG, &h->LsG) && upload_sell(a, sf.UG, &h->UsG);
    }
    for (int i = 0; ok && i < 3; ++i) ok = a.get(&h->w[i], std::max<int64_t>(h->n, 1));
    ok = ok && a.get(&h->ghost, std::max<int64_t>(h->n_ghost, 1)) && a.get(&h->flag, 1);
    if (ok) {
        unsigned long long init = ULLONG_MAX;
        ok = cudaMemcpy(h->flag, &init, sizeof(init), cudaMemcpyHostToDevice) == cudaSuccess;
    }
    if (!ok) {
        cudaGetLastError();
        g_setup_err = "nsm_setup: device allocation or upload failed";
        free_handle(h);
        return NSM_ERR_OOM;
    }
    *out = h;
    return NSM_OK;
}

void nsm_destroy(nsm_handle *h) { free_handle(h); }

nsm_status nsm_info(const nsm_handle *h, int64_t *n_local, int64_t *n_ghost, int64_t *nnz_offdiag,
                    int64_t *device_bytes) {
    if (!h) return NSM_ERR_ARG;
    if (n_local) *n_local = h->n;
    if (n_ghost) *n_ghost = h->n_ghost;
    if (nnz_offdiag) *nnz_offdiag = h->nnz_off;
    if (device_bytes) *device_bytes = h->device_bytes;
    return NSM_OK;
}

nsm_status nsm_stats(const nsm_handle *h, int64_t *kernel_launches, int64_t *halo_exchanges) {
    if (!h) return NSM_ERR_ARG;
    if (kernel_launches) *kernel_launches = h->launches;
    if (halo_exchanges) *halo_exchanges = h->exchanges;
    return NSM_OK;
}

nsm_status nsm_residual(nsm_handle *h, const double *b, const double *x, double *r, void *stream) {
    if (!h) return NSM_ERR_ARG;
    if ((h->n > 0 && (!b || !x || !r)) || overlap(r, b, h->n) || overlap(r, x, h->n)) {
        h->err = "nsm_residual: NULL or aliased vector";
        return NSM_ERR_ARG;
    }
    return residual_into(h, b, x, r, false, S(stream));
}

nsm_status nsm_spmv(nsm_handle *h, const double *x, double *y, void *stream) {
    if (!h) return NSM_ERR_ARG;
    if ((h->n > 0 && (!x || !y)) || overlap(x, y, h->n)) { h->err = "nsm_spmv: NULL or aliased vector"; return NSM_ERR_ARG; }
    return residual_into(h, nullptr, x, y, true, S(stream));
}

static nsm_status tri_solve(nsm_handle *h, bool lower, const double *r, double *x, int k, void *stream) {
    if (!h) return NSM_ERR_ARG;
    if (k < 0 || (h->n > 0 && (!r || !x)) || overlap(r, x, h->n)) {
        h->err = lower ? "nsm_lsolve: bad argument (k < 0, NULL or aliased vector)"
                       : "nsm_usolve: bad argument (k < 0, NULL or aliased vector)";
        return NSM_ERR_ARG;
    }
    cudaStream_t s = S(stream);
    const Sell *T;
    const double *dT;
    if (h->has_ilu) { T = lower ? &h->Ls : &h->Us; dT = lower ? nullptr : h->dU; }
    else { T = lower ? &h->L : &h->U; dT = h->d; }
    if (k == 0) {
        cudaError_t e = launch_scale(false, h->n, r, dT, x, h->flag, ++h->sweep_counter, s);
        if (h->n > 0) ++h->launches;
        return e == cudaSuccess ? NSM_OK : cuda_fail(h, e, "scale launch");
    }
    return run_sweeps(h, Stage{T, dT, r, k}, h->w[0], h->w[1], EPI_STORE, x, nullptr, nullptr, nullptr, s);
}

nsm_status nsm_lsolve(nsm_handle *h, const double *r, double *x, int k, void *stream) {
    return tri_solve(h, true, r, x, k, stream);
}
nsm_status nsm_usolve(nsm_handle *h, const double *r, double *x, int k, void *stream) {
    return tri_solve(h, false, r, x, k, stream);
}

nsm_status nsm_smooth(nsm_handle *h, nsm_kind kind, const double *b, double *x, int nu, int k_l, int k_u,
                      int x_is_zero, void *stream) {
    if (!h) return NSM_ERR_ARG;
    if (nu < 0 || k_l < 0 || (kind == NSM_ILU0 && k_u < 0) || (h->n > 0 && (!b || !x)) || overlap(b, x, h->n)) {
        h->err = "nsm_smooth: bad argument (negative count, NULL or aliased vector)";
        return NSM_ERR_ARG;
    }
    if (kind != NSM_PGS && kind != NSM_ILU0) { h->err = "nsm_smooth: unknown kind"; return NSM_ERR_ARG; }
    if (kind == NSM_ILU0 && !h->has_ilu) { h->err = "nsm_smooth: ILU0 requested on a handle without factors"; return NSM_ERR_STATE; }
    cudaStream_t s = S(stream);
    double *R = h->w[0], *W0 = h->w[1], *W1 = h->w[2];
    for (int it = 0; it < nu; ++it) {
        // row a2: residual; x == 0 => r = b exactly (reading R3)
        const double *rhs = b;
        if (!(it == 0 && x_is_zero)) {
            nsm_status st = residual_into(h, b, x, R, false, s);
            if (st != NSM_OK) return st;
            rhs = R;
        }
        nsm_status st = NSM_OK;
        if (kind == NSM_PGS) {
            // rows a3/a4: k_l sweeps g <- D^{-1}(r - L g), last one fused with x += g
            if (k_l == 0) {
                cudaError_t e = launch_scale(true, h->n, rhs, h->d, x, h->flag, ++h->sweep_counter, s);
                if (h->n > 0) ++h->launches;
                if (e != cudaSuccess) return cuda_fail(h, e, "scale launch");
            } else {
                st = run_sweeps(h, Stage{&h->L, h->d, rhs, k_l}, W0, W1, EPI_XADD, nullptr, x, nullptr, nullptr, s);
            }
        } else {
            // row a5: y = sum_{j<=kL} (-Ls)^j r ; z = sum_{j<=kU} (-DU^{-1}Us)^j DU^{-1} y ; x += z
            const double *y = rhs;
            double *ybuf = nullptr;
            if (k_l > 0) {
                // L sweeps ping-pong in W0/W1; the last writes y (and z0 = y/dU if k_u >= 1
                // is gathered on the fly by the first U sweep, so only y is stored)
                ybuf = (k_l & 1) ? W0 : W1;
                if (k_u == 0)
                    st = run_sweeps(h, Stage{&h->Ls, nullptr, rhs, k_l}, W0, W1, EPI_XADD_SCALE, nullptr, x, h->dU,
                                    nullptr, s);
                else
                    st = run_sweeps(h, Stage{&h->Ls, nullptr, rhs, k_l}, W0, W1, EPI_STORE, ybuf, nullptr, nullptr,
                                    nullptr, s);
                if (st != NSM_OK) return st;
                y = ybuf;
            } else if (k_u == 0) {
                cudaError_t e = launch_scale(true, h->n, rhs, h->dU, x, h->flag, ++h->sweep_counter, s);
                if (h->n > 0) ++h->launches;
                if (e != cudaSuccess) return cuda_fail(h, e, "scale launch");
            }
            if (k_u > 0) {
                // scratch for the z ping-pong: the two work vectors not holding y
                // (R is free once the L stage has consumed the residual)
                double *za, *zb;
                if (y == W0) { za = R; zb = W1; }
                else if (y == W1) { za = R; zb = W0; }
                else { za = W0; zb = W1; }
                st = run_sweeps(h, Stage{&h->Us, h->dU, y, k_u}, za, zb, EPI_XADD, nullptr, x, nullptr, nullptr, s);
            }
        }
        if (st != NSM_OK) return st;
    }
    return NSM_OK;
}

nsm_status nsm_check(nsm_handle *h, int64_t *first_bad_sweep, void *stream) {
    if (!h) return NSM_ERR_ARG;
    cudaError_t e = cudaStreamSynchronize(S(stream));
    if (e != cudaSuccess) return cuda_fail(h, e, "nsm_check");
    unsigned long long v = 0, init = ULLONG_MAX;
    e = cudaMemcpy(&v, h->flag, sizeof(v), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(h->flag, &init, sizeof(init), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(h, e, "nsm_check");
    if (first_bad_sweep) *first_bad_sweep = v == ULLONG_MAX ? -1 : (int64_t)v;
    if (v != ULLONG_MAX) {
        h->err = "non-finite value produced by sweep " + std::to_string((long long)v);
        return NSM_ERR_NONFINITE;
    }
    return NSM_OK;
}

}  // extern "C"
