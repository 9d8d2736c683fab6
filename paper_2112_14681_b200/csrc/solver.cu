// solver.cu — the GPU-resident solver around the smoothers (SURVEY.md §8(f)
// NEXT-1 / NEXT-2): transfer operators, the C-AMG V(1,1) cycle with the
// Neumann-series smoothers on every level, and the paper's one-reduce
// truncated-Neumann MGS-GMRES (Algorithm 1).
//
// Everything on the vectors runs in this file's kernels or the smoother
// handles; the host keeps only the small (k x k) Arnoldi / correction
// matrices and performs ONE device->host read per GMRES iteration — the
// single global reduction of Algorithm 1 step 6.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "nsm_internal.h"

using namespace nsm;

// ------------------------------------------------------------------ kernels --
namespace {

constexpr int kThr = 256;

// programmatic dependent launch (see kernels.cu): wait for the predecessor
// before touching memory, then let dependents be scheduled
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" :::);
}
template <class K, class... Args>
cudaError_t launch_pdl(K kernel, unsigned grid, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThr);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// y = alpha * M x + beta * y   (CSR, one thread per row, ascending columns)
__global__ void __launch_bounds__(kThr) k_csr_spmv(int64_t nrows, const int64_t *__restrict__ rp,
                                                   const int32_t *__restrict__ ci, const double *__restrict__ va,
                                                   const double *__restrict__ x, double *__restrict__ y, double alpha,
                                                   double beta) {
    pdl_enter();
    const int64_t i = (int64_t)blockIdx.x * kThr + threadIdx.x;
    if (i >= nrows) return;
    double s = 0.0;
    // chunks of 8 entries: loads and gathers issued together, products added
    // in ascending column order (the order of the one-by-one loop)
    constexpr int C = 8;
    for (int64_t p0 = __ldg(rp + i), e = __ldg(rp + i + 1); p0 < e; p0 += C) {
        double pr[C];
#pragma unroll
        for (int t = 0; t < C; ++t)
            if (p0 + t < e) pr[t] = __dmul_rn(__ldg(va + p0 + t), __ldg(x + __ldg(ci + p0 + t)));
#pragma unroll
        for (int t = 0; t < C; ++t)
            if (p0 + t < e) s = __dadd_rn(s, pr[t]);
    }
    const double v = __dmul_rn(alpha, s);
    y[i] = beta == 0.0 ? v : __dadd_rn(v, __dmul_rn(beta, y[i]));
}

// the same for small operators with wide rows (restriction R = P^T onto a
// coarse level): one warp per row, products of 32 entries at once, added in
// ascending column order through shuffles (bit-identical to k_csr_spmv)
__global__ void __launch_bounds__(kThr) k_csr_spmv_wide(int64_t nrows, const int64_t *__restrict__ rp,
                                                        const int32_t *__restrict__ ci,
                                                        const double *__restrict__ va, const double *__restrict__ x,
                                                        double *__restrict__ y, double alpha, double beta) {
    pdl_enter();
    const int64_t i = ((int64_t)blockIdx.x * kThr + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= nrows) return;
    double s = 0.0;
    const int64_t b = __ldg(rp + i), e = __ldg(rp + i + 1);
    for (int64_t p0 = b; p0 < e; p0 += 32) {
        const int64_t p = p0 + lane;
        const double pr = p < e ? __dmul_rn(__ldg(va + p), __ldg(x + __ldg(ci + p))) : 0.0;
        const int m = (int)(e - p0 < 32 ? e - p0 : 32);
        for (int t = 0; t < m; ++t) s = __dadd_rn(s, __shfl_sync(0xffffffffu, pr, t));
    }
    if (lane != 0) return;
    const double v = __dmul_rn(alpha, s);
    y[i] = beta == 0.0 ? v : __dadd_rn(v, __dmul_rn(beta, y[i]));
}

// y = Minv x, dense row-major n x n (coarse-level solve): one warp per row
__global__ void __launch_bounds__(kThr) k_dense_gemv(int n, const double *__restrict__ Minv,
                                                     const double *__restrict__ x, double *__restrict__ y) {
    pdl_enter();
    const int row = (int)(((int64_t)blockIdx.x * kThr + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (row >= n) return;
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s += __ldg(Minv + (int64_t)row * n + j) * __ldg(x + j);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[row] = s;
}

// Fused multi-dot (Algorithm 1 step 6, K4 of SURVEY.md §2.2): for j < nb,
// part[blk][2j] = sum_rows V_j u, part[blk][2j+1] = sum_rows V_j w, and the
// last pair (j = nb) with u itself: u.u, u.w.  V is read once; the block's
// chunk of u and w stays in L1.  Deterministic: fixed per-block order, then
// k_sum_parts adds the blocks in order.
__global__ void __launch_bounds__(kThr) k_multidot(int64_t n, int nb, const double *__restrict__ V,
                                                   const double *__restrict__ u, const double *__restrict__ w,
                                                   double *__restrict__ part) {
    __shared__ double red[2][kThr / 32];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(n, r0 + chunk);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int j = 0; j <= nb; ++j) {
        const double *vj = j < nb ? V + (int64_t)j * n : u;
        double su = 0.0, sw = 0.0;
        for (int64_t i = r0 + threadIdx.x; i < r1; i += kThr) {
            const double v = __ldg(vj + i);
            su += v * __ldg(u + i);
            sw += v * __ldg(w + i);
        }
        for (int o = 16; o; o >>= 1) {
            su += __shfl_xor_sync(0xffffffffu, su, o);
            sw += __shfl_xor_sync(0xffffffffu, sw, o);
        }
        if (lane == 0) { red[0][wid] = su; red[1][wid] = sw; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = 0.0, c = 0.0;
            for (int q = 0; q < kThr / 32; ++q) { a += red[0][q]; c += red[1][q]; }
            part[(int64_t)blockIdx.x * 2 * (nb + 1) + 2 * j] = a;
            part[(int64_t)blockIdx.x * 2 * (nb + 1) + 2 * j + 1] = c;
        }
        __syncthreads();
    }
}

__global__ void k_sum_parts(int nblk, int m, const double *__restrict__ part, double *__restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * m + j];
    out[j] = s;
}

// out = alpha * w - sum_{j < nb} V_j h_j   (Algorithm 1 step 12; V read once)
// (w may be null: out = -sum ..., used with alpha = 0 / h negated for V y)
__global__ void __launch_bounds__(kThr) k_multiaxpy(int64_t n, int nb, const double *__restrict__ V,
                                                    const double *__restrict__ h, double alpha,
                                                    const double *__restrict__ w, double *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * kThr + threadIdx.x;
    if (i >= n) return;
    double s = w ? alpha * w[i] : 0.0;
    for (int j = 0; j < nb; ++j) s -= __ldg(V + (int64_t)j * n + i) * __ldg(h + j);
    out[i] = s;
}

// out = a * x
__global__ void __launch_bounds__(kThr) k_scal(int64_t n, double a, const double *__restrict__ x,
                                               double *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * kThr + threadIdx.x;
    if (i < n) out[i] = a * x[i];
}

inline unsigned blocks(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kThr - 1) / kThr); }

}  // namespace

// Load every solver kernel now (lazy module loading synchronises the context:
// a first launch while a peer rank's halo / reduction wait spins on this
// device would stall until the timeout).
void nsm::preload_solver_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_csr_spmv);
    cudaFuncGetAttributes(&a, k_csr_spmv_wide);
    cudaFuncGetAttributes(&a, k_dense_gemv);
    cudaFuncGetAttributes(&a, k_multidot);
    cudaFuncGetAttributes(&a, k_sum_parts);
    cudaFuncGetAttributes(&a, k_multiaxpy);
    cudaFuncGetAttributes(&a, k_scal);
}

// ------------------------------------------------------------ sparse matrix --
struct nsm_spmat {
    int device = 0;
    int64_t nrows = 0, ncols = 0, nnz = 0, maxrow = 0;
    int64_t *rp = nullptr;
    int32_t *ci = nullptr;
    double *va = nullptr;
};

// GMRES workspace, kept across nsm_gmres calls (in the preconditioner object):
// the Krylov basis grows on demand, host buffers are pinned, and the captured
// V-cycle + SpMV graph is reused until the operator, the stream or a smoother
// setting changes.
struct GmresWs {
    int device = 0;
    int64_t n = -1;
    int cap = 0;                       // basis columns allocated
    int m1cap = 0;                     // reduction buffers sized for this many columns
    int nblk = 1;
    double *V = nullptr, *u = nullptr, *w = nullptr, *z = nullptr, *part = nullptr, *red = nullptr, *hd = nullptr;
    double *hred = nullptr, *hh = nullptr;  // pinned host mirrors
    cudaGraphExec_t gexec = nullptr;
    std::vector<uint64_t> gsig;        // (uid, configuration generation) of the operator and every
                                       // smoother handle the graph was captured with
    cudaStream_t gs = nullptr;
    bool stale = true;
    cudaStream_t own = nullptr;        // private stream when the caller's cannot be captured (legacy default)
    cudaEvent_t ev = nullptr;
    void release() {
        cudaFree(V); cudaFree(u); cudaFree(w); cudaFree(z); cudaFree(part); cudaFree(red); cudaFree(hd);
        cudaFreeHost(hred); cudaFreeHost(hh);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (own) cudaStreamDestroy(own);
        if (ev) cudaEventDestroy(ev);
        *this = GmresWs();
    }
};

struct nsm_amg {
    int device = 0, nlevels = 0;
    GmresWs ws;
    std::vector<nsm_handle *> S;          // borrowed smoother handles, levels 0 .. nlevels-1
    std::vector<nsm_spmat *> P, R;        // owned transfer operators
    std::vector<int64_t> n;               // level sizes 0 .. nlevels
    struct Cfg { nsm_kind kind = NSM_PGS; int nu_pre = 1, nu_post = 1, k_l = 2, k_u = 2; };
    std::vector<Cfg> cfg;
    std::vector<double *> b, x, r;        // level work vectors (levels 1 .. nlevels; r on 0 .. nlevels-1)
    double *Minv = nullptr;               // dense inverse of the coarsest matrix
    double *rpart = nullptr;              // distributed finest level: this rank's share of R r (n_1)
    int nc = 0;
    std::string err;
};

namespace {
thread_local std::string g_solver_err;

nsm_status fail(std::string *dst, const std::string &msg, nsm_status st) {
    *dst = msg;
    return st;
}

// Gauss-Jordan inverse with partial pivoting (coarse-level direct solve,
// P:L550-552 "the coarse solver ... is often a direct solver").
bool dense_inverse(int n, std::vector<double> &a, std::vector<double> &inv) {
    inv.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) inv[(size_t)i * n + i] = 1.0;
    for (int c = 0; c < n; ++c) {
        int p = c;
        for (int r = c + 1; r < n; ++r)
            if (std::fabs(a[(size_t)r * n + c]) > std::fabs(a[(size_t)p * n + c])) p = r;
        if (a[(size_t)p * n + c] == 0.0) return false;
        if (p != c)
            for (int j = 0; j < n; ++j) {
                std::swap(a[(size_t)p * n + j], a[(size_t)c * n + j]);
                std::swap(inv[(size_t)p * n + j], inv[(size_t)c * n + j]);
            }
        const double d = a[(size_t)c * n + c];
        for (int j = 0; j < n; ++j) { a[(size_t)c * n + j] /= d; inv[(size_t)c * n + j] /= d; }
        for (int r = 0; r < n; ++r) {
            if (r == c) continue;
            const double f = a[(size_t)r * n + c];
            if (f == 0.0) continue;
            for (int j = 0; j < n; ++j) {
                a[(size_t)r * n + j] -= f * a[(size_t)c * n + j];
                inv[(size_t)r * n + j] -= f * inv[(size_t)c * n + j];
            }
        }
    }
    return true;
}

nsm_status spmat_from_host(const nsm_csr *M, int device, nsm_spmat **out, std::string *err) {
    if (!M || !M->rowptr || M->nrows < 0 || (M->rowptr[M->nrows] > 0 && (!M->colind || !M->val)))
        return fail(err, "nsm_spmat_setup: bad CSR", NSM_ERR_ARG);
    if (M->ncols >= ((int64_t)1 << 31)) return fail(err, "nsm_spmat_setup: too many columns for int32", NSM_ERR_ARG);
    const int64_t nnz = M->rowptr[M->nrows];
    std::vector<int32_t> c32(nnz);
    for (int64_t p = 0; p < nnz; ++p) {
        if (M->colind[p] < 0 || M->colind[p] >= M->ncols) return fail(err, "nsm_spmat_setup: column out of range", NSM_ERR_PATTERN);
        c32[p] = (int32_t)M->colind[p];
    }
    if (cudaSetDevice(device) != cudaSuccess) return fail(err, "cudaSetDevice failed", NSM_ERR_CUDA);
    nsm_spmat *S = new nsm_spmat();
    S->device = device;
    S->nrows = M->nrows;
    S->ncols = M->ncols;
    S->nnz = nnz;
    for (int64_t i = 0; i < M->nrows; ++i) S->maxrow = std::max(S->maxrow, M->rowptr[i + 1] - M->rowptr[i]);
    bool ok = cudaMalloc(&S->rp, (M->nrows + 1) * sizeof(int64_t)) == cudaSuccess &&
              cudaMalloc(&S->ci, std::max<int64_t>(nnz, 1) * sizeof(int32_t)) == cudaSuccess &&
              cudaMalloc(&S->va, std::max<int64_t>(nnz, 1) * sizeof(double)) == cudaSuccess &&
              cudaMemcpy(S->rp, M->rowptr, (M->nrows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice) == cudaSuccess &&
              (nnz == 0 || (cudaMemcpy(S->ci, c32.data(), nnz * sizeof(int32_t), cudaMemcpyHostToDevice) == cudaSuccess &&
                            cudaMemcpy(S->va, M->val, nnz * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess));
    if (!ok) {
        cudaFree(S->rp); cudaFree(S->ci); cudaFree(S->va);
        delete S;
        return fail(err, "nsm_spmat_setup: device allocation failed", NSM_ERR_OOM);
    }
    *out = S;
    return NSM_OK;
}

cudaError_t spmat_apply(const nsm_spmat *M, const double *x, double *y, double alpha, double beta, cudaStream_t s) {
    if (M->nrows == 0) return cudaSuccess;
    if (M->maxrow > 24 && M->nrows <= 4096)  // few, wide rows: warp per row
        launch_pdl(k_csr_spmv_wide, blocks(M->nrows * 32), s, M->nrows, (const int64_t *)M->rp, (const int32_t *)M->ci,
                   (const double *)M->va, x, y, alpha, beta);
    else
        launch_pdl(k_csr_spmv, blocks(M->nrows), s, M->nrows, (const int64_t *)M->rp, (const int32_t *)M->ci,
                   (const double *)M->va, x, y, alpha, beta);
    return cudaGetLastError();
}

// transpose of a host CSR (R = P^T), columns ascending per row
void transpose(const nsm_csr *P, std::vector<int64_t> &rp, std::vector<int64_t> &ci, std::vector<double> &va) {
    const int64_t nnz = P->rowptr[P->nrows];
    rp.assign(P->ncols + 1, 0);
    for (int64_t p = 0; p < nnz; ++p) rp[P->colind[p] + 1]++;
    for (int64_t j = 0; j < P->ncols; ++j) rp[j + 1] += rp[j];
    ci.resize(nnz);
    va.resize(nnz);
    std::vector<int64_t> pos(rp.begin(), rp.end() - 1);
    for (int64_t i = 0; i < P->nrows; ++i)
        for (int64_t p = P->rowptr[i]; p < P->rowptr[i + 1]; ++p) {
            const int64_t q = pos[P->colind[p]]++;
            ci[q] = i;
            va[q] = P->val[p];
        }
}

nsm_status amg_cycle(nsm_amg *M, int lev, const double *b, double *x, cudaStream_t s) {
    if (lev == M->nlevels) {
        launch_pdl(k_dense_gemv, (unsigned)((M->nc * 32 + kThr - 1) / kThr), s, M->nc, (const double *)M->Minv, b, x);
        cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? NSM_OK : fail(&M->err, cudaGetErrorString(e), NSM_ERR_CUDA);
    }
    const nsm_amg::Cfg &c = M->cfg[lev];
    nsm_handle *S = M->S[lev];
    // pre-smoothing from x = 0, residual, restriction, coarse correction,
    // prolongation, post-smoothing
    nsm_status st = nsm_smooth(S, c.kind, b, x, c.nu_pre, c.k_l, c.k_u, 1, s);
    if (st == NSM_OK) st = nsm_residual(S, b, x, M->r[lev], s);
    if (st != NSM_OK) return fail(&M->err, std::string("level ") + std::to_string(lev) + ": " + nsm_last_error(S), st);
    cudaError_t e;
    if (nsm_is_distributed(S)) {
        // the rank's rows of the fine level restrict to a share of the
        // (replicated) coarse right-hand side: b_{l+1} = sum over ranks of
        // P_p^T r_p, summed on the device over peer memory (nsm_comm)
        if (lev != 0) return fail(&M->err, "only the finest level may be distributed (coarse levels are replicated)", NSM_ERR_STATE);
        nsm_comm *c = nsm_handle_comm(S);
        if (!c) return fail(&M->err, "distributed finest level without a comm (nsm_set_comm)", NSM_ERR_STATE);
        if (comm_capacity(c) < M->n[1]) return fail(&M->err, "comm capacity below the first coarse level's size", NSM_ERR_ARG);
        if (!M->rpart) return fail(&M->err, "distributed level 0 set up after nsm_amg_setup", NSM_ERR_STATE);
        e = spmat_apply(M->R[lev], M->r[lev], M->rpart, 1.0, 0.0, s);
        if (e != cudaSuccess) return fail(&M->err, cudaGetErrorString(e), NSM_ERR_CUDA);
        st = comm_allreduce(c, M->rpart, M->b[lev + 1], M->n[1], s);
        if (st != NSM_OK) return fail(&M->err, "coarse restriction all-reduce failed", st);
    } else {
        e = spmat_apply(M->R[lev], M->r[lev], M->b[lev + 1], 1.0, 0.0, s);
        if (e != cudaSuccess) return fail(&M->err, cudaGetErrorString(e), NSM_ERR_CUDA);
    }
    st = amg_cycle(M, lev + 1, M->b[lev + 1], M->x[lev + 1], s);
    if (st != NSM_OK) return st;
    e = spmat_apply(M->P[lev], M->x[lev + 1], x, 1.0, 1.0, s);
    if (e != cudaSuccess) return fail(&M->err, cudaGetErrorString(e), NSM_ERR_CUDA);
    st = nsm_smooth(S, c.kind, b, x, c.nu_post, c.k_l, c.k_u, 0, s);
    if (st != NSM_OK) return fail(&M->err, std::string("level ") + std::to_string(lev) + ": " + nsm_last_error(S), st);
    return NSM_OK;
}

}  // namespace

extern "C" {

nsm_status nsm_spmat_setup(nsm_spmat **out, const nsm_csr *M, int device) {
    if (!out) return NSM_ERR_ARG;
    *out = nullptr;
    return spmat_from_host(M, device, out, &g_solver_err);
}

nsm_status nsm_spmat_apply(nsm_spmat *M, const double *x, double *y, double alpha, double beta, void *stream) {
    if (!M || (M->nrows > 0 && (!x || !y))) return NSM_ERR_ARG;
    return spmat_apply(M, x, y, alpha, beta, (cudaStream_t)stream) == cudaSuccess ? NSM_OK : NSM_ERR_CUDA;
}

void nsm_spmat_destroy(nsm_spmat *M) {
    if (!M) return;
    cudaSetDevice(M->device);
    cudaDeviceSynchronize();
    cudaFree(M->rp);
    cudaFree(M->ci);
    cudaFree(M->va);
    delete M;
}

void nsm_amg_destroy(nsm_amg *M) {
    if (!M) return;
    cudaSetDevice(M->device);
    cudaDeviceSynchronize();
    for (nsm_spmat *p : M->P) nsm_spmat_destroy(p);
    for (nsm_spmat *p : M->R) nsm_spmat_destroy(p);
    for (double *p : M->b) cudaFree(p);
    for (double *p : M->x) cudaFree(p);
    for (double *p : M->r) cudaFree(p);
    cudaFree(M->Minv);
    cudaFree(M->rpart);
    M->ws.release();
    delete M;
}

nsm_status nsm_amg_setup(nsm_amg **out, int nlevels, nsm_handle *const *smoothers, const nsm_csr *const *P,
                         const nsm_csr *coarse, int device) {
    if (!out || nlevels < 0 || !coarse || (nlevels > 0 && (!smoothers || !P)))
        return fail(&g_solver_err, "nsm_amg_setup: bad argument", NSM_ERR_ARG);
    *out = nullptr;
    if (coarse->nrows != coarse->ncols || coarse->nrows > 8192 || coarse->nrows < 1)
        return fail(&g_solver_err, "nsm_amg_setup: the coarse matrix must be square with 1..8192 rows", NSM_ERR_ARG);
    nsm_amg *M = new nsm_amg();
    M->device = device;
    DeviceScope devscope(device);
    preload_solver_kernels();
    M->nlevels = nlevels;
    M->cfg.resize(nlevels);
    nsm_status st = NSM_OK;
    for (int l = 0; l < nlevels && st == NSM_OK; ++l) {
        int64_t nl = 0;
        nsm_info(smoothers[l], &nl, nullptr, nullptr, nullptr);
        if (!P[l] || P[l]->nrows != nl) {
            st = fail(&g_solver_err, "nsm_amg_setup: P[" + std::to_string(l) + "] shape mismatch", NSM_ERR_ARG);
            break;
        }
        M->S.push_back(smoothers[l]);
        M->n.push_back(nl);
        nsm_spmat *p = nullptr, *r = nullptr;
        st = spmat_from_host(P[l], device, &p, &g_solver_err);
        if (st != NSM_OK) break;
        M->P.push_back(p);
        std::vector<int64_t> rrp, rci;
        std::vector<double> rva;
        transpose(P[l], rrp, rci, rva);
        nsm_csr Rt{P[l]->ncols, P[l]->nrows, rrp.data(), rci.data(), rva.data()};
        st = spmat_from_host(&Rt, device, &r, &g_solver_err);
        if (st != NSM_OK) break;
        M->R.push_back(r);
    }
    if (st == NSM_OK) {
        M->n.push_back(coarse->nrows);
        for (int l = 0; l < nlevels; ++l)
            if (M->P[l]->ncols != M->n[l + 1])
                st = fail(&g_solver_err, "nsm_amg_setup: P[" + std::to_string(l) + "] columns != next level size",
                          NSM_ERR_ARG);
    }
    if (st == NSM_OK) {
        M->nc = (int)coarse->nrows;
        std::vector<double> a((size_t)M->nc * M->nc, 0.0), inv;
        for (int i = 0; i < M->nc; ++i)
            for (int64_t p = coarse->rowptr[i]; p < coarse->rowptr[i + 1]; ++p)
                a[(size_t)i * M->nc + coarse->colind[p]] += coarse->val[p];
        if (!dense_inverse(M->nc, a, inv)) st = fail(&g_solver_err, "nsm_amg_setup: singular coarse matrix", NSM_ERR_ZERO_DIAG);
        else if (cudaMalloc(&M->Minv, inv.size() * sizeof(double)) != cudaSuccess ||
                 cudaMemcpy(M->Minv, inv.data(), inv.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
            st = fail(&g_solver_err, "nsm_amg_setup: device allocation failed", NSM_ERR_OOM);
    }
    // level vectors: r_l for l < nlevels; b_l, x_l for 1 <= l <= nlevels
    M->b.assign(nlevels + 1, nullptr);
    M->x.assign(nlevels + 1, nullptr);
    M->r.assign(nlevels, nullptr);
    // distributed finest level: this rank's share of the restriction (allocated
    // here, not in the cycle: no allocation inside a distributed solve)
    if (st == NSM_OK && nlevels > 0 && nsm_is_distributed(M->S[0]) &&
        cudaMalloc(&M->rpart, std::max<int64_t>(M->n[1], 1) * sizeof(double)) != cudaSuccess) {
        st = NSM_ERR_OOM;
        g_solver_err = "nsm_amg_setup: device allocation failed";
    }
    for (int l = 0; l <= nlevels && st == NSM_OK; ++l) {
        const size_t bytes = std::max<int64_t>(M->n[l], 1) * sizeof(double);
        if (l < nlevels && cudaMalloc(&M->r[l], bytes) != cudaSuccess) st = NSM_ERR_OOM;
        if (l >= 1 && (cudaMalloc(&M->b[l], bytes) != cudaSuccess || cudaMalloc(&M->x[l], bytes) != cudaSuccess))
            st = NSM_ERR_OOM;
        if (st != NSM_OK) g_solver_err = "nsm_amg_setup: device allocation failed";
    }
    if (st != NSM_OK) {
        nsm_amg_destroy(M);
        return st;
    }
    *out = M;
    return NSM_OK;
}

nsm_status nsm_amg_set_smoother(nsm_amg *M, int level, nsm_kind kind, int nu_pre, int nu_post, int k_l, int k_u) {
    if (!M || level < 0 || level >= M->nlevels || nu_pre < 0 || nu_post < 0 || k_l < 0 || k_u < 0) return NSM_ERR_ARG;
    M->cfg[level] = nsm_amg::Cfg{kind, nu_pre, nu_post, k_l, k_u};
    M->ws.stale = true;  // the captured V-cycle graph no longer matches
    return NSM_OK;
}

nsm_status nsm_amg_vcycle(nsm_amg *M, const double *b, double *x, void *stream) {
    if (!M || !b || !x || b == x) return NSM_ERR_ARG;
    DeviceScope dev(M->device);
    return amg_cycle(M, 0, b, x, (cudaStream_t)stream);
}

const char *nsm_solver_last_error(const nsm_amg *M) { return M ? M->err.c_str() : g_solver_err.c_str(); }

// ---- Algorithm 1: one-reduce MGS-GMRES with T = I - L (or (I + L)^{-1}) ----
nsm_status nsm_gmres(nsm_handle *A, nsm_amg *M, const double *b, double *x, int maxit, double tol, int t_mode,
                     int *iters, double *hist, void *stream) {
    if (!A || !b || !x || maxit < 1 || tol <= 0 || (t_mode != 0 && t_mode != 1)) {
        g_solver_err = "nsm_gmres: bad argument";
        return NSM_ERR_ARG;
    }
    DeviceScope devscope(nsm_handle_device(A));
    cudaStream_t s = (cudaStream_t)stream;
    int64_t n = 0;
    nsm_info(A, &n, nullptr, nullptr, nullptr);
    const int m1 = maxit + 1;
    // a distributed operator reduces its dot products across ranks (step 6's
    // "Global synchronization") through its comm; without one each rank
    // would build its own Krylov coefficients
    nsm_comm *comm = nsm_is_distributed(A) ? nsm_handle_comm(A) : nullptr;
    if (nsm_is_distributed(A) && !comm) {
        g_solver_err = "nsm_gmres: a distributed operator needs a comm for the global reduction (nsm_set_comm)";
        return NSM_ERR_STATE;
    }
    if (comm && comm_capacity(comm) < 2 * (int64_t)(maxit + 2)) {
        g_solver_err = "nsm_gmres: comm capacity below 2 (maxit + 2)";
        return NSM_ERR_ARG;
    }
    if (M && nsm_is_distributed(A) != (M->nlevels > 0 && nsm_is_distributed(M->S[0]))) {
        g_solver_err = "nsm_gmres: operator and finest smoother differ in distribution";
        return NSM_ERR_ARG;
    }
    GmresWs local;
    GmresWs &W = M ? M->ws : local;   // persistent with a preconditioner object
    // Basis capacity >= cols (keeps columns 0 .. cap-1).  Stream-ordered
    // allocation: no device-wide synchronisation in the middle of a solve
    // (cudaFree would wait for every stream of the device — with ranks sharing
    // a device, for a peer's halo / reduction wait on a put this rank has not
    // launched yet).
    auto grow = [&](int cols) -> bool {
        if (cols <= W.cap) return true;
        const int nc = std::min(m1, std::max(cols, std::max(32, 2 * W.cap)));
        double *nv = nullptr;
        if (cudaMallocAsync((void **)&nv, (size_t)nc * std::max<int64_t>(n, 1) * sizeof(double), s) != cudaSuccess)
            return false;
        if (W.V && W.cap > 0 &&
            cudaMemcpyAsync(nv, W.V, (size_t)W.cap * n * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return false;
        if (W.V) cudaFreeAsync(W.V, s);
        W.V = nv;
        W.cap = nc;
        return true;
    };
    bool ok = true;
    int dev = 0;
    cudaGetDevice(&dev);
    if (W.n != n || W.device != dev) {   // new operator size or device: start over
        W.release();
        W.n = n;
        W.device = dev;
        W.nblk = (int)std::min<int64_t>(1184, std::max<int64_t>(1, n / 2048));
        ok = cudaMalloc(&W.u, std::max<int64_t>(n, 1) * sizeof(double)) == cudaSuccess &&
             cudaMalloc(&W.w, std::max<int64_t>(n, 1) * sizeof(double)) == cudaSuccess &&
             cudaMalloc(&W.z, std::max<int64_t>(n, 1) * sizeof(double)) == cudaSuccess;
    }
    if (ok && W.m1cap < m1) {
        cudaFree(W.part); cudaFree(W.red); cudaFree(W.hd); cudaFreeHost(W.hred); cudaFreeHost(W.hh);
        W.part = W.red = W.hd = W.hred = W.hh = nullptr;
        ok = cudaMalloc(&W.part, (size_t)W.nblk * 2 * (m1 + 1) * sizeof(double)) == cudaSuccess &&
             cudaMalloc(&W.red, 2 * (size_t)(m1 + 1) * sizeof(double)) == cudaSuccess &&
             cudaMalloc(&W.hd, (size_t)(m1 + 1) * sizeof(double)) == cudaSuccess &&
             cudaMallocHost(&W.hred, 2 * (size_t)(m1 + 1) * sizeof(double)) == cudaSuccess &&
             cudaMallocHost(&W.hh, (size_t)(m1 + 1) * sizeof(double)) == cudaSuccess;
        W.m1cap = ok ? m1 : 0;
    }
    ok = ok && grow(std::min(m1, 32));
    if (!ok) {
        cudaGetLastError();
        if (!M) local.release();
        g_solver_err = "nsm_gmres: device allocation failed";
        return NSM_ERR_OOM;
    }
    double *V = W.V, *u = W.u, *w = W.w, *z = W.z, *part = W.part, *red = W.red, *hd = W.hd;
    const int nblk = W.nblk;
    // The legacy default stream cannot be captured into a graph: run the solve
    // on a private non-blocking stream ordered after the caller's prior work
    // (the solve ends with a host synchronisation, so later work on the
    // caller's stream sees its result).
    {
        cudaStreamCaptureStatus cst;
        const bool capturable = s != nullptr && s != cudaStreamLegacy &&
                                cudaStreamIsCapturing(s, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusNone;
        if (!capturable && !nsm_is_distributed(A)) {
            if (!W.own && (cudaStreamCreateWithFlags(&W.own, cudaStreamNonBlocking) != cudaSuccess ||
                           cudaEventCreateWithFlags(&W.ev, cudaEventDisableTiming) != cudaSuccess)) {
                cudaGetLastError();
                W.own = nullptr;
            }
            if (W.own && cudaEventRecord(W.ev, s) == cudaSuccess && cudaStreamWaitEvent(W.own, W.ev, 0) == cudaSuccess)
                s = W.own;
        }
    }
    auto cleanup = [&]() { if (!M) local.release(); };
    // signature of everything baked into the captured launch sequence: the
    // operator and smoother handles (by unique id, not address) and their
    // option / Ruiz generations (a changed option changes the launches)
    std::vector<uint64_t> sig{nsm_handle_uid(A), nsm_handle_cfg_gen(A)};
    if (M)
        for (nsm_handle *S : M->S) { sig.push_back(nsm_handle_uid(S)); sig.push_back(nsm_handle_cfg_gen(S)); }
    if (W.gexec && (W.stale || W.gsig != sig || W.gs != s)) {
        cudaGraphExecDestroy(W.gexec);
        W.gexec = nullptr;
    }
    cudaGraphExec_t &gexec = W.gexec;
    bool use_graph = !nsm_is_distributed(A);
    if (M)
        for (nsm_handle *S : M->S) use_graph = use_graph && !nsm_is_distributed(S);
    auto precond = [&](const double *in, double *out) -> nsm_status {
        if (M) return nsm_amg_vcycle(M, in, out, s);
        return cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, s) == cudaSuccess ? NSM_OK
                                                                                                       : NSM_ERR_CUDA;
    };
    std::vector<double> Lm((size_t)m1 * m1, 0.0), H((size_t)m1 * maxit, 0.0), cs(maxit), sn(maxit), g(m1 + 1, 0.0);
    std::vector<double> zc, h;
    double *hred = W.hred;
    auto Hat = [&](int i, int j) -> double & { return H[(size_t)i * maxit + j]; };
    nsm_status st = NSM_OK;
    double beta = 0.0;
    int m = 0;
    std::vector<double> hv{1.0};
    // u = b (x0 = 0)
    cudaMemcpyAsync(u, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
    for (int k = 0; k <= maxit && st == NSM_OK; ++k) {
        if (k < maxit) {
            // step 5: w = A M u.  The V-cycle + SpMV is a fixed sequence of
            // ~10 launches per level on fixed buffers (u -> z -> w), so it is
            // captured once into a CUDA graph and replayed (single-rank
            // handles only: a halo exchange bakes its sequence number in).
            if (use_graph && !gexec) {
                cudaGraph_t graph = nullptr;
                bool ok = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
                if (ok) {
                    st = precond(u, z);
                    if (st == NSM_OK) st = nsm_spmv(A, z, w, s);
                    ok = cudaStreamEndCapture(s, &graph) == cudaSuccess && st == NSM_OK &&
                         cudaGraphInstantiate(&gexec, graph, 0) == cudaSuccess;
                    W.gsig = sig;
                    W.gs = s;
                    W.stale = false;
                    if (graph) cudaGraphDestroy(graph);
                }
                if (!ok) {  // fall back to plain launches
                    cudaGetLastError();
                    if (gexec) cudaGraphExecDestroy(gexec);
                    gexec = nullptr;
                    use_graph = false;
                    st = NSM_OK;
                }
            }
            if (gexec) {
                if (cudaGraphLaunch(gexec, s) != cudaSuccess) { st = NSM_ERR_CUDA; break; }
            } else {
                st = precond(u, z);                               // z = M u
                if (st == NSM_OK) st = nsm_spmv(A, z, w, s);      // w = A M u
                if (st != NSM_OK) break;
            }
        }
        // step 6: the single reduction [V_k, u]^T [u, w]
        k_multidot<<<nblk, kThr, 0, s>>>(n, k, V, u, k < maxit ? w : u, part);
        k_sum_parts<<<(2 * (k + 1) + 127) / 128, 128, 0, s>>>(nblk, 2 * (k + 1), part, red);
        if (comm && (st = comm_allreduce(comm, red, red, 2 * (k + 1), s)) != NSM_OK) break;
        cudaMemcpyAsync(hred, red, 2 * (k + 1) * sizeof(double), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) { st = NSM_ERR_CUDA; break; }
        if (comm && comm_failed(comm)) {
            g_solver_err = "nsm_gmres: the global reduction timed out waiting for a rank";
            st = NSM_ERR_DIST;
            break;
        }
        const double nu = hred[2 * k], mu = hred[2 * k + 1];
        const double rho = std::sqrt(nu);                     // step 7 (lagged norm)
        if (k == 0) { beta = rho; g[0] = beta; }
        if (k > 0) {                                          // complete column k-1, Givens
            const int j = k - 1;
            Hat(j + 1, j) = rho;
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * Hat(i, j) + sn[i] * Hat(i + 1, j);
                Hat(i + 1, j) = -sn[i] * Hat(i, j) + cs[i] * Hat(i + 1, j);
                Hat(i, j) = t;
            }
            const double den = std::hypot(Hat(j, j), Hat(j + 1, j));
            cs[j] = Hat(j, j) / den;
            sn[j] = Hat(j + 1, j) / den;
            Hat(j, j) = den;
            Hat(j + 1, j) = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            hv.push_back(std::fabs(g[j + 1]) / beta);
            if (hv.back() < tol || k == maxit) { m = k; break; }
        }
        if (rho == 0.0) { m = k; break; }                     // exact solution (happy breakdown)
        // step 8: v_k = u / rho
        if (!grow(k + 1)) { st = NSM_ERR_OOM; break; }
        V = W.V;
        k_scal<<<blocks(n), kThr, 0, s>>>(n, 1.0 / rho, u, V + (size_t)k * n);
        // steps 9-11: z = [c, mu/rho] / rho, L row k = a / rho, h = T z
        zc.assign(k + 1, 0.0);
        for (int i = 0; i < k; ++i) {
            zc[i] = hred[2 * i + 1] / rho;
            Lm[(size_t)k * m1 + i] = hred[2 * i] / rho;
        }
        zc[k] = mu / rho / rho;
        h.assign(k + 1, 0.0);
        for (int i = 0; i <= k; ++i) {
            double acc = zc[i];
            if (t_mode == 0) {                                // T = I - L  (truncated Neumann)
                for (int j = 0; j < i; ++j) acc -= Lm[(size_t)i * m1 + j] * zc[j];
            } else {                                          // T = (I + L)^{-1}: forward substitution
                for (int j = 0; j < i; ++j) acc -= Lm[(size_t)i * m1 + j] * h[j];
            }
            h[i] = acc;
            Hat(i, k) = acc;
        }
        // step 12: u = w / rho - V_{k+1} h
        std::copy(h.begin(), h.end(), W.hh);
        cudaMemcpyAsync(hd, W.hh, (k + 1) * sizeof(double), cudaMemcpyHostToDevice, s);
        k_multiaxpy<<<blocks(n), kThr, 0, s>>>(n, k + 1, V, hd, 1.0 / rho, w, u);
        if (cudaGetLastError() != cudaSuccess) { st = NSM_ERR_CUDA; break; }
    }
    if (st == NSM_OK && m > 0) {
        // y = H^{-1} g (upper triangular m x m), x = M (V_m y)
        std::vector<double> y(m);
        for (int i = m - 1; i >= 0; --i) {
            double acc = g[i];
            for (int j = i + 1; j < m; ++j) acc -= Hat(i, j) * y[j];
            y[i] = acc / Hat(i, i);
        }
        for (double &v : y) v = -v;                            // multiaxpy subtracts
        std::copy(y.begin(), y.end(), W.hh);
        cudaMemcpyAsync(hd, W.hh, m * sizeof(double), cudaMemcpyHostToDevice, s);
        k_multiaxpy<<<blocks(n), kThr, 0, s>>>(n, m, V, hd, 0.0, nullptr, u);
        st = precond(u, x);
        if (cudaStreamSynchronize(s) != cudaSuccess) st = NSM_ERR_CUDA;
    } else if (st == NSM_OK) {
        cudaMemsetAsync(x, 0, n * sizeof(double), s);
        cudaStreamSynchronize(s);
    }
    if (iters) *iters = m;
    if (hist) std::copy(hv.begin(), hv.end(), hist);
    cleanup();
    if (st != NSM_OK && g_solver_err.empty()) g_solver_err = "nsm_gmres: failed";
    return st;
}

}  // extern "C"
