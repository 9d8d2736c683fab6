// chow_patel.cu — ILU(0) factors on the GPU by Chow-Patel fixed-point sweeps
// (the set-up algorithm the paper names as future
// work; reading R19).
//
// The ILU(0) factors solve (L U)_ij = a_ij on the pattern S of A (L unit
// lower).  As a fixed point:
//     l_ij = ( a_ij - sum_{k<j} l_ik u_kj ) / u_jj      (i > j)
//     u_ij =   a_ij - sum_{k<i} l_ik u_kj               (i <= j)
// iterated synchronously (each sweep reads only the previous sweep) from
// l_ij = a_ij / a_jj, u_ij = a_ij.  Everything runs on the device (the host
// only uploads the CSR): validation, diagonal positions, and the sweeps, one
// thread per row, each (k, j) partner found by binary search in row k.  Every
// entry is formed with the same IEEE
// operations in the same order as the IKJ elimination (one subtraction per
// k, then the division), so once converged the result equals the host
// nsm_ilu0 bit for bit.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "nsm_internal.h"

namespace nsm {

namespace {

// One thread per row.  Validates the row (strictly ascending columns, a
// nonzero diagonal) and records the diagonal's position.
__global__ void k_cp_prep(int64_t n, int64_t rb, const int64_t *__restrict__ rp, const int64_t *__restrict__ ci,
                          const double *__restrict__ a, int64_t *__restrict__ dpos, unsigned long long *bad_pattern,
                          unsigned long long *bad_diag) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t d = -1;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        if (p > rp[i] && ci[p] <= ci[p - 1]) atomicMin(bad_pattern, (unsigned long long)i);
        if (ci[p] == rb + i) d = p;
    }
    dpos[i] = d;
    if (d < 0 || a[d] == 0.0) atomicMin(bad_diag, (unsigned long long)i);
}

// Initial guess l_ij = a_ij / a_jj, u_ij = a_ij; off-block entries 0.
__global__ void k_cp_init(int64_t n, int64_t rb, const int64_t *__restrict__ rp, const int64_t *__restrict__ ci,
                          const double *__restrict__ a, const int64_t *__restrict__ dpos, double *__restrict__ w0,
                          double *__restrict__ w1) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int64_t j = ci[p] - rb;
        double v = 0.0;
        if (j >= 0 && j < n) v = j < i ? __ddiv_rn(a[p], a[dpos[j]]) : a[p];
        w0[p] = v;
        w1[p] = v;
    }
}

// One synchronous sweep, one thread per row: for each in-block entry (i, j),
// s = a_ij - sum over k < min(i, j) (ascending, (i,k) and (k,j) in the
// pattern) of l_ik u_kj, divided by u_jj for L entries.  (k, j) is found by
// binary search in row k.
__global__ void k_cp_sweep(int64_t n, int64_t rb, const int64_t *__restrict__ rp, const int64_t *__restrict__ ci,
                           const double *__restrict__ a, const int64_t *__restrict__ dpos,
                           const double *__restrict__ old, double *__restrict__ w, unsigned int *bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p0 = rp[i], p1 = rp[i + 1];
    for (int64_t p = p0; p < p1; ++p) {
        const int64_t gj = ci[p], j = gj - rb;
        if (j < 0 || j >= n) continue;
        const int64_t mlim = j < i ? j : i;
        double s = a[p];
        for (int64_t q = p0; q < p1; ++q) {
            const int64_t k = ci[q] - rb;
            if (k < 0) continue;
            if (k >= mlim) break;
            int64_t lo = rp[k], hi = rp[k + 1];   // (k, j) in row k?
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (ci[mid] < gj) lo = mid + 1;
                else hi = mid;
            }
            if (lo < rp[k + 1] && ci[lo] == gj) s = __dsub_rn(s, __dmul_rn(old[q], old[lo]));
        }
        if (j < i) {
            const double d = old[dpos[j]];
            if (d == 0.0) atomicOr(bad, 1u);
            s = __ddiv_rn(s, d);
        }
        w[p] = s;
    }
}

}  // namespace

nsm_status ilu0_fixed_point_device(const nsm_csr *A, int64_t rb, int sweeps, double *fval, int device,
                                   std::string *err) {
    const int64_t n = A->nrows;
    const int64_t *rp = A->rowptr, *ci = A->colind;
    const double *va = A->val;
    if (!rp || !fval || n < 0 || sweeps < 0 || (rp[n] > 0 && (!ci || !va))) {
        *err = "nsm_ilu0_fixed_point: bad argument";
        return NSM_ERR_ARG;
    }
    const int64_t nnz = rp[n];
    if (cudaSetDevice(device) != cudaSuccess) {
        *err = "nsm_ilu0_fixed_point: cudaSetDevice failed";
        return NSM_ERR_CUDA;
    }
    int64_t *d_rp = nullptr, *d_ci = nullptr, *d_dpos = nullptr;
    double *d_a = nullptr, *d_w[2] = {nullptr, nullptr};
    unsigned long long *d_badrow = nullptr;  // [pattern, diagonal]
    unsigned int *d_bad = nullptr;
    auto cleanup = [&]() {
        cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_dpos); cudaFree(d_a);
        cudaFree(d_w[0]); cudaFree(d_w[1]); cudaFree(d_badrow); cudaFree(d_bad);
    };
    cudaError_t ce = cudaSuccess;
    auto ok = [&](cudaError_t e) { if (ce == cudaSuccess) ce = e; return ce == cudaSuccess; };
    const size_t nb = (size_t)std::max<int64_t>(nnz, 1) * 8;
    ok(cudaMalloc(&d_rp, (size_t)(n + 1) * 8));
    ok(cudaMalloc(&d_ci, nb));
    ok(cudaMalloc(&d_dpos, (size_t)std::max<int64_t>(n, 1) * 8));
    ok(cudaMalloc(&d_a, nb));
    ok(cudaMalloc(&d_w[0], nb));
    ok(cudaMalloc(&d_w[1], nb));
    ok(cudaMalloc(&d_badrow, 2 * sizeof(unsigned long long)));
    ok(cudaMalloc(&d_bad, sizeof(unsigned int)));
    if (ce != cudaSuccess) {
        cleanup();
        cudaGetLastError();
        *err = "nsm_ilu0_fixed_point: device allocation failed";
        return NSM_ERR_OOM;
    }
    ok(cudaMemcpy(d_rp, rp, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice));
    if (nnz > 0) {
        ok(cudaMemcpy(d_ci, ci, (size_t)nnz * 8, cudaMemcpyHostToDevice));
        ok(cudaMemcpy(d_a, va, (size_t)nnz * 8, cudaMemcpyHostToDevice));
    }
    ok(cudaMemset(d_badrow, 0xff, 2 * sizeof(unsigned long long)));
    ok(cudaMemset(d_bad, 0, sizeof(unsigned int)));
    const unsigned grid = (unsigned)std::max<int64_t>((n + 127) / 128, 1);
    int cur = 0;
    unsigned long long badrow[2] = {~0ull, ~0ull};
    if (n > 0) {
        k_cp_prep<<<grid, 128>>>(n, rb, d_rp, d_ci, d_a, d_dpos, d_badrow, d_badrow + 1);
        ok(cudaGetLastError());
        ok(cudaMemcpy(badrow, d_badrow, sizeof(badrow), cudaMemcpyDeviceToHost));
        if (ce == cudaSuccess && badrow[0] == ~0ull && badrow[1] == ~0ull) {
            k_cp_init<<<grid, 128>>>(n, rb, d_rp, d_ci, d_a, d_dpos, d_w[0], d_w[1]);
            ok(cudaGetLastError());
            for (int s = 0; s < sweeps && ce == cudaSuccess; ++s) {
                k_cp_sweep<<<grid, 128>>>(n, rb, d_rp, d_ci, d_a, d_dpos, d_w[cur], d_w[cur ^ 1], d_bad);
                ok(cudaGetLastError());
                cur ^= 1;
            }
        }
    }
    unsigned int bad = 0;
    if (ce == cudaSuccess && badrow[0] == ~0ull && badrow[1] == ~0ull) {
        ok(cudaMemcpy(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost));
        if (nnz > 0) ok(cudaMemcpy(fval, d_w[cur], (size_t)nnz * 8, cudaMemcpyDeviceToHost));
    }
    cleanup();
    if (ce != cudaSuccess) {
        *err = std::string("nsm_ilu0_fixed_point: ") + cudaGetErrorString(ce);
        return NSM_ERR_CUDA;
    }
    if (badrow[0] != ~0ull) {
        *err = "nsm_ilu0_fixed_point: columns not strictly ascending in global row " + std::to_string(rb + (int64_t)badrow[0]);
        return NSM_ERR_PATTERN;
    }
    if (badrow[1] != ~0ull) {
        *err = "nsm_ilu0_fixed_point: missing or zero diagonal at global row " + std::to_string(rb + (int64_t)badrow[1]);
        return NSM_ERR_ZERO_DIAG;
    }
    if (bad) {
        *err = "nsm_ilu0_fixed_point: zero pivot u_jj during the sweeps";
        return NSM_ERR_ZERO_DIAG;
    }
    return NSM_OK;
}

}  // namespace nsm
