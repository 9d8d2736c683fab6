// builder_gpu.cu — the split-triangular SELL-32 builder on the device
// (SURVEY.md §8(f) NEXT-4 "a GPU split/SELL builder"; the paper's set-up cost
// outlook).  Single rank: A (and the ILU factor F) arrive as a
// DEVICE CSR; the split A = L + D + U, the diagonal, the
// l1-Jacobi diagonal, the compact or offset-aligned SELL-32 packing of L and
// U and the bandwidths are computed by the kernels below and produce exactly
// the arrays builder.cpp's build_split produces on the host (same
// classification, same padding convention, same layout decision) — the
// parity tests compare them entry by entry.
//
// Steps (one thread per row, one warp per slice):
//   1. k_rows: validate each row (ascending in-range columns, a nonzero
//      finite diagonal), count its strictly-lower entries, store d and the
//      l1 diagonal (ascending |a_ij| sum), bandwidths by atomicMax;
//   2. k_slices: per slice and part the width (longest row) and the sorted
//      union of the rows' column offsets (warp-wide repeated minimum over the
//      32 rows' ascending lists), capped at 2 w + 8 entries;
//   3. the layout decision of builder.cpp (few pads, little widening) from
//      three sums; slice pointers by an exclusive scan of the slice sizes;
//   4. k_fill: entries and pads written column-major per slice (and the
//      slice offsets for the offset-aligned layout).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "nsm_internal.h"

namespace nsm {

namespace {

constexpr int kThr = 256;

inline unsigned blocks_of(int64_t n, int per = kThr) { return (unsigned)std::max<int64_t>(1, (n + per - 1) / per); }

struct RowStats {
    unsigned long long bad;     // min over bad rows of (row << 2 | kind): 1 pattern, 2 diagonal
    unsigned long long bw[2];   // lower / upper bandwidth
    unsigned long long nnz_off; // off-diagonal entries
    unsigned long long maxcnt[2];
};

__global__ void __launch_bounds__(kThr) k_rows(int64_t n, int64_t ncols, const int64_t *__restrict__ rp,
                                               const int64_t *__restrict__ ci, const double *__restrict__ va,
                                               int32_t *__restrict__ cntL, double *__restrict__ d,
                                               double *__restrict__ dl1, RowStats *st) {
    const int64_t i = (int64_t)blockIdx.x * kThr + threadIdx.x;
    if (i >= n) return;
    const int64_t b = rp[i], e = rp[i + 1];
    int kind = 0;
    bool has_d = false;
    double di = 0.0, l1 = 0.0;
    int32_t nl = 0;
    if (e < b) kind = 1;
    for (int64_t p = b; kind == 0 && p < e; ++p) {
        const int64_t c = ci[p];
        if (c < 0 || c >= ncols || (p > b && ci[p - 1] >= c)) { kind = 1; break; }
        const double v = va[p];
        if (c == i) {
            has_d = v != 0.0 && isfinite(v);
            di = v;
        } else {
            l1 = l1 + fabs(v);        // ascending columns, as builder.cpp
            if (c < i) ++nl;
        }
    }
    if (kind == 0 && !has_d) kind = 2;
    if (kind) {
        atomicMin(&st->bad, ((unsigned long long)i << 2) | (unsigned long long)kind);
        return;
    }
    cntL[i] = nl;
    d[i] = di;
    dl1[i] = di + l1;
    const int32_t nu = (int32_t)(e - b) - nl - 1;
    if (nl > 0) atomicMax(&st->bw[0], (unsigned long long)(i - ci[b]));
    if (nu > 0) atomicMax(&st->bw[1], (unsigned long long)(ci[e - 1] - i));
    atomicAdd(&st->nnz_off, (unsigned long long)(e - b - 1));
    atomicMax(&st->maxcnt[0], (unsigned long long)nl);
    atomicMax(&st->maxcnt[1], (unsigned long long)nu);
}

// entries of row i in part P (0: strictly lower, 1: strictly upper)
__device__ __forceinline__ void part_range(int P, int64_t i, const int64_t *rp, const int32_t *cntL, int64_t *first,
                                           int32_t *cnt) {
    const int64_t b = rp[i], e = rp[i + 1];
    const int32_t nl = cntL[i];
    if (P == 0) { *first = b; *cnt = nl; }
    else { *first = b + nl + 1; *cnt = (int32_t)(e - b) - nl - 1; }
}

struct SliceStats {
    unsigned long long sum_u, sum_c, nnz, overflow, maxu, maxc;
};

// one warp per slice: width and (capped) sorted union of column offsets
__global__ void __launch_bounds__(kThr) k_slices(int P, int64_t n, int64_t ns, const int64_t *__restrict__ rp,
                                                 const int64_t *__restrict__ ci, const int32_t *__restrict__ cntL,
                                                 int32_t ucap, int32_t *__restrict__ wid, int32_t *__restrict__ ucnt,
                                                 int32_t *__restrict__ uni, SliceStats *st) {
    const int64_t s = ((int64_t)blockIdx.x * kThr + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= ns) return;
    const int64_t i = s * kSlice + lane;
    int64_t first = 0;
    int32_t cnt = 0;
    if (i < n) part_range(P, i, rp, cntL, &first, &cnt);
    int32_t w = cnt;
    for (int o = 16; o; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
    unsigned long long nz = (unsigned long long)cnt;
    for (int o = 16; o; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
    // union: repeatedly take the smallest head offset over the 32 rows
    int32_t q = 0, u = 0;
    const int32_t cap = min(ucap, 2 * w + 8);
    bool over = false;
    while (true) {
        const int64_t head = q < cnt ? ci[first + q] - i : INT64_MAX;
        long long m = (long long)head;
        for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (m == INT64_MAX) break;
        if (u >= cap) { over = true; break; }
        if (lane == 0) uni[s * ucap + u] = (int32_t)m;
        ++u;
        if (head == m) ++q;
    }
    if (lane == 0) {
        wid[s] = w;
        ucnt[s] = u;
        atomicAdd(&st->sum_u, (unsigned long long)u);
        atomicAdd(&st->sum_c, (unsigned long long)w);
        atomicAdd(&st->nnz, nz);
        atomicMax(&st->maxu, (unsigned long long)u);
        atomicMax(&st->maxc, (unsigned long long)w);
        if (over) atomicOr(&st->overflow, 1ull);
    }
}

__global__ void k_slice_sizes(int64_t ns, int aligned, const int32_t *__restrict__ wid,
                              const int32_t *__restrict__ ucnt, int64_t *__restrict__ sz) {
    const int64_t s = (int64_t)blockIdx.x * kThr + threadIdx.x;
    if (s < ns) sz[s] = (int64_t)(aligned ? ucnt[s] : wid[s]) * kSlice;
    if (s == ns) sz[s] = 0;
}

// one warp per slice: column-major entries, pads (val 0) as builder.cpp
__global__ void __launch_bounds__(kThr) k_fill(int P, int aligned, int64_t n, int64_t ns,
                                               const int64_t *__restrict__ rp, const int64_t *__restrict__ ci,
                                               const double *__restrict__ va, const int32_t *__restrict__ cntL,
                                               const int32_t *__restrict__ wid, const int32_t *__restrict__ ucnt,
                                               const int32_t *__restrict__ uni, int32_t ucap,
                                               const int64_t *__restrict__ ptr, int32_t *__restrict__ col,
                                               double *__restrict__ val, int32_t *__restrict__ off) {
    const int64_t s = ((int64_t)blockIdx.x * kThr + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= ns) return;
    const int64_t i = s * kSlice + lane;
    int64_t first = 0;
    int32_t cnt = 0;
    if (i < n) part_range(P, i, rp, cntL, &first, &cnt);
    const int64_t base = ptr[s];
    if (aligned) {
        const int32_t u = ucnt[s];
        int32_t q = 0;
        for (int32_t j = 0; j < u; ++j) {
            const int32_t o = uni[s * ucap + j];
            const int64_t e = base + (int64_t)j * kSlice + lane;
            const int64_t c = i + o;
            if (i < n && q < cnt && ci[first + q] == c) {
                col[e] = (int32_t)c;
                val[e] = va[first + q];
                ++q;
            } else {  // pad: val 0 at row + offset (or the row itself when out of range)
                col[e] = (int32_t)((i < n && c >= 0 && c < n) ? c : (i < n ? i : 0));
                val[e] = 0.0;
            }
            if (lane == 0) off[base / kSlice + j] = o;
        }
    } else {
        const int32_t w = wid[s];
        const int32_t pad = (int32_t)(i < n ? i : 0);
        for (int32_t j = 0; j < w; ++j) {
            const int64_t e = base + (int64_t)j * kSlice + lane;
            if (j < cnt) {
                col[e] = (int32_t)ci[first + j];
                val[e] = va[first + j];
            } else {
                col[e] = pad;
                val[e] = 0.0;
            }
        }
    }
}

template <class T>
bool dalloc(T **p, int64_t count, int64_t *bytes) {
    *p = nullptr;
    if (count <= 0) return true;
    if (cudaMalloc((void **)p, (size_t)count * sizeof(T)) != cudaSuccess) { *p = nullptr; return false; }
    if (bytes) *bytes += count * (int64_t)sizeof(T);
    return true;
}

// One part (P = 0 strictly lower, 1 strictly upper) of the split.
nsm_status build_part(int P, int64_t n, const int64_t *rp, const int64_t *ci, const double *va, const int32_t *cntL,
                      int64_t maxcnt, Sell *out, SellHost *host_geo, int64_t *bytes, std::string *err) {
    const int64_t ns = (n + kSlice - 1) / kSlice;
    const int32_t ucap = (int32_t)(2 * maxcnt + 8);
    int32_t *wid = nullptr, *ucnt = nullptr, *uni = nullptr;
    int64_t *sz = nullptr;
    SliceStats *st = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    nsm_status rc = NSM_OK;
    auto fail = [&](const char *m) { *err = m; rc = NSM_ERR_OOM; };
    if (!dalloc(&wid, ns, nullptr) || !dalloc(&ucnt, ns, nullptr) || !dalloc(&uni, ns * (int64_t)ucap, nullptr) ||
        !dalloc(&sz, ns + 1, nullptr) || !dalloc(&st, 1, nullptr) || cudaMemset(st, 0, sizeof(SliceStats)) != cudaSuccess) {
        fail("nsm_setup_device: temporary allocation failed");
    }
    SliceStats hs{};
    int aligned = 0;
    if (rc == NSM_OK) {
        k_slices<<<blocks_of(ns * 32), kThr>>>(P, n, ns, rp, ci, cntL, ucap, wid, ucnt, uni, st);
        if (cudaMemcpy(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost) != cudaSuccess) fail("nsm_setup_device: slice pass failed");
    }
    if (rc == NSM_OK) {
        // builder.cpp's decision: offset-aligned if it widens the slices by at
        // most 15 %, pads are at most 3 % of the stored entries and no slice's
        // union exceeds 2 w + 8
        const uint64_t su = hs.sum_u, sc = hs.sum_c, nz = hs.nnz;
        aligned = !(sc == 0 || hs.overflow || su * 100 > sc * 115 || (su * kSlice - nz) * 100 > su * kSlice * 3);
        k_slice_sizes<<<blocks_of(ns + 1), kThr>>>(ns, aligned, wid, ucnt, sz);
        cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sz, sz, (int)(ns + 1));
        if (cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 1)) != cudaSuccess) fail("nsm_setup_device: scan allocation failed");
    }
    int64_t tot = 0;
    if (rc == NSM_OK) {
        cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sz, sz, (int)(ns + 1));
        if (cudaMemcpy(&tot, sz + ns, sizeof(tot), cudaMemcpyDeviceToHost) != cudaSuccess) fail("nsm_setup_device: scan failed");
    }
    if (rc == NSM_OK) {
        out->ptr = sz;     // ownership moves to the part
        sz = nullptr;
        *bytes += (ns + 1) * (int64_t)sizeof(int64_t);
        out->padded = tot;
        out->nnz = (int64_t)hs.nnz;
        out->maxw = (int32_t)(aligned ? hs.maxu : hs.maxc);
        if (!dalloc(&out->col, tot, bytes) || !dalloc(&out->val, tot, bytes) ||
            (aligned && !dalloc(&out->off, tot / kSlice, bytes)))
            fail("nsm_setup_device: device allocation failed");
    }
    if (rc == NSM_OK && tot > 0) {
        k_fill<<<blocks_of(ns * 32), kThr>>>(P, aligned, n, ns, rp, ci, va, cntL, wid, ucnt, uni, ucap, out->ptr,
                                             out->col, out->val, out->off);
        if (cudaGetLastError() != cudaSuccess) fail("nsm_setup_device: fill kernel failed");
    }
    if (rc == NSM_OK && host_geo) {  // slice pointers and offsets on the host: gather-window plans
        host_geo->ptr.resize(ns + 1);
        host_geo->off.assign(aligned ? tot / kSlice : 0, 0);
        if (cudaMemcpy(host_geo->ptr.data(), out->ptr, (ns + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess ||
            (aligned && tot > 0 &&
             cudaMemcpy(host_geo->off.data(), out->off, (tot / kSlice) * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess))
            fail("nsm_setup_device: slice geometry copy failed");
        host_geo->maxw = out->maxw;
        host_geo->nnz = out->nnz;
    }
    cudaFree(wid);
    cudaFree(ucnt);
    cudaFree(uni);
    cudaFree(sz);
    cudaFree(st);
    cudaFree(tmp);
    return rc;
}

}  // namespace

nsm_status build_split_device(const nsm_csr *A, DevSplit *out, int64_t *bytes, std::string *err) {
    const int64_t n = A->nrows;
    if (n < 0 || !A->rowptr || A->ncols != n) {
        *err = "nsm_setup_device: A must be a square device CSR";
        return NSM_ERR_ARG;
    }
    if (n >= (int64_t)1 << 31) {
        *err = "nsm_setup_device: more than 2^31-1 rows is not supported (int32 device indices)";
        return NSM_ERR_ARG;
    }
    int64_t rp0 = 0, nnz = 0;
    if (cudaMemcpy(&rp0, A->rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&nnz, A->rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        *err = "nsm_setup_device: rowptr is not readable device memory";
        return NSM_ERR_ARG;
    }
    if (rp0 != 0) { *err = "nsm_setup: rowptr[0] != 0"; return NSM_ERR_PATTERN; }
    if (nnz > 0 && (!A->colind || !A->val)) { *err = "nsm_setup_device: NULL column or value array"; return NSM_ERR_ARG; }
    out->n = n;
    RowStats *st = nullptr;
    int32_t *cntL = nullptr;
    RowStats hs{};
    hs.bad = ~0ull;
    bool ok = dalloc(&st, 1, nullptr) && cudaMemcpy(st, &hs, sizeof(hs), cudaMemcpyHostToDevice) == cudaSuccess &&
              dalloc(&cntL, std::max<int64_t>(n, 1), nullptr) && dalloc(&out->d, std::max<int64_t>(n, 1), bytes) &&
              dalloc(&out->dl1, std::max<int64_t>(n, 1), bytes);
    if (ok && n > 0) {
        k_rows<<<blocks_of(n), kThr>>>(n, A->ncols, A->rowptr, A->colind, A->val, cntL, out->d, out->dl1, st);
        ok = cudaMemcpy(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost) == cudaSuccess;
    }
    nsm_status rc = NSM_OK;
    if (!ok) {
        cudaGetLastError();
        *err = "nsm_setup_device: row pass failed";
        rc = NSM_ERR_CUDA;
    } else if (hs.bad != ~0ull) {
        const int64_t row = (int64_t)(hs.bad >> 2);
        if ((hs.bad & 3) == 1) {
            *err = "nsm_setup: CSR pattern invariant violated at global row " + std::to_string(row);
            rc = NSM_ERR_PATTERN;
        } else {
            *err = "nsm_setup: missing or zero diagonal at global row " + std::to_string(row);
            rc = NSM_ERR_ZERO_DIAG;
        }
    }
    if (rc == NSM_OK) {
        out->nnz_off = (int64_t)hs.nnz_off;
        out->bw_lower = (int64_t)hs.bw[0];
        out->bw_upper = (int64_t)hs.bw[1];
        rc = build_part(0, n, A->rowptr, A->colind, A->val, cntL, (int64_t)hs.maxcnt[0], &out->L, &out->Lh, bytes, err);
        if (rc == NSM_OK)
            rc = build_part(1, n, A->rowptr, A->colind, A->val, cntL, (int64_t)hs.maxcnt[1], &out->U, &out->Uh, bytes, err);
    }
    if (rc == NSM_OK && cudaDeviceSynchronize() != cudaSuccess) {
        cudaGetLastError();
        *err = "nsm_setup_device: builder kernels failed";
        rc = NSM_ERR_CUDA;
    }
    cudaFree(st);
    cudaFree(cntL);
    return rc;
}

}  // namespace nsm
