// transpose.cu — U read as L^T for a symmetric A (DESIGN.md §6 "Symmetric
// residual").
//
// The residual r = b - (L + D + U) x (the first step of every
// smoother application, Alg. 1 line 4 / P:L485) streams both strict
// triangles.  When A is symmetric — the paper's pressure-Poisson systems
// (Nalu-Wind) are — U = L^T holds the same numbers as L, and
// the windowed residual kernel (stream.cu) can take U's values from L's
// value array instead of streaming U: the residual's matrix bytes drop from
// 2 x 8 B to 8 B (+ 0.5 B of map) per strict entry.  Values, products and
// the order of the additions are unchanged (the row's U entries still
// multiply in ascending column order), so results stay bit-identical; the
// map is only installed when every value it would produce — real entries
// and pads — equals U's stored value bit for bit (checked here on the
// device), otherwise the kernels stream U as before.
//
// With the offset-aligned layout slot j of U's slice s holds offset o for
// all 32 rows; the mirrored entries A(i + o, i) of rows i = 32 s + l are L's
// entries of rows 32 s + o + l at offset -o: at most two of L's slices
// (sa = (32 s + o) / 32 and sa + 1), one slot in each.  One warp per U
// slice finds those slots (a ballot over the slices' offset lists), writes
// the map entry (nsm_internal.h tmap_addr decodes it) and compares all 32
// values with U's.  The map is dense per slice (U.maxw entries), so a kernel
// locates the entries of any slice without reading U's slice pointers.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "nsm_internal.h"

namespace nsm {

namespace {

constexpr int kWarpsPerBlock = 8;

// Element index of the slot holding offset `o` in L's slice q (-1: none).
__device__ __forceinline__ int64_t find_slot(int64_t q, int64_t nslices, const int64_t *__restrict__ lptr,
                                             const int32_t *__restrict__ loff, int32_t o, int lane) {
    if (q >= nslices) return -1;
    const int64_t b = lptr[q], w = (lptr[q + 1] - b) / kSlice;
    for (int64_t k0 = 0; k0 < w; k0 += 32) {
        const int64_t k = k0 + lane;
        const unsigned hit = __ballot_sync(0xffffffffu, k < w && loff[b / kSlice + k] == o);
        if (hit) return b + (k0 + __ffs(hit) - 1) * kSlice;
    }
    return -1;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_tmap(int64_t n, int64_t nslices, int32_t tw, const int64_t *__restrict__ lptr, const int32_t *__restrict__ loff,
           const double *__restrict__ lval, const int64_t *__restrict__ uptr, const int32_t *__restrict__ uoff,
           const double *__restrict__ uval, int2 *__restrict__ tmap, unsigned int *mismatch) {
    const int64_t s = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s >= nslices) return;
    const int64_t ub = uptr[s], w = (uptr[s + 1] - ub) / kSlice;
    const int64_t i = s * kSlice + lane;
    bool bad = false;
    for (int64_t j = 0; j < tw; ++j) {
        int2 t = make_int2(INT32_MIN, INT32_MIN);
        if (j < w) {
            const int32_t o = uoff[ub / kSlice + j];  // > 0: a strictly upper offset
            const int64_t r0 = s * kSlice + o;         // mirrored row of lane 0
            const int64_t sa = r0 / kSlice;
            const int sh = (int)(r0 % kSlice);
            const int64_t ea = find_slot(sa, nslices, lptr, loff, -o, lane);
            const int64_t eb = sh ? find_slot(sa + 1, nslices, lptr, loff, -o, lane) : -1;
            t.x = ea >= 0 ? (int32_t)(ea + sh) : (INT32_MIN | sh);
            t.y = eb >= 0 ? (int32_t)(eb + sh - kSlice) : INT32_MIN;
            if (i < n) {
                const int64_t a = tmap_addr(t.x, t.y, lane);
                const double m = a >= 0 ? lval[a] : 0.0;
                const double u = uval[ub + j * kSlice + lane];
                bad |= __double_as_longlong(m) != __double_as_longlong(u);
            }
        }
        if (lane == 0) tmap[s * tw + j] = t;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(mismatch, 1u);
}

}  // namespace

cudaError_t build_tmap(int64_t n, const Sell &L, Sell *U, int64_t *bytes, bool *built) {
    *built = false;
    // (the producer holds a tile's 8 x maxw entries in 4 registers per lane: maxw <= 16)
    if (!L.off || !U->off || n <= 0 || U->padded == 0 || U->maxw > 16 || L.padded >= ((int64_t)1 << 31) - 64)
        return cudaSuccess;
    const int64_t nslices = (n + kSlice - 1) / kSlice;
    const int32_t tw = std::max(U->maxw, 1);
    const int64_t entries = nslices * tw;
    int2 *tm = nullptr;
    unsigned int *flag = nullptr;
    cudaError_t e = cudaMalloc((void **)&tm, (size_t)entries * sizeof(int2));
    if (e == cudaSuccess) e = cudaMalloc((void **)&flag, sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemset(flag, 0, sizeof(unsigned int));
    if (e == cudaSuccess) {
        const int64_t blocks = (nslices + kWarpsPerBlock - 1) / kWarpsPerBlock;
        k_tmap<<<(unsigned)blocks, kWarpsPerBlock * 32>>>(n, nslices, tw, L.ptr, L.off, L.val, U->ptr, U->off, U->val,
                                                         tm, flag);
        e = cudaGetLastError();
    }
    unsigned int mismatch = 1;
    if (e == cudaSuccess) e = cudaMemcpy(&mismatch, flag, sizeof(mismatch), cudaMemcpyDeviceToHost);
    cudaFree(flag);
    if (e != cudaSuccess || mismatch) {
        cudaFree(tm);
        return e;
    }
    U->tmap = tm;
    U->tmap_w = tw;
    *bytes += entries * (int64_t)sizeof(int2);
    *built = true;
    return cudaSuccess;
}

}  // namespace nsm
