// stream_dev.cuh — device-side building blocks of the bulk-copy pipelined
// kernels: shared-memory stage layout, the producer warp that
// stages a tile (values, offsets / window positions, slice header, gather
// window) and the consumers' register chunks.  Used by stream.cu (one kernel
// per pass) and coupled.cu (the passes of one application as concurrent
// warp groups).  Included inside namespace nsm.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "nsm_internal.h"
#include "ptx.cuh"

namespace nsm {

namespace {

constexpr int kTS = kTileSlices;          // slices (consumer warps) per tile
constexpr int kThreadsT = (kTS + 1) * 32; // + 1 producer warp

using ptx::mbar_arrive;
using ptx::mbar_expect_tx;
using ptx::mbar_init;
using ptx::mbar_wait;
using ptx::bulk_g2s;
__device__ __forceinline__ uint64_t policy_evict_first_t() { return ptx::policy_evict_first(); }

// Programmatic dependent launch: the kernels are launched with
// programmatic stream serialisation, so a kernel's CTAs may start while the
// previous kernel drains.  Only the immutable matrix streams (the producer's
// bulk copies) are touched before griddepcontrol.wait; everything produced
// by the previous kernel (x, r, g, y, z) is read after it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

struct GatherPlainT {
    const double *__restrict__ g;
    __device__ __forceinline__ double operator()(int32_t c) const { return __ldg(g + c); }
};
struct GatherScaledT {
    const double *__restrict__ rhs;
    const double *__restrict__ d;
    __device__ __forceinline__ double operator()(int32_t c) const { return __ddiv_rn(__ldg(rhs + c), __ldg(d + c)); }
};

// Shared-memory layout: full[NST], empty[NST] mbarriers, then NST stages of
// NP parts of {val[cap], col[cap]} with cap = kTS * 32 * maxw entries.
// With the offset-aligned layout (ofs) only the values are staged (8 B per
// entry); columns are row + offset.  That layout's parts also carry a header
// written by the producer warp: per slice of the tile, {first entry relative
// to the tile, width}, so consumers take the slice geometry from shared memory
// after the stage wait instead of a global round trip of their own per tile.
constexpr int kHdrBytes = kTS * 2 * 4;

#ifndef NSM_RES_PREFETCH_U
#define NSM_RES_PREFETCH_U 1  // wide-row residual: prefetch U's gathers to L1 (C3 -1.2 %; tools/experiments/README.md)
#endif

struct Layout {
    int nst, np;
    int64_t cap;  // entries per part per stage
    int eb;       // staged bytes per entry: 12 (values + columns) or 8 (values; + the slices' offsets + header)
    int64_t wcap = 0;  // gather-window doubles per stage (windowed kernels), after all stages' parts
    __host__ __device__ static int64_t ofs_bytes(int64_t cap) { return (cap / kSlice * 4 + 15) / 16 * 16; }
    __host__ __device__ static int64_t part_bytes(int64_t cap, int eb) {
        return eb == 12 ? cap * 12 : cap * 8 + ofs_bytes(cap) + kHdrBytes;
    }
    __device__ __forceinline__ int32_t *hdr(char *s, int st, int p) const {  // eb 8 only
        return (int32_t *)(s + 128 + ((int64_t)st * np + p) * part_bytes(cap, eb) + cap * 8 + ofs_bytes(cap));
    }
    __device__ __forceinline__ uint64_t *full(char *s) const { return (uint64_t *)s; }
    __device__ __forceinline__ uint64_t *empty(char *s) const { return (uint64_t *)s + nst; }
    __device__ __forceinline__ double *val(char *s, int st, int p) const {
        return (double *)(s + 128 + ((int64_t)st * np + p) * part_bytes(cap, eb));
    }
    __device__ __forceinline__ int32_t *col(char *s, int st, int p) const {   // eb 12: columns; eb 8: offsets
        return (int32_t *)(s + 128 + ((int64_t)st * np + p) * part_bytes(cap, eb) + cap * 8);
    }
    __device__ __forceinline__ double *win(char *s, int st) const {
        return (double *)(s + 128 + (int64_t)nst * np * part_bytes(cap, eb)) + (int64_t)st * wcap;
    }
};

__device__ __forceinline__ void init_barriers(const Layout &Ly, char *sm) {
    if (threadIdx.x == 0) {
        for (int st = 0; st < Ly.nst; ++st) {
            mbar_init(Ly.full(sm) + st, 1);
            mbar_init(Ly.empty(sm) + st, kTS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

// Producer: stream the parts' segments of each of this CTA's tiles.
// Producer warp: stream the parts' segments of each of this CTA's tiles.  Lane
// 0 issues the bulk copies; with the offset-aligned layout (eb 8) the whole
// warp also copies the tile's slice offsets into the stage (plain loads; a
// 4-byte-aligned segment the bulk engine cannot take), ordered before the
// stage's arrival by __syncwarp.  Software-pipelined: the slice pointers and
// offsets of the CTA's next tile are loaded while the current one is staged,
// so neither round trip sits on the producer's per-tile path.
constexpr int kOfsPerLane = 4;  // staged offsets per lane and part (8 slices x 16 entries)

template <int NP>
struct TileRefs {
    int64_t b[NP], e[NP];
    int64_t sp[NP];  // lanes 0..kTS: slice pointer of slice s0 + lane (clamped to the tile end)
    int32_t o[NP][kOfsPerLane];
    // windowed kernels: this tile's gather-window segments, lane k holds segment k
    int32_t nseg, sg_len, sg_base;
    int64_t sg_lo;
    int32_t wg0;  // producer_deep: the tile's first window segment (between its two load phases)
};

// Entry-position arrays staged into the "offsets" slot: the column offsets,
// or (windowed kernels) the gather-window positions.
template <int NP>
__device__ __forceinline__ const int32_t *staged_pos(const SellView (&P)[NP], const WinView &W, bool win, int p) {
    return win ? W.wpos[p] : P[p].off;
}

template <int NP>
__device__ __forceinline__ void tile_refs(const Layout &Ly, const SellView (&P)[NP], int64_t s_begin, int64_t s_end,
                                          int64_t t, int lane, TileRefs<NP> &r, const WinView &W, bool win) {
    const int64_t s0 = s_begin + t * kTS, s1 = min(s0 + kTS, s_end);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        r.b[p] = __ldg(P[p].ptr + s0);
        r.e[p] = __ldg(P[p].ptr + s1);
    }
    if (Ly.eb == 8) {
#pragma unroll
        for (int p = 0; p < NP; ++p) r.sp[p] = lane <= kTS ? __ldg(P[p].ptr + min(s0 + lane, s1)) : 0;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int64_t no = (r.e[p] - r.b[p]) / kSlice;
            const int32_t *go = staged_pos<NP>(P, W, win, p) + r.b[p] / kSlice;
#pragma unroll
            for (int q = 0; q < kOfsPerLane; ++q) {
                const int64_t k = lane + 32 * q;
                r.o[p][q] = k < no ? __ldg(go + k) : 0;
            }
        }
    }
    if (win) {  // tile s0 / kTS of the window plan (s_begin is a multiple of kTS)
        const int64_t wt = s0 / kTS;
        const int32_t g0 = __ldg(W.tseg + wt), g1 = __ldg(W.tseg + wt + 1);
        r.nseg = g1 - g0;
        if (lane < r.nseg) {
            r.sg_lo = __ldg(W.glo + g0 + lane);
            r.sg_len = __ldg(W.len + g0 + lane);
            r.sg_base = __ldg(W.sbase + g0 + lane);
        }
    }
}

// Compact layout (values + columns, 12 B per entry): one lane, no prefetch
// (the software-pipelined warp version below measured ~1.5 % slower here).
template <int NP>
__device__ __forceinline__ void producer_compact(const Layout &Ly, char *sm, const SellView (&P)[NP], int64_t s_begin,
                                                 int64_t s_end, int64_t ntiles) {
    const uint64_t pol = policy_evict_first_t();
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % Ly.nst;
        const uint32_t use = (uint32_t)(it / Ly.nst);
        if (it >= Ly.nst) mbar_wait(Ly.empty(sm) + st, (use - 1) & 1);
        const int64_t s0 = s_begin + t * kTS, s1 = min(s0 + kTS, s_end);
        int64_t b[NP], e[NP];
        uint32_t bytes = 0;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            b[p] = __ldg(P[p].ptr + s0);
            e[p] = __ldg(P[p].ptr + s1);
            bytes += (uint32_t)((e[p] - b[p]) * 12);
        }
        mbar_expect_tx(Ly.full(sm) + st, bytes);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            if (e[p] > b[p]) {
                bulk_g2s(Ly.val(sm, st, p), P[p].val + b[p], (uint32_t)((e[p] - b[p]) * 8), Ly.full(sm) + st, pol);
                bulk_g2s(Ly.col(sm, st, p), P[p].col + b[p], (uint32_t)((e[p] - b[p]) * 4), Ly.full(sm) + st, pol);
            }
        }
    }
    pdl_trigger();  // all of this CTA's copies are issued: dependents may be scheduled
}

// WIN: also stage the tile's gather window of `vec` (the vector the
// consumers gather: x for the residual, the previous iterate for a sweep):
// each lane owns one segment, bulk-copies its in-range, 16-byte-aligned part
// and writes the rest itself (zeros outside [0, n), an odd last element).
// `vec` is written by the previous kernel, so with programmatic dependent
// launch the producer waits for it before the first window copy.
// Hook points of the producer (coupled.cu): the tile sequence (first tile,
// stride), a wait before a tile is staged (dependencies on other warp groups'
// progress), extra bulk-copied bytes per tile and their copies, and the L2
// policy of each part's values.  NoHook is the one-kernel-per-pass schedule.
struct NoHook {
    __device__ __forceinline__ int64_t first() const { return blockIdx.x; }
    __device__ __forceinline__ int64_t stride() const { return gridDim.x; }
    __device__ __forceinline__ void before(int64_t, int, int) {}
    __device__ __forceinline__ uint32_t extra_bytes(int64_t) const { return 0; }
    __device__ __forceinline__ void extra_copy(int64_t, int, uint64_t *) const {}
    __device__ __forceinline__ uint64_t val_policy(int, uint64_t pol) const { return pol; }
};

template <int NP, bool WIN = false, class Hook = NoHook>
__device__ __forceinline__ void producer(const Layout &Ly, char *sm, const SellView (&P)[NP], int64_t s_begin,
                                         int64_t s_end, int64_t ntiles, int lane, const WinView &W = WinView{},
                                         const double *vec = nullptr, int64_t n = 0, Hook hook = Hook{}) {
    const uint64_t pol = policy_evict_first_t();
    const uint64_t pol_win = ptx::policy_evict_normal();  // neighbouring tiles (other CTAs) gather it too
    int it = 0, st = 0;
    uint32_t ph = 0;  // (it / nst) & 1
    TileRefs<NP> cur, nxt;
    const int64_t t_first = hook.first(), t_stride = hook.stride();
    if (WIN) pdl_wait();
    if (t_first < ntiles) tile_refs<NP>(Ly, P, s_begin, s_end, t_first, lane, cur, W, WIN);
    for (int64_t t = t_first; t < ntiles; t += t_stride, ++it) {
        if (t + t_stride < ntiles) tile_refs<NP>(Ly, P, s_begin, s_end, t + t_stride, lane, nxt, W, WIN);  // prefetch
        if (it >= Ly.nst) mbar_wait(Ly.empty(sm) + st, ph ^ 1);
        hook.before(t, st, lane);
        uint32_t bytes = hook.extra_bytes(t);
#pragma unroll
        for (int p = 0; p < NP; ++p) bytes += (uint32_t)((cur.e[p] - cur.b[p]) * Ly.eb);
        int64_t wa = 0;         // this lane's window segment: bulk part [wa, wa + wbytes / 8)
        uint32_t wbytes = 0;
        if (WIN && lane < cur.nseg) {
            double *ws = Ly.win(sm, st) + cur.sg_base - cur.sg_lo;  // ws[q] = window slot of vec[q]
            const int64_t lo = cur.sg_lo, hi = lo + cur.sg_len;
            const int64_t a = max(lo, (int64_t)0), e = min(hi, n);
            for (int64_t q = lo; q < min(a, hi); ++q) ws[q] = 0.0;           // below row 0
            for (int64_t q = max(e, lo); q < hi; ++q) ws[q] = 0.0;           // past row n - 1
            if (e > a) {
                const int64_t be = e & ~(int64_t)1;
                if (be < e) ws[e - 1] = __ldcg(vec + e - 1);                  // odd n: last element
                wa = a;
                wbytes = be > a ? (uint32_t)((be - a) * 8) : 0u;
            }
        }
        if (WIN) {
            uint32_t wsum = wbytes;
#pragma unroll
            for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
            bytes += wsum;
        }
        if (Ly.eb == 8) {
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                int32_t *so = Ly.col(sm, st, p);
                const int64_t no = (cur.e[p] - cur.b[p]) / kSlice;
#pragma unroll
                for (int q = 0; q < kOfsPerLane; ++q) {
                    const int64_t k = lane + 32 * q;
                    if (k < no) so[k] = cur.o[p][q];
                }
                const int32_t *go = staged_pos<NP>(P, W, WIN, p) + cur.b[p] / kSlice;  // wider tiles (not staged above)
                for (int64_t k = lane + 32 * kOfsPerLane; k < no; k += 32) so[k] = __ldg(go + k);
                const int64_t nsp = __shfl_down_sync(0xffffffffu, cur.sp[p], 1);
                if (lane < kTS) {
                    int32_t *h = Ly.hdr(sm, st, p);
                    h[2 * lane] = (int32_t)(cur.sp[p] - cur.b[p]);
                    h[2 * lane + 1] = (int32_t)((nsp - cur.sp[p]) / kSlice);
                }
            }
            __syncwarp();
        }
        if (WIN) __syncwarp();  // the window's plain stores precede the arrival (release)
        if (lane == 0) {
            mbar_expect_tx(Ly.full(sm) + st, bytes);  // bulk-copied bytes (values, and columns with eb 12)
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const int64_t b = cur.b[p], e = cur.e[p];
                if (e > b) {
                    bulk_g2s(Ly.val(sm, st, p), P[p].val + b, (uint32_t)((e - b) * 8), Ly.full(sm) + st,
                             hook.val_policy(p, pol));
                    if (Ly.eb == 12)
                        bulk_g2s(Ly.col(sm, st, p), P[p].col + b, (uint32_t)((e - b) * 4), Ly.full(sm) + st, pol);
                }
            }
            hook.extra_copy(t, st, Ly.full(sm) + st);
        }
        if (WIN) {
            __syncwarp();  // the expected byte count is registered before any window copy completes
            if (wbytes)
                bulk_g2s(Ly.win(sm, st) + cur.sg_base + (wa - cur.sg_lo), vec + wa, wbytes, Ly.full(sm) + st, pol_win);
        }
        __syncwarp();
        cur = nxt;
        if (++st == Ly.nst) { st = 0; ph ^= 1; }
    }
    if (lane == 0) pdl_trigger();  // all of this CTA's copies are issued: dependents may be scheduled
}

// Two-phase tile references for producer_deep: phase A loads what depends
// only on the tile index (slice pointers, the window plan's segment range),
// phase B what depends on phase A (offsets / window positions, segments).
template <int NP>
__device__ __forceinline__ void tile_refs_a(const SellView (&P)[NP], int64_t s_begin, int64_t s_end, int64_t t,
                                            int lane, TileRefs<NP> &r, const WinView &W) {
    const int64_t s0 = s_begin + t * kTS, s1 = min(s0 + kTS, s_end);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        r.b[p] = __ldg(P[p].ptr + s0);
        r.e[p] = __ldg(P[p].ptr + s1);
        r.sp[p] = lane <= kTS ? __ldg(P[p].ptr + min(s0 + lane, s1)) : 0;
    }
    const int64_t wt = s0 / kTS;
    r.wg0 = __ldg(W.tseg + wt);
    r.nseg = __ldg(W.tseg + wt + 1);   // the end; phase B turns it into the count
}
template <int NP>
__device__ __forceinline__ void tile_refs_b(const SellView (&P)[NP], int lane, TileRefs<NP> &r, const WinView &W) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int64_t no = (r.e[p] - r.b[p]) / kSlice;
        const int32_t *go = W.wpos[p] + r.b[p] / kSlice;
#pragma unroll
        for (int q = 0; q < kOfsPerLane; ++q) {
            const int64_t k = lane + 32 * q;
            r.o[p][q] = k < no ? __ldg(go + k) : 0;
        }
    }
    r.nseg -= r.wg0;
    if (lane < r.nseg) {
        r.sg_lo = __ldg(W.glo + r.wg0 + lane);
        r.sg_len = __ldg(W.len + r.wg0 + lane);
        r.sg_base = __ldg(W.sbase + r.wg0 + lane);
    }
}

// The windowed producer (offset-aligned parts, gather window) with its tile
// references loaded three tiles ahead in two phases, so neither dependent
// round trip sits on the producer's per-tile path: one producer warp then
// keeps up with tiles arriving at several times the per-pass rate (the
// coupled sweeps, coupled.cu).  Same staging as producer<NP, true, Hook>.
template <int NP, class Hook>
__device__ __forceinline__ void producer_deep(const Layout &Ly, char *sm, const SellView (&P)[NP], int64_t s_begin,
                                              int64_t s_end, int64_t ntiles, int lane, const WinView &W,
                                              const double *vec, int64_t n, Hook hook) {
    const uint64_t pol = policy_evict_first_t();
    const uint64_t pol_win = ptx::policy_evict_normal();
    int it = 0, st = 0;
    uint32_t ph = 0;
    const int64_t t_first = hook.first(), G = hook.stride();
    // cur: tile t (complete); nxt: t + G (phase A landed, phase B in flight); nn: t + 2G (phase A in flight)
    TileRefs<NP> cur, nxt, nn;
    if (t_first < ntiles) {
        tile_refs_a<NP>(P, s_begin, s_end, t_first, lane, cur, W);
        tile_refs_b<NP>(P, lane, cur, W);
    }
    if (t_first + G < ntiles) {
        tile_refs_a<NP>(P, s_begin, s_end, t_first + G, lane, nxt, W);
        tile_refs_b<NP>(P, lane, nxt, W);
    }
    if (t_first + 2 * G < ntiles) tile_refs_a<NP>(P, s_begin, s_end, t_first + 2 * G, lane, nn, W);
    for (int64_t t = t_first; t < ntiles; t += G, ++it) {
        if (it >= Ly.nst) mbar_wait(Ly.empty(sm) + st, ph ^ 1);
        hook.before(t, st, lane);
        uint32_t bytes = hook.extra_bytes(t);
#pragma unroll
        for (int p = 0; p < NP; ++p) bytes += (uint32_t)((cur.e[p] - cur.b[p]) * 8);
        int64_t wa = 0;
        uint32_t wbytes = 0;
        if (lane < cur.nseg) {
            double *ws = Ly.win(sm, st) + cur.sg_base - cur.sg_lo;
            const int64_t lo = cur.sg_lo, hi = lo + cur.sg_len;
            const int64_t a = max(lo, (int64_t)0), e = min(hi, n);
            for (int64_t q = lo; q < min(a, hi); ++q) ws[q] = 0.0;
            for (int64_t q = max(e, lo); q < hi; ++q) ws[q] = 0.0;
            if (e > a) {
                const int64_t be = e & ~(int64_t)1;
                if (be < e) ws[e - 1] = __ldcg(vec + e - 1);
                wa = a;
                wbytes = be > a ? (uint32_t)((be - a) * 8) : 0u;
            }
        }
        {
            uint32_t wsum = wbytes;
#pragma unroll
            for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
            bytes += wsum;
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            int32_t *so = Ly.col(sm, st, p);
            const int64_t no = (cur.e[p] - cur.b[p]) / kSlice;
#pragma unroll
            for (int q = 0; q < kOfsPerLane; ++q) {
                const int64_t k = lane + 32 * q;
                if (k < no) so[k] = cur.o[p][q];
            }
            const int32_t *go = W.wpos[p] + cur.b[p] / kSlice;
            for (int64_t k = lane + 32 * kOfsPerLane; k < no; k += 32) so[k] = __ldg(go + k);
            const int64_t nsp = __shfl_down_sync(0xffffffffu, cur.sp[p], 1);
            if (lane < kTS) {
                int32_t *h = Ly.hdr(sm, st, p);
                h[2 * lane] = (int32_t)(cur.sp[p] - cur.b[p]);
                h[2 * lane + 1] = (int32_t)((nsp - cur.sp[p]) / kSlice);
            }
        }
        __syncwarp();  // the plain stores (offsets, header, window fill) precede the arrival
        if (lane == 0) {
            mbar_expect_tx(Ly.full(sm) + st, bytes);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const int64_t b = cur.b[p], e = cur.e[p];
                if (e > b)
                    bulk_g2s(Ly.val(sm, st, p), P[p].val + b, (uint32_t)((e - b) * 8), Ly.full(sm) + st,
                             hook.val_policy(p, pol));
            }
            hook.extra_copy(t, st, Ly.full(sm) + st);
        }
        __syncwarp();  // the expected byte count is registered before any window copy completes
        if (wbytes)
            bulk_g2s(Ly.win(sm, st) + cur.sg_base + (wa - cur.sg_lo), vec + wa, wbytes, Ly.full(sm) + st, pol_win);
        __syncwarp();
        // rotate: each slot's loads were issued one iteration ago
        cur = nxt;
        nxt = nn;
        if (t + 2 * G < ntiles) tile_refs_b<NP>(P, lane, nxt, W);
        if (t + 3 * G < ntiles) tile_refs_a<NP>(P, s_begin, s_end, t + 3 * G, lane, nn, W);
        if (++st == Ly.nst) { st = 0; ph ^= 1; }
    }
}

// Register chunk of one row taken from the staged copy: the first CH entries
// (predicated on the slice width w) are read from shared memory, all their
// gathers issued together, and multiplied; add() sums them in stored order
// and continues with any entries beyond CH one by one.
// Slice offsets of the offset-aligned layout, loaded (warp-uniform) before
// the stage wait: column of entry j = row + o[j], or the row itself when out
// of range (a pad) — the builder's column for that pad, so the products are
// those of the column-array path.
// Slice offsets of the offset-aligned layout, staged by the producer: column of
// entry j = row + o[j], or the row itself when out of range (a pad) — the
// builder's column for that pad, so the products are those of the
// column-array path.
template <int CH>
struct Offsets {
    const int32_t *so;    // this slice's offsets in the stage
    __device__ __forceinline__ void at(const int32_t *stage_offs, int64_t lo) { so = stage_offs + lo / kSlice; }
    // 32-bit unsigned arithmetic (rows and columns < 2^31): one compare on
    // the gather's dependent path (the 64-bit form cost ~10 % on C3).  Only
    // called for rows i < n (load_ofs gives the lanes past n width 0).
    __device__ __forceinline__ static int32_t col(int64_t i, int32_t off, int64_t n) {
        const uint32_t c = (uint32_t)((int32_t)i + off);
        return c < (uint32_t)n ? (int32_t)c : (int32_t)i;
    }
};

template <int CH>
struct StagedChunk {
    double v[CH];
    int32_t c[CH];
    const double *sv;
    const int32_t *sc;
    const int32_t *otail;  // offset-aligned layout: offsets of the entries beyond CH
    int64_t row, n;
    int w;
    __device__ __forceinline__ void load(const double *sv_, const int32_t *sc_, int64_t off, int w_, int lane) {
        sv = sv_ + off + lane;
        sc = sc_ + off + lane;
        otail = nullptr;
        w = w_;
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) {
                v[j] = sv[j * kSlice];
                c[j] = sc[j * kSlice];
            }
    }
    __device__ __forceinline__ void load_ofs(const double *sv_, const Offsets<CH> &of, int64_t off, int w_, int lane,
                                             int64_t row_, int64_t n_) {
        sv = sv_ + off + lane;
        otail = of.so;
        row = row_;
        n = n_;
        w = row_ < n_ ? w_ : 0;  // lanes past n in the last slice: nothing (a pad's column i would be out of bounds)
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) {
                v[j] = sv[j * kSlice];
                c[j] = Offsets<CH>::col(row, of.so[j], n);
            }
    }
    template <class G>
    __device__ __forceinline__ void gather_mul(const G &g) {
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) v[j] = __dmul_rn(v[j], g(c[j]));
    }
    template <class G>
    __device__ __forceinline__ double add(double acc, const G &g) const {
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) acc = __dadd_rn(acc, v[j]);
        for (int j = CH; j < w; ++j) {
            const int32_t cj = otail ? Offsets<CH>::col(row, otail[j], n) : sc[j * kSlice];
            acc = __dadd_rn(acc, __dmul_rn(sv[j * kSlice], g(cj)));
        }
        return acc;
    }
};


// Windowed gathers (WIN kernels): entry j of this lane's row multiplies the
// gathered vector's value at window slot wp[j] + lane (staged by the
// producer with the tile), so a row's products need shared-memory loads only.
// Same products and the same stored-order additions as StagedChunk.
template <int CH>
struct WinChunk {
    double v[CH];
    const double *sv;   // this lane's values of the slice
    const int32_t *wp;  // the slice's window positions (warp-uniform)
    const double *ws;   // window + lane
    int w;
    __device__ __forceinline__ void load(const double *sv_, const int32_t *stage_pos, const double *win, int64_t off,
                                         int w_, int lane, bool row) {
        sv = sv_ + off + lane;
        wp = stage_pos + off / kSlice;
        ws = win + lane;
        w = row ? w_ : 0;
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) v[j] = __dmul_rn(sv[j * kSlice], ws[wp[j]]);
    }
    __device__ __forceinline__ double add(double acc) const {
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) acc = __dadd_rn(acc, v[j]);
        for (int j = CH; j < w; ++j) acc = __dadd_rn(acc, __dmul_rn(sv[j * kSlice], ws[wp[j]]));
        return acc;
    }
};

// The same sum in chunks of CH entries (each chunk's products in flight
// together, added in stored order): fewer registers than one wide chunk.
template <int CH>
__device__ __forceinline__ double win_sum_chunked(const double *sv_, const int32_t *stage_pos, const double *win,
                                                  int64_t off, int w, int lane, bool row, double acc) {
    const double *sv = sv_ + off + lane;
    const int32_t *wp = stage_pos + off / kSlice;
    const double *ws = win + lane;
    if (!row) return acc;
    for (int j0 = 0; j0 < w; j0 += CH) {
        double v[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j0 + j < w) v[j] = __dmul_rn(sv[(j0 + j) * kSlice], ws[wp[j0 + j]]);
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j0 + j < w) acc = __dadd_rn(acc, v[j]);
    }
    return acc;
}

}  // namespace

}  // namespace nsm
