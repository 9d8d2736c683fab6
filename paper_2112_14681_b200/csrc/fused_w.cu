// fused_w.cu — one-pass pGS application for offset-aligned (stencil-like)
// matrices with gather windows: the residual, the k Jacobi sweeps and the x
// update in ONE launch that reads each matrix entry from HBM about once
// (SURVEY.md §7.3, §8(d) "fused floor"; the pGS application of P:L743-785):
//
//   phase 0 (tile u):  r = b - A x,  g(0) = r / d        (eq:jr-initial-guess)
//   phase j (tile u):  g(j) = (r - L g(j-1)) / d         (eq:jacobi), j = 1..k
//                      the last one x += g(k)
//
// Dependencies.  Phase j of 256-row tile u needs phase j-1 of the tiles
// within L's bandwidth below it, [u - DT, u].  Work item w bundles phase j of
// tile w - jD, j = 0..k (D > DT); items are dealt round-robin to a
// cooperative grid (item w to CTA w mod G) and every CTA runs its items'
// units in (item, phase) order.
//
// Readiness is tracked PER PHASE: prog[j][c] counts the items of CTA c whose
// phase-j unit is complete, so "phase j done for all items < F_j" with
// F_j = min_c (c + count_j(c) G).  Before staging unit (j, u) of item w the
// producer warp requires
//   F_{j-1} > w - D                        (its gathered iterate g(j-1) and r)
//   F_0 > u + DA            (j = k)        (x of tile u: every residual reading it is done)
//   F_{j+1} > u - Mg + DT + (j+1) D (j < k) (the ring slot it writes is no longer read)
//   F_k > u - Mr + kD       (j = 0)        (the r slot it writes is no longer read)
// each a statement about strictly earlier (item, phase) pairs, so the lowest
// unfinished unit can always proceed (deadlock-free with all CTAs resident).
// With per-phase frontiers D need only exceed DT by a small margin: the
// matrix rows a later phase re-reads were streamed about k D tiles earlier
// (C3: ~2 planes, ~30 MB) and are still in L2, and the iterates live in
// L2-resident rings of a few MB.
//
// Data movement (all through shared memory, no gathers from global memory):
// the producer warp stages, per unit, the tile's values of L (and U for
// phase 0), the window positions and slice geometry, and the gather window —
// of x for phase 0 (builder.cpp's residual window), of the ring g(j-1) for a
// sweep (the L window mapped into the ring) — with cp.async.bulk, after the
// readiness wait (acquire + proxy fence: the ring was written by other CTAs
// through the generic proxy).  Consumers (one row per thread) read own-row
// vectors directly, multiply values by window entries and add in stored
// order: the same arithmetic as the per-pass kernels and the oracle, so
// results are bit-identical.  Each unit is published by the last consumer
// warp to finish it (CTA-scope acq_rel count, then red.release.gpu).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <map>
#include <mutex>
#include <tuple>

#include "nsm_internal.h"
#include "ptx.cuh"

namespace nsm {

namespace {

constexpr int kWC = 8;                    // consumer warps = slices per tile
constexpr int kRowsW = kWC * kSlice;      // 256 rows per tile (the window plans' tiles)
constexpr int kThreadsW = (kWC + 1) * 32;
constexpr int kMaxStW = 4;
constexpr int kHdrW = 256;                // barriers, counters, unit descriptors
constexpr int64_t kSmemMaxW = 220 * 1024;

struct FwParams {
    int64_t n, nslices, ntiles, nitems;
    int k, D, DT, DA, fresh, maxph;
    int64_t Mr, Mg;                // ring lengths in tiles (powers of two)
    SellView L, U;
    WinView WR, WL;                // gather windows of U and of L
    // per-tile padded copies of the windows (fw_tables): positions [t][pst],
    // segment count [t], segments [t][32] = {glo lo, glo hi, len, sbase}, so a
    // unit's metadata loads do not depend on each other
    const int32_t *tposL, *tposU, *nsegL, *nsegU;
    const int4 *tsegL, *tsegU;
    int pst;
    int64_t tpp, nplanes;          // plane schedule: tiles per plane (= grid), planes
    const double *d, *b;
    double *x;
    double *ring_r, *ring_g;       // ring_g: k rings of Mg tiles each
    unsigned long long *prog;      // [kMaxPhW][pstride] per-CTA progress per phase
    int64_t pstride;
    unsigned long long *flag;
    int64_t sweep_id0;
    unsigned int *err;
    unsigned long long timeout_ns;
    unsigned int *sync;            // [0] epoch, [1] CTAs finished, [4..5] polls, [6..7] poll ns (u64)
    int nst;
    int64_t cap;                   // entries per part per stage
    int64_t wcap;                  // window doubles per stage
    int64_t stage_bytes;
};

struct UDescW {
    int u;        // tile, -1: empty unit
    int j;
};

__device__ __forceinline__ uint64_t *fullb(char *s) { return (uint64_t *)s; }
__device__ __forceinline__ uint64_t *emptyb(char *s) { return (uint64_t *)s + kMaxStW; }
__device__ __forceinline__ unsigned int *pubc(char *s) { return (unsigned int *)(s + 2 * kMaxStW * 8); }
__device__ __forceinline__ UDescW *udw(char *s) { return (UDescW *)(s + 2 * kMaxStW * 8 + kMaxStW * 4); }

struct StageW {
    char *base;
    int64_t cap;
    // one part per unit: values, window positions, slice geometry, window
    __device__ __forceinline__ double *val(int) const { return (double *)base; }
    __device__ __forceinline__ int32_t *pos(int) const { return (int32_t *)(base + cap * 8); }
    __device__ __forceinline__ int2 *hdr(int) const {
        return (int2 *)(base + cap * 8 + (((cap / kSlice) * 4 + 15) / 16) * 16);
    }
    __device__ __forceinline__ double *win() const {
        return (double *)(base + cap * 8 + (((cap / kSlice) * 4 + 15) / 16) * 16 + kWC * 8);
    }
};
__host__ __device__ inline int64_t stage_bytes_w(int64_t cap, int64_t wcap) {
    return ((cap * 8 + (((cap / kSlice) * 4 + 15) / 16) * 16 + kWC * 8 + wcap * 8) + 127) / 128 * 128;
}
__device__ __forceinline__ StageW stage_w(char *sm, const FwParams &p, int st) {
    return StageW{sm + kHdrW + (int64_t)st * p.stage_bytes, p.cap};
}

// all items < F have their phase-ph unit complete (acquire reads)
__device__ __forceinline__ int64_t frontier(const FwParams &p, int ph, unsigned int epoch, int lane) {
    const int64_t G = gridDim.x;
    int64_t f = INT64_MAX;
    const unsigned long long *pr = p.prog + (int64_t)ph * p.pstride;
    for (int64_t c = lane; c < G; c += 32) {
        const unsigned long long v = ptx::ld_acquire_gpu_u64(pr + c);
        const int64_t cnt = (unsigned int)(v >> 32) == epoch ? (int64_t)(v & 0xffffffffull) : 0;
        f = min(f, c + cnt * G);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) f = min(f, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)f, o));
    return f;
}

// Bulk copy of the 16-byte-aligned part [a, e & ~1) of a window piece (a
// even; the odd last element, if any, is written by the caller before the
// stage's arrival).  Ring sources map row q to ring[q & mask]; a piece never
// crosses the ring end (split by the caller).
__device__ __forceinline__ uint32_t copy_piece(double *wslot, const double *src, int64_t a, int64_t e, uint64_t *bar,
                                               uint64_t pol) {
    if (e <= a) return 0;
    const int64_t be = e & ~(int64_t)1;
    if (be > a) {
        ptx::bulk_g2s(wslot, src, (uint32_t)((be - a) * 8), bar, pol);
        return (uint32_t)((be - a) * 8);
    }
    return 0;
}

template <int CH>
struct WinSum {
    // sum_j val[j] * win[pos[j] + lane] over the slice's entries, in stored
    // order (products of the first CH issued together)
    __device__ __forceinline__ static double run(const double *sv, const int32_t *wp, const double *ws, int w,
                                                 double acc) {
        double v[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) v[j] = __dmul_rn(sv[j * kSlice], ws[wp[j]]);
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) acc = __dadd_rn(acc, v[j]);
        for (int j = CH; j < w; ++j) acc = __dadd_rn(acc, __dmul_rn(sv[j * kSlice], ws[wp[j]]));
        return acc;
    }
};

// Stage one unit (producer warp): slice geometry, window positions, window
// segments (zero-filled outside [0, n), odd last element by a plain load,
// the rest by bulk copies from x or from the ring g(j-1)) and the part's
// values, all counted on the stage's full barrier.
struct UnitMeta {
    int64_t w, u;
    int sidx;
    bool live, valid;
    int64_t pv;                 // lanes 0..8: slice pointers of the unit's part
    int32_t nseg;               // window segments
    int4 seg;                   // lane k: segment k
    int32_t pos[4];             // window positions pos[lane + 32 r]
};
__device__ __forceinline__ int phase_of_unit(int sidx) { return sidx <= 1 ? 0 : sidx - 1; }

__device__ __forceinline__ void load_unit_meta(const FwParams &p, UnitMeta &M, int64_t w, int64_t u, int sidx,
                                               bool live, bool valid, int lane) {
    M.w = w;
    M.u = u;
    M.sidx = sidx;
    M.live = live;
    M.valid = valid;
    M.pv = 0;
    M.nseg = 0;
    if (!valid) return;
    const int64_t s0 = u * kWC, s1 = min(s0 + kWC, p.nslices);
    if (lane <= kWC) M.pv = __ldg((sidx == 1 ? p.U.ptr : p.L.ptr) + min(s0 + lane, s1));
    const bool up = sidx == 1;
    M.nseg = __ldg((up ? p.nsegU : p.nsegL) + u);
    M.seg = __ldg((up ? p.tsegU : p.tsegL) + u * 32 + lane);
    const int32_t *tp = (up ? p.tposU : p.tposL) + u * p.pst;
#pragma unroll
    for (int r = 0; r < 4; ++r) M.pos[r] = lane + 32 * r < p.pst ? __ldg(tp + lane + 32 * r) : 0;
}

__device__ __forceinline__ void stage_unit_w(const FwParams &p, char *sm, int st, const UnitMeta &cur, int K,
                                             int lane, uint64_t pol_first, uint64_t pol_keep) {
    const int sidx = cur.sidx, j = phase_of_unit(sidx);
    const int64_t u = cur.u;
    const int64_t gmask = p.Mg * kRowsW - 1;
    const StageW S = stage_w(sm, p, st);
    const SellView &P = sidx == 1 ? p.U : p.L;
    const int64_t pnext = __shfl_down_sync(0xffffffffu, cur.pv, 1);
    const int64_t b0 = __shfl_sync(0xffffffffu, cur.pv, 0), e0 = __shfl_sync(0xffffffffu, cur.pv, kWC);
    if (lane < kWC) S.hdr(0)[lane] = make_int2((int)(cur.pv - b0), (int)((pnext - cur.pv) / kSlice));
    const int64_t ne = (e0 - b0) / kSlice;
#pragma unroll
    for (int r = 0; r < 4; ++r)
        if (lane + 32 * r < ne) S.pos(0)[lane + 32 * r] = cur.pos[r];
    for (int64_t e = lane + 128; e < ne; e += 32)   // tiles wider than 128 entry positions
        S.pos(0)[e] = __ldg((sidx == 1 ? p.tposU : p.tposL) + u * p.pst + e);
    // window segments: lane k owns segment k
    double *ws = S.win();
    uint64_t *bar = fullb(sm) + st;
    int64_t wa = 0, we = 0, wl0 = 0;
    double *wdst = nullptr;
    const double *vsrc = sidx <= 1 ? p.x : p.ring_g + (int64_t)(j - 1) * p.Mg * kRowsW;
    const bool ring = sidx >= 2;
    if (lane < cur.nseg) {
        const int64_t lo = (int64_t)(((uint64_t)(uint32_t)cur.seg.y << 32) | (uint32_t)cur.seg.x);
        const int64_t hi = lo + cur.seg.z;
        wdst = ws + cur.seg.w;
        wl0 = lo;
        const int64_t a = max(lo, (int64_t)0), e = min(hi, p.n);
        for (int64_t q = lo; q < min(a, hi); ++q) wdst[q - lo] = 0.0;   // below row 0
        for (int64_t q = max(e, lo); q < hi; ++q) wdst[q - lo] = 0.0;  // past row n - 1
        wa = a;
        we = e;
        if (e > a && (e & 1))  // odd n: the last element by a plain load (the only odd end)
            wdst[e - 1 - lo] = __ldcg(vsrc + (ring ? ((e - 1) & gmask) : e - 1));
    }
    // bytes of the bulk copies (matrix values, window pieces)
    const int64_t rl = p.Mg * kRowsW;
    int64_t cut = we;
    uint32_t wbytes = 0;
    if (we > wa) {
        if (!ring) {
            const int64_t be = we & ~(int64_t)1;
            wbytes = be > wa ? (uint32_t)((be - wa) * 8) : 0;
        } else {  // ring pieces: split where the ring wraps
            cut = min(we, (wa / rl + 1) * rl);
            const int64_t be1 = cut & ~(int64_t)1, be2 = we & ~(int64_t)1;
            wbytes = (be1 > wa ? (uint32_t)((be1 - wa) * 8) : 0) + (be2 > cut ? (uint32_t)((be2 - cut) * 8) : 0);
        }
    }
    uint32_t wsum = wbytes;
#pragma unroll
    for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    __syncwarp();
    if (lane == 0) {
        udw(sm)[st] = UDescW{(int)u, sidx};
        ptx::mbar_expect_tx(bar, (uint32_t)((e0 - b0) * 8) + wsum);
        // L's values are re-read by the sweeps: keep them in L2
        if (e0 > b0)
            ptx::bulk_g2s(S.val(0), P.val + b0, (uint32_t)((e0 - b0) * 8), bar,
                          (sidx == 1 || j == K) ? pol_first : pol_keep);
    }
    __syncwarp();
    if (we > wa) {
        if (!ring) {
            copy_piece(wdst + (wa - wl0), vsrc + wa, wa, we, bar, pol_keep);
        } else {
            copy_piece(wdst + (wa - wl0), vsrc + (wa & gmask), wa, cut, bar, pol_keep);
            if (we > cut) copy_piece(wdst + (cut - wl0), vsrc + (cut & gmask), cut, we, bar, pol_keep);
        }
    }
    __syncwarp();
    
}

// Units of an item (s = 0 .. K + 1): s = 0 / 1 = phase 0 over L / U (the
// residual's two triangles, each with its own gather window of x; the row
// sum continues in the consumer's registers from s = 0 to s = 1, so the
// additions keep the stored order L, D, U), s >= 2 = sweep j = s - 1 over L
// with the window of the ring g(j-1).  Every unit stages ONE part and one
// window (~38 KB for C3), so two CTAs fit per SM.
template <int CH>
__global__ void __launch_bounds__(kThreadsW, 2) k_fused_pgs_w(const __grid_constant__ FwParams p) {
    extern __shared__ __align__(128) char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const unsigned int epoch = *(volatile unsigned int *)&p.sync[0];
    if (threadIdx.x == 0) {
        for (int st = 0; st < p.nst; ++st) {
            ptx::mbar_init(fullb(sm) + st, 1);
            ptx::mbar_init(emptyb(sm) + st, kWC);
            pubc(sm)[st] = 0;
        }
        ptx::mbar_init_fence();
    }
    __syncthreads();
    const int K = p.k;
    const int NS = K + 2;                 // units per item
    const int64_t NT = p.ntiles;
    const int64_t rmask = p.Mr * kRowsW - 1, gmask = p.Mg * kRowsW - 1;
    auto phase_of = [](int sidx) { return sidx <= 1 ? 0 : sidx - 1; };

    if (warp == kWC) {
        // ------------------------------------------------------------ producer
        const uint64_t pol_first = ptx::policy_evict_first(), pol_keep = ptx::policy_evict_normal();
        // F[q]: phase q is done for all items < F[q] (acquire reads of the
        // progress counters; a proxy fence orders the following bulk copies).
        // Every phase-advancing unit refreshes one phase's view asynchronously
        // (counter loads issued at the end of one unit, reduced at the end of
        // the next), so the producer rarely waits.
        int64_t F[kMaxPhW];
#pragma unroll
        for (int q = 0; q < kMaxPhW; ++q) F[q] = 0;
        bool proxy_dirty = false;
        int st = 0;
        uint32_t round = 0;
        unsigned long long polls = 0, poll_ns = 0, t_empty = 0, t_need = 0, t_all = 0, n_acq = 0;
        auto need = [&](int ph, int64_t t) {  // phase ph done for every item <= t
            if (t < F[ph]) return;
            const uint64_t t0 = ptx::globaltimer_ns();
            ++polls;
            while (true) {
                F[ph] = max(F[ph], frontier(p, ph, epoch, lane));
                if (t < F[ph]) break;
                if (ptx::globaltimer_ns() - t0 > p.timeout_ns) {
                    if (lane == 0) atomicOr(p.err, 2u);
                    F[ph] = INT64_MAX;
                    break;
                }
                __nanosleep(64);
            }
            proxy_dirty = true;
            poll_ns += ptx::globaltimer_ns() - t0;
        };
        constexpr int kPR = 10;   // counters per lane (grids <= 320 CTAs)
        unsigned long long rv[kPR];
        int rph = -1;
        auto refresh_issue = [&](int ph) {
            rph = ph;
            const unsigned long long *pr = p.prog + (int64_t)ph * p.pstride;
#pragma unroll
            for (int r = 0; r < kPR; ++r) {
                const int64_t cc = lane + 32 * r;
                rv[r] = cc < G ? ptx::ld_acquire_gpu_u64(pr + cc) : 0ull;
            }
        };
        auto refresh_reduce = [&]() {
            if (rph < 0) return;
            int64_t f = INT64_MAX;
#pragma unroll
            for (int r = 0; r < kPR; ++r) {
                const int64_t cc = lane + 32 * r;
                if (cc < G) {
                    const int64_t cnt = (unsigned int)(rv[r] >> 32) == epoch ? (int64_t)(rv[r] & 0xffffffffull) : 0;
                    f = min(f, cc + cnt * G);
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) f = min(f, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)f, o));
            if (f > F[rph]) {
                F[rph] = f;
                proxy_dirty = true;
            }
            rph = -1;
        };
        // unit metadata, loaded one unit ahead (two dependent round trips:
        // slice pointers / segment range, then positions / segments)
        auto load1 = [&](UnitMeta &M, int64_t w, int sidx) {
            const bool live = w < p.nitems;
            const int64_t u = w - (int64_t)phase_of(sidx) * p.D;
            load_unit_meta(p, M, w, u, sidx, live, live && u >= 0 && u < NT && !(sidx <= 1 && p.fresh), lane);
        };
        UnitMeta ma, mb;
        int64_t wn = c;
        int sn = 0;
        auto advance = [&]() {
            if (++sn == NS) { sn = 0; wn += G; }
        };
        load1(ma, wn, sn);
        advance();
        // one unit; the two Meta records alternate roles (no register copy,
        // so the next unit's loads overlap this unit's staging)
        auto step = [&](UnitMeta &cur, UnitMeta &nxt) -> bool {
            if (!cur.live) return false;
            load1(nxt, wn, sn);   // the next unit's metadata
            advance();
            const int sidx = cur.sidx, j = phase_of(sidx);
            const int64_t w = cur.w, u = cur.u;
            const uint64_t tA = ptx::globaltimer_ns();
            if (round > 0) ptx::mbar_wait(emptyb(sm) + st, (round - 1) & 1);
            const uint64_t tB = ptx::globaltimer_ns();
            t_empty += tB - tA;
            if (!cur.valid) {
                if (lane == 0) {
                    udw(sm)[st] = UDescW{-1, sidx};
                    ptx::mbar_arrive(fullb(sm) + st);
                }
                __syncwarp();
            } else {
                if (j >= 1) need(j - 1, w - p.D);
                if (j == K) need(0, u + p.DA);
                if (sidx <= 1 && u >= p.Mr) need(K, u - p.Mr + (int64_t)K * p.D);
                if (sidx != 1 && j < K && u >= p.Mg) need(j + 1, u - p.Mg + p.DT + (int64_t)(j + 1) * p.D);
                if (proxy_dirty) {  // the bulk copies below read what the new frontiers published
                    __syncwarp();
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    proxy_dirty = false;
                    ++n_acq;
                }
                const uint64_t tC = ptx::globaltimer_ns();
                t_need += tC - tB;
                stage_unit_w(p, sm, st, cur, K, lane, pol_first, pol_keep);
            }
            if (sidx != 0) {  // units that complete a phase refresh that phase's view
                refresh_reduce();
                refresh_issue(j);
            }
            t_all += ptx::globaltimer_ns() - tA;
            if (++st == p.nst) { st = 0; ++round; }
            return true;
        };
        while (step(ma, mb) && step(mb, ma)) {
        }
        // end of the sequence
        if (round > 0) ptx::mbar_wait(emptyb(sm) + st, (round - 1) & 1);
        if (lane == 0) {
            udw(sm)[st] = UDescW{-2, 0};
            ptx::mbar_arrive(fullb(sm) + st);
            // statistics (nsm_fused_counters)
            atomicAdd((unsigned long long *)(p.sync + 4), polls);
            atomicAdd((unsigned long long *)(p.sync + 6), poll_ns);
            atomicAdd((unsigned long long *)(p.sync + 8), t_empty);
            atomicAdd((unsigned long long *)(p.sync + 10), t_need);
            atomicAdd((unsigned long long *)(p.sync + 12), t_all);
            atomicAdd((unsigned long long *)(p.sync + 14), n_acq);
        }
    } else {
        // ----------------------------------------------------------- consumers
        int st = 0;
        uint32_t par = 0;
        double acc = 0.0, di = 1.0, bi = 0.0, xi = 0.0;   // carried from unit s = 0 to s = 1
        for (int64_t w = c, m = 0;; w += G, ++m) {
            bool end = false;
            for (int sidx = 0; sidx < NS; ++sidx) {
                const int j = phase_of(sidx);
                const int64_t u = w - (int64_t)j * p.D;
                const bool valid = w < p.nitems && u >= 0 && u < NT;
                const int64_t i = u * kRowsW + warp * kSlice + lane;
                const bool row = valid && i < p.n;
                // own-row vectors: immutable (d, b), or written only by this unit (x of tile u, j = K)
                if (sidx != 1) {
                    di = 1.0;
                    bi = 0.0;
                    xi = 0.0;
                    if (row) {
                        di = __ldg(p.d + i);
                        if (j == 0) {
                            bi = __ldg(p.b + i);
                            if (!p.fresh) xi = __ldg(p.x + i);
                        } else if (j == K && !p.fresh) {
                            xi = p.x[i];
                        }
                    }
                }
                ptx::mbar_wait(fullb(sm) + st, par);
                const UDescW un = udw(sm)[st];
                if (un.u == -2) { end = true; break; }
                double res = 0.0;
                if (un.u >= 0 && row) {
                    const StageW S = stage_w(sm, p, st);
                    const int2 h = S.hdr(0)[warp];
                    const double *ws = S.win() + lane;
                    if (sidx == 0) {
                        acc = WinSum<CH>::run(S.val(0) + h.x + lane, S.pos(0) + h.x / kSlice, ws, h.y, 0.0);
                    } else if (sidx == 1) {
                        acc = __dadd_rn(acc, __dmul_rn(di, xi));
                        acc = WinSum<CH>::run(S.val(0) + h.x + lane, S.pos(0) + h.x / kSlice, ws, h.y, acc);
                    } else {
                        res = WinSum<CH>::run(S.val(0) + h.x + lane, S.pos(0) + h.x / kSlice, ws, h.y, 0.0);
                    }
                }
                if (row) {
                    if (sidx == 1) {
                        const double r = p.fresh ? bi : __dsub_rn(bi, acc);   // x = 0: r = b (reading R3)
                        p.ring_r[i & rmask] = r;
                        p.ring_g[i & gmask] = __ddiv_rn(r, di);   // g(0) = D^{-1} r
                    } else if (sidx >= 2) {
                        const double ri = __ldcg(p.ring_r + (i & rmask));
                        const double v = __ddiv_rn(__dsub_rn(ri, res), di);
                        if (!isfinite(v)) atomicMin(p.flag, (unsigned long long)(p.sweep_id0 + j - 1));
                        if (j < K) p.ring_g[(int64_t)j * p.Mg * kRowsW + (i & gmask)] = v;
                        else p.x[i] = p.fresh ? v : __dadd_rn(xi, v);
                    }
                }
                // publish "phase j of this CTA's items <= m is complete" (units
                // s >= 1): the last warp to finish the unit (CTA-scope acq_rel
                // count, then a gpu-scope release); the stage is released
                // after the count, so no warp reaches the stage's next unit
                // before every warp has counted this one
                __syncwarp();
                if (lane == 0) {
                    const unsigned int prev = ptx::atom_add_acqrel_cta_shared(pubc(sm) + st, 1u);
                    if (sidx != 0 && (prev + 1) % kWC == 0)
                        ptx::red_max_release_gpu_u64(p.prog + (int64_t)j * p.pstride + c,
                                                     ((unsigned long long)epoch << 32) | (unsigned long long)(m + 1));
                    ptx::mbar_arrive(emptyb(sm) + st);
                }
                if (++st == p.nst) { st = 0; par ^= 1; }
            }
            if (end) break;
        }
    }
    // ---- the last CTA out advances the epoch for the next launch
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(&p.sync[1], 1u);
        if (prev == gridDim.x - 1) {
            p.sync[1] = 0;
            p.sync[0] = epoch + 1 == 0 ? 1 : epoch + 1;
            __threadfence();
        }
    }
}


// ---------------------------------------------------------------------------
// Plane wavefront (structured grids: rows in planes of tpp tiles, every
// coupling of a tile's rows within the tiles of the lines c-2 .. c+2 (tile
// index mod tpp) of the same and the two neighbouring planes — lexicographic
// 7- / 27-point stencils with 256-row grid lines; checked on the host).  CTA
// c owns line c of every plane.  Step s: phase 0 on plane s (units L, U),
// phase j on plane s - j.  Every dependency of step s lies in step s - 1 of
// CTAs c-2 .. c+2, so readiness is a wait on at most five step counters
// (neighbours stay within one step of each other); with k >= 2 the x update
// of plane s - k never meets a residual of plane >= s - 1 that reads it.
template <int CH>
__global__ void __launch_bounds__(kThreadsW, 2) k_fused_pgs_planes(const __grid_constant__ FwParams p) {
    extern __shared__ __align__(128) char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const unsigned int epoch = *(volatile unsigned int *)&p.sync[0];
    if (threadIdx.x == 0) {
        for (int st = 0; st < p.nst; ++st) {
            ptx::mbar_init(fullb(sm) + st, 1);
            ptx::mbar_init(emptyb(sm) + st, kWC);
            pubc(sm)[st] = 0;
        }
        ptx::mbar_init_fence();
    }
    __syncthreads();
    const int K = p.k;
    const int NS = K + 2;                 // units per step
    const int64_t NT = p.ntiles, NP = p.nplanes, nsteps = NP + K;
    const int64_t rmask = p.Mr * kRowsW - 1, gmask = p.Mg * kRowsW - 1;
    auto tile_of = [&](int64_t step, int sidx, int64_t &u) -> bool {
        const int64_t plane = step - phase_of_unit(sidx);
        u = plane * p.tpp + c;
        return plane >= 0 && plane < NP && u < NT;
    };

    if (warp == kWC) {
        // ------------------------------------------------------------ producer
        const uint64_t pol_first = ptx::policy_evict_first(), pol_keep = ptx::policy_evict_normal();
        int st = 0;
        uint32_t round = 0;
        int64_t ready[kMaxPhW];   // CTAs c-2 .. c+2 have completed phase q of every step < ready[q]
#pragma unroll
        for (int q = 0; q < kMaxPhW; ++q) ready[q] = 0;
        unsigned long long polls = 0, poll_ns = 0, t_empty = 0, t_need = 0, t_all = 0, n_acq = 0;
        auto wait_phase = [&](int ph, int64_t s) {  // neighbours (and this CTA) completed phase ph of step s - 1
            if (s <= ready[ph]) return;
            const uint64_t t0 = ptx::globaltimer_ns();
            ++polls;
            while (true) {
                int64_t mn = INT64_MAX;
                if (lane < 5) {
                    const int64_t cc = c + lane - 2;
                    if (cc >= 0 && cc < G) {
                        const unsigned long long v = ptx::ld_acquire_gpu_u64(p.prog + (int64_t)ph * p.pstride + cc);
                        mn = (unsigned int)(v >> 32) == epoch ? (int64_t)(v & 0xffffffffull) : 0;
                    }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) mn = min(mn, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mn, o));
                if (mn >= s) {
                    ready[ph] = mn;
                    break;
                }
                if (ptx::globaltimer_ns() - t0 > p.timeout_ns) {
                    if (lane == 0) atomicOr(p.err, 2u);
                    ready[ph] = INT64_MAX;
                    break;
                }
                __nanosleep(32);
            }
            __syncwarp();
            asm volatile("fence.proxy.async.global;" ::: "memory");  // order the ring's bulk copies after it
            ++n_acq;
            poll_ns += ptx::globaltimer_ns() - t0;
        };
        auto load1 = [&](UnitMeta &M, int64_t sstep, int sidx) {
            int64_t u = 0;
            const bool live = sstep < nsteps;
            const bool in = live && tile_of(sstep, sidx, u);
            load_unit_meta(p, M, sstep, u, sidx, live, in && !(sidx <= 1 && p.fresh), lane);
        };
        UnitMeta ma, mb;
        int64_t sn_step = 0;
        int sn = 0;
        auto advance = [&]() {
            if (++sn == NS) { sn = 0; ++sn_step; }
        };
        load1(ma, sn_step, sn);
        advance();
        auto step = [&](UnitMeta &cur, UnitMeta &nxt) -> bool {
            if (!cur.live) return false;
            load1(nxt, sn_step, sn);
            advance();
            const int sidx = cur.sidx;
            const uint64_t tA = ptx::globaltimer_ns();
            if (round > 0) ptx::mbar_wait(emptyb(sm) + st, (round - 1) & 1);
            const uint64_t tB = ptx::globaltimer_ns();
            t_empty += tB - tA;
            if (!cur.valid) {
                if (lane == 0) {
                    udw(sm)[st] = UDescW{-1, sidx};
                    ptx::mbar_arrive(fullb(sm) + st);
                }
                __syncwarp();
            } else {
#ifndef NSM_FW_NOWAIT   // timing experiment only: readiness skipped (results wrong)
                if (sidx >= 2) wait_phase(sidx - 2, cur.w);   // phase j reads phase j - 1 of step w - 1
#endif
                t_need += ptx::globaltimer_ns() - tB;
                stage_unit_w(p, sm, st, cur, K, lane, pol_first, pol_keep);
            }
            t_all += ptx::globaltimer_ns() - tA;
            if (++st == p.nst) { st = 0; ++round; }
            return true;
        };
        while (step(ma, mb) && step(mb, ma)) {
        }
        if (round > 0) ptx::mbar_wait(emptyb(sm) + st, (round - 1) & 1);
        if (lane == 0) {
            udw(sm)[st] = UDescW{-2, 0};
            ptx::mbar_arrive(fullb(sm) + st);
            atomicAdd((unsigned long long *)(p.sync + 4), polls);
            atomicAdd((unsigned long long *)(p.sync + 6), poll_ns);
            atomicAdd((unsigned long long *)(p.sync + 8), t_empty);
            atomicAdd((unsigned long long *)(p.sync + 10), t_need);
            atomicAdd((unsigned long long *)(p.sync + 12), t_all);
            atomicAdd((unsigned long long *)(p.sync + 14), n_acq);
        }
    } else {
        // ----------------------------------------------------------- consumers
        int st = 0;
        uint32_t par = 0;
        double acc = 0.0, di = 1.0, bi = 0.0, xi = 0.0;   // carried from unit s = 0 to s = 1
        for (int64_t sstep = 0;; ++sstep) {
            bool end = false;
            for (int sidx = 0; sidx < NS; ++sidx) {
                const int j = phase_of_unit(sidx);
                int64_t u = 0;
                const bool valid = sstep < nsteps && tile_of(sstep, sidx, u);
                const int64_t i = u * kRowsW + warp * kSlice + lane;
                const bool row = valid && i < p.n;
                if (sidx != 1) {
                    di = 1.0;
                    bi = 0.0;
                    xi = 0.0;
                    if (row) {
                        di = __ldg(p.d + i);
                        if (j == 0) {
                            bi = __ldg(p.b + i);
                            if (!p.fresh) xi = __ldg(p.x + i);
                        } else if (j == K && !p.fresh) {
                            xi = p.x[i];
                        }
                    }
                }
                ptx::mbar_wait(fullb(sm) + st, par);
                const UDescW un = udw(sm)[st];
                if (un.u == -2) { end = true; break; }
                double res = 0.0;
                if (un.u >= 0 && row) {
                    const StageW S = stage_w(sm, p, st);
                    const int2 h = S.hdr(0)[warp];
                    const double *ws = S.win() + lane;
                    if (sidx == 0) {
                        acc = WinSum<CH>::run(S.val(0) + h.x + lane, S.pos(0) + h.x / kSlice, ws, h.y, 0.0);
                    } else if (sidx == 1) {
                        acc = __dadd_rn(acc, __dmul_rn(di, xi));
                        acc = WinSum<CH>::run(S.val(0) + h.x + lane, S.pos(0) + h.x / kSlice, ws, h.y, acc);
                    } else {
                        res = WinSum<CH>::run(S.val(0) + h.x + lane, S.pos(0) + h.x / kSlice, ws, h.y, 0.0);
                    }
                }
                if (row) {
                    if (sidx == 1) {
                        const double r = p.fresh ? bi : __dsub_rn(bi, acc);   // x = 0: r = b (reading R3)
                        p.ring_r[i & rmask] = r;
                        p.ring_g[i & gmask] = __ddiv_rn(r, di);   // g(0) = D^{-1} r
                    } else if (sidx >= 2) {
                        const double ri = __ldcg(p.ring_r + (i & rmask));
                        const double v = __ddiv_rn(__dsub_rn(ri, res), di);
                        if (!isfinite(v)) atomicMin(p.flag, (unsigned long long)(p.sweep_id0 + j - 1));
                        if (j < K) p.ring_g[(int64_t)j * p.Mg * kRowsW + (i & gmask)] = v;
                        else p.x[i] = p.fresh ? v : __dadd_rn(xi, v);
                    }
                }
                // the last warp to finish a phase's unit publishes "phase j of
                // steps <= sstep complete" (CTA-scope acq_rel count, gpu-scope release)
                __syncwarp();
                if (lane == 0) {
                    const unsigned int prev = ptx::atom_add_acqrel_cta_shared(pubc(sm) + st, 1u);
                    if (sidx != 0 && (prev + 1) % kWC == 0)
                        ptx::red_max_release_gpu_u64(p.prog + (int64_t)j * p.pstride + c,
                                                     ((unsigned long long)epoch << 32) | (unsigned long long)(sstep + 1));
                    ptx::mbar_arrive(emptyb(sm) + st);
                }
                if (++st == p.nst) { st = 0; par ^= 1; }
            }
            if (end) break;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(&p.sync[1], 1u);
        if (prev == gridDim.x - 1) {
            p.sync[1] = 0;
            p.sync[0] = epoch + 1 == 0 ? 1 : epoch + 1;
            __threadfence();
        }
    }
}

// Plane-structure check of a part for the plane wavefront: every stored
// entry with a nonzero value (pads and explicit zeros multiply whatever they
// gather by 0: any finite value gives the same sum) couples tile (plane pl,
// line c) to a tile within two lines in the same or a neighbouring plane
// (upper: not below pl - 1; lower: not above pl).
__global__ void k_plane_check(int64_t n, int64_t nslices, int64_t tpp, const int64_t *__restrict__ ptr,
                              const int32_t *__restrict__ col, const double *__restrict__ val, int upper,
                              unsigned int *bad) {
    const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= nslices) return;
    const int64_t i = s * kSlice + lane;
    if (i >= n) return;
    const int64_t t = i / kRowsW, pl = t / tpp, c = t % tpp;
    const int64_t w = (ptr[s + 1] - ptr[s]) / kSlice;
    for (int64_t j = 0; j < w; ++j) {
        const int64_t e = ptr[s] + j * kSlice + lane;
        if (val[e] == 0.0) continue;
        const int64_t tq = col[e] / kRowsW, pq = tq / tpp, cq = tq % tpp;
        if (cq < c - 2 || cq > c + 2 || pq < pl - 1 || pq > pl + (upper ? 1 : 0)) atomicOr(bad, 1u);
    }
}

// Per-tile padded window tables (one warp per tile): positions, segment
// count and segments of window W, for the one-pass kernel's independent loads.
__global__ void k_fw_tables(int64_t ntiles, int64_t nslices, const int64_t *__restrict__ ptr, WinView W, int pst,
                            int32_t *__restrict__ tpos, int32_t *__restrict__ nseg, int4 *__restrict__ tseg) {
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= ntiles) return;
    const int64_t s0 = t * kWC, s1 = min(s0 + kWC, nslices);
    const int64_t b = ptr[s0] / kSlice, e = ptr[s1] / kSlice;
    for (int64_t k = lane; k < pst; k += 32) tpos[t * pst + k] = k < e - b ? W.wpos[0][b + k] : 0;
    const int32_t g0 = W.tseg[t], g1 = W.tseg[t + 1];
    if (lane == 0) nseg[t] = g1 - g0;
    int4 v = make_int4(0, 0, 0, 0);
    if (lane < g1 - g0) {
        const int64_t lo = W.glo[g0 + lane];
        v = make_int4((int)(uint32_t)(uint64_t)lo, (int)(uint32_t)((uint64_t)lo >> 32), W.len[g0 + lane], W.sbase[g0 + lane]);
    }
    tseg[t * 32 + lane] = v;
}

const void *pick_w(int ch, bool planes) {
    if (planes)
        return ch <= 4 ? (const void *)k_fused_pgs_planes<4>
                       : (ch <= 8 ? (const void *)k_fused_pgs_planes<8> : (const void *)k_fused_pgs_planes<16>);
    return ch <= 4 ? (const void *)k_fused_pgs_w<4> : (ch <= 8 ? (const void *)k_fused_pgs_w<8> : (const void *)k_fused_pgs_w<16>);
}

int sm_count_w() {
    static int nsm[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!nsm[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        nsm[dev] = v > 0 ? v : 148;
    }
    return nsm[dev];
}

struct GeoW {
    int nst = 0, per_sm = 0;
    size_t smem = 0;
};

// stages: maximise co-resident CTAs (<= 2 by the launch bounds), then depth
GeoW geometry_w(const void *k, int64_t stage_bytes) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, int64_t>, GeoW> cache;
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    auto key = std::make_tuple(dev, k, stage_bytes);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMaxW);
    GeoW g;
    int best = -1;
    for (int nst = 2; nst <= kMaxStW; ++nst) {
        const int64_t smem = kHdrW + nst * stage_bytes;
        if (smem > kSmemMaxW) break;
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kThreadsW, (size_t)smem);
        per = std::min(per, 2);
        if (per > 0 && per >= best) {
            best = per;
            g.nst = nst;
            g.per_sm = per;
            g.smem = (size_t)smem;
        }
    }
    cache[key] = g;
    return g;
}

int64_t pow2_ge(int64_t v) {
    int64_t q = 1;
    while (q < v) q <<= 1;
    return q;
}

}  // namespace

FusedWShape fused_w_shape(int maxw, int64_t wmax, int k, int64_t n, int DT, int DA, int d_extra, int64_t tpp) {
    FusedWShape sh;
    if (k < 1 || k > kMaxPhW - 1 || n <= 0) return sh;
    const bool planes = tpp > 0;
    if (planes && k < 2) return sh;  // the plane schedule needs k >= 2 (the x update two planes back)
    const int ch = maxw <= 4 ? 4 : (maxw <= 8 ? 8 : 16);
    const void *kern = pick_w(ch, planes);
    const int64_t cap = (int64_t)kRowsW * std::max(maxw, 1);
    const int64_t wcap = (wmax + 31) / 32 * 32;
    const int64_t sbytes = stage_bytes_w(cap, wcap);
    const GeoW g = geometry_w(kern, sbytes);
    if (!g.nst) return sh;
    sh.kernel = kern;
    sh.nst = g.nst;
    sh.smem = g.smem;
    sh.cap = cap;
    sh.wcap = wcap;
    sh.stage_bytes = sbytes;
    sh.ntiles = (n + kRowsW - 1) / kRowsW;
    const int64_t tp2 = pow2_ge(sh.ntiles);
    if (planes) {
        // one CTA per line of a plane, all co-resident
        if (tpp > (int64_t)sm_count_w() * g.per_sm) return sh;
        sh.grid = (int)tpp;
        sh.tpp = tpp;
        sh.nplanes = (sh.ntiles + tpp - 1) / tpp;
        sh.D = 0;
        sh.nitems = sh.nplanes + k;
        // rings: k + 2 planes (r is read k steps after it was written, an
        // iterate up to two; a slot is rewritten k + 2 steps later, and
        // neighbours stay within one step of each other)
        sh.Mr = sh.Mg = std::min(pow2_ge((int64_t)(k + 2) * tpp), tp2);
        sh.ok = true;
        return sh;
    }
    sh.grid = (int)std::min<int64_t>((int64_t)sm_count_w() * g.per_sm, std::max<int64_t>(sh.ntiles, 1));
    // skew: above the bandwidth, and (automatic) above one grid of items, so a
    // unit's dependencies were processed in an earlier round
    sh.D = std::max(DT, DA) + (d_extra > 0 ? d_extra : std::max(16, sh.grid + 32 - std::max(DT, DA)));
    sh.nitems = sh.ntiles + (int64_t)k * sh.D;
    // rings (tiles): every slot's previous occupant is at least two grids of
    // items older than the reuse conditions require
    sh.Mr = std::min(pow2_ge((int64_t)k * sh.D + 2 * sh.grid + 1), tp2);
    sh.Mg = std::min(pow2_ge((int64_t)sh.D + DT + 2 * sh.grid + 1), tp2);
    sh.ok = true;
    return sh;
}

cudaError_t launch_fused_w(const FusedWLaunch &L, cudaStream_t st) {
    const FusedWShape &sh = L.shape;
    if (!sh.ok) return cudaErrorInvalidConfiguration;
    FwParams p{};
    p.n = L.n;
    p.nslices = (L.n + kSlice - 1) / kSlice;
    p.ntiles = sh.ntiles;
    p.nitems = sh.nitems;
    p.k = L.k;
    p.D = sh.D;
    p.DT = L.DT;
    p.DA = L.DA;
    p.fresh = L.fresh;
    p.Mr = sh.Mr;
    p.Mg = sh.Mg;
    p.L = view(*L.Lp);
    p.U = view(*L.Up);
    auto wv = [&](const Window *w) {
        return WinView{w->tseg, w->glo, w->len, w->sbase, {w->wpos[0], w->wpos[1]}, (int32_t)sh.wcap};
    };
    p.WR = wv(L.wu);
    p.tposL = L.tposL;
    p.tposU = L.tposU;
    p.nsegL = L.nsegL;
    p.nsegU = L.nsegU;
    p.tsegL = L.tsegL;
    p.tsegU = L.tsegU;
    p.pst = L.pst;
    p.tpp = sh.tpp;
    p.nplanes = sh.nplanes;
    p.WL = wv(L.wl);
    p.d = L.d;
    p.b = L.b;
    p.x = L.x;
    p.ring_r = L.ring_r;
    p.ring_g = L.ring_g;
    p.prog = L.prog;
    p.pstride = L.pstride;
    p.flag = L.flag;
    p.sweep_id0 = L.sweep_id0;
    p.err = L.err;
    p.timeout_ns = L.timeout_ns;
    p.sync = L.sync;
    p.nst = sh.nst;
    p.cap = sh.cap;
    p.wcap = sh.wcap;
    p.stage_bytes = sh.stage_bytes;
    void *args[] = {&p};
    return cudaLaunchCooperativeKernel(sh.kernel, dim3((unsigned)sh.grid), dim3(kThreadsW), args, sh.smem, st);
}

cudaError_t fused_w_tables(int64_t n, const Sell &T, const Window &w, int pst, int32_t *tpos, int32_t *nseg,
                           int4 *tseg) {
    const int64_t nt = (n + kRowsW - 1) / kRowsW, ns = (n + kSlice - 1) / kSlice;
    const WinView W{w.tseg, w.glo, w.len, w.sbase, {w.wpos[0], w.wpos[1]}, 0};
    k_fw_tables<<<(unsigned)((nt * 32 + 255) / 256), 256>>>(nt, ns, T.ptr, W, pst, tpos, nseg, tseg);
    const cudaError_t e = cudaGetLastError();
    return e != cudaSuccess ? e : cudaDeviceSynchronize();
}

bool fused_w_plane_check(int64_t n, int64_t tpp, const Sell &L, const Sell &U) {
    const int64_t ns = (n + kSlice - 1) / kSlice;
    unsigned int *bad = nullptr, hb = 0;
    if (cudaMalloc(&bad, sizeof(unsigned int)) != cudaSuccess) return false;
    bool ok = cudaMemset(bad, 0, sizeof(unsigned int)) == cudaSuccess;
    for (int part = 0; ok && part < 2; ++part) {
        const Sell &T = part == 0 ? L : U;
        if (T.padded == 0) continue;
        k_plane_check<<<(unsigned)((ns * 32 + 255) / 256), 256>>>(n, ns, tpp, T.ptr, T.col, T.val, part, bad);
    }
    ok = ok && cudaGetLastError() == cudaSuccess &&
         cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost) == cudaSuccess && hb == 0;
    cudaFree(bad);
    return ok;
}

void preload_fused_w_kernels() {
    cudaFuncAttributes a;
    for (int ch : {4, 8, 16})
        for (bool planes : {false, true}) cudaFuncGetAttributes(&a, pick_w(ch, planes));
    cudaFuncGetAttributes(&a, k_plane_check);
    cudaFuncGetAttributes(&a, k_fw_tables);
}

}  // namespace nsm
