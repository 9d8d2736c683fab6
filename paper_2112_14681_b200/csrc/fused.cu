// fused.cu — phase-skewed fused smoother passes (DESIGN.md §6 "Fused
// phase-skewed passes"; SURVEY.md §7.3, §8(d) "fused floor").
//
// One launch computes a whole Jacobi-iterated triangular solve together with
// the residual that feeds it, reading every matrix entry from HBM once:
//
//   pGS:   r = b - A x,  g(0) = D^{-1} r,
//                       g(j) = D^{-1}(r - L g(j-1))  j = 1..k,   x += g(k)
//   ILU pass 1 (Alg. 2, eq:LUiterMat P:L826-828):
//                       r = b - A x,  y(0) = r,  y(j) = r - L_s y(j-1),
//                       then y and z(0) = D_U^{-1} y are stored
//   ILU pass 2 (LDU form P:L858-866, walked top-down):
//                       z(j) = D_U^{-1}(y - U_s z(j-1)),   x += z(k)
//
// (backward pGS, is pGS with U and a top-down walk).
//
// Schedule.  Rows are cut into tiles of 256 (8 SELL-32 slices).  Phase j of
// tile u needs phase j-1 of tiles [u - DT, u] (DT: the triangle's bandwidth
// in tiles), so a plain wavefront serialises the phases of each tile.
// Instead, WORK ITEM w bundles phase j0 of tile w, phase j0+1 of tile w-D,
// ..., phase k of tile w-(k-j0)D: every dependency of item w lies in items
// [w - D - DT, w - D], at least D - DT = Dw items back.  Items are dealt
// round-robin to a cooperative (co-resident) grid, item w to CTA w mod G,
// and each CTA runs its items in order.  Before item w starts, all items
// <= w - Dw must be done (one condition per item, tracked by per-item done
// flags and a shared watermark); with Dw above the grid size it is almost
// always already true.  The iterates g(j) of the last few thousand tiles
// live in L2-resident ring buffers indexed by (row & mask); the triangle
// slices a later phase re-reads are fetched with an L2 evict_normal policy,
// the rest evict_first, so HBM sees the matrix about once.
//
// Warp roles (one CTA = 8 consumer warps + producer warp + sync warp):
//   producer  stages, per unit, the tile's matrix slices, the per-slice
//             offsets and the tile's immutable vector segments (d, b, x, ...)
//             HBM/L2 -> shared memory with cp.async.bulk (mbarrier pipeline);
//   sync      runs one item ahead of the consumers: waits for "items <= w -
//             Dw done" and signals a shared-memory barrier; when the
//             consumers finish an item it publishes the item's done flag
//             (fence + st.release);
//   consumers one slice per warp, one row per thread: no global
//             synchronisation on their path.
//
// Ring and in-place-x safety (all with the single wait "items <= w-Dw done"):
//   * g(j) slot of tile u is reused by tile u+Mg: its last reader is item
//     u + DT + (j+1-j0)D  <=  w - Dw   when Mg >= D + DT + Dw;
//   * r slot: last reader item u + (k-j0)D  <=  w - Dw  when Mr >= kD + Dw;
//   * x of tile u is overwritten by item u + kD, after every residual that
//     reads it (tiles up to u + DA, DA = A's bandwidth) when kD - DA >= Dw.
// D = Dw + max(DT, DA) satisfies all three for k >= 1.
//
// Deadlock freedom: all CTAs are co-resident (cooperative launch); an item
// depends only on items at least Dw lower; a sync warp waits for item w +
// G's condition only after publishing item w, and G < Dw, so the lowest
// unpublished item always makes progress.  Waits are bounded
// (NSM_OPT_HALO_TIMEOUT_MS) and flag an error instead of hanging.  The
// launch state (watermark, epoch of the done flags) is reset by the last CTA
// to leave, so launches are self-contained and may be captured into graphs.
//
// Arithmetic: every row sum uses the operations and order of the per-pass
// kernels (and of the oracle): results are bit-identical.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <map>
#include <tuple>
#include <mutex>
#include <utility>

#include "nsm_internal.h"
#include "ptx.cuh"

namespace nsm {

namespace {

constexpr int kWarpsC = 8;                  // consumer warps
constexpr int kRPT = 1;                     // rows per consumer thread (2 measured slower: spills)
constexpr int kTSF = kWarpsC * kRPT;        // slices per tile
constexpr int kRowsF = kTSF * kSlice;       // 256 rows per tile
constexpr int kWarpP = kWarpsC, kWarpS = kWarpsC + 1;
constexpr int kThreadsF = (kWarpsC + 2) * 32;  // + producer warp + sync warp
constexpr int kMaxStages = 8;
constexpr int kSlots = 4;                   // item slots of the ready / done barriers
constexpr int kNVec = 4;                    // vector segments staged per unit
constexpr int kHeader = 384 + kMaxStages * 2 * kTSF * 8;  // barriers, unit descriptors, per-stage slice offsets
constexpr int64_t kSmemMaxF = 220 * 1024;
constexpr int64_t kVecBytes = (int64_t)kRowsF * 8;

struct SkewParams {
    int64_t n, nslices, ntiles, nitems;
    int64_t nbig;             // scheduling tiles of B x 256 rows (items, D, rings count these)
    int B;
    int desc;                 // walk tiles top-down (logical tile u = physical ntiles-1-u)
    int k, j0, D, Dw;         // sweeps; first phase (0: residual, 1: none); skew; wait distance
    int epi, scaled_g0, vec_bulk;
    SellView A0, A1;          // phase 0: residual parts (strict lower, strict upper of A)
    SellView T;               // swept triangle
    const double *dA, *b, *xin;
    const double *dT, *rhs, *g0;
    double *x, *out1, *out2;
    const double *dn;
    double *ring_r, *ring_g;
    int64_t rmask, gmask, gstride;
    unsigned long long *flag;
    int64_t sweep_id0;
    unsigned int *err;
    unsigned long long timeout_ns;
    SkewSync *sync;
    unsigned long long *prog;   // per-CTA progress counters
    int nst, keep0, keep1;
    int64_t cap0, cap1, stage_bytes;
    unsigned long long *trace;  // debug (NSM_DEBUG_SKEW_TRACE): per-unit timestamps of two CTAs
};
constexpr int kTraceUnits = 2048;
__device__ __forceinline__ void trace_at(const SkewParams &p, int role, int unit, int slot) {
    if (!p.trace || unit >= kTraceUnits) return;
    const int cta = blockIdx.x == 0 ? 0 : (blockIdx.x == gridDim.x / 2 ? 1 : -1);
    if (cta < 0) return;
    p.trace[((cta * 3 + role) * kTraceUnits + unit) * 4 + slot] = ptx::globaltimer_ns();
}

// shared memory: [full x8][empty x8][ready x4][idone x4] ... [slice offsets][stages]
__device__ __forceinline__ uint64_t *full_bar(char *s) { return (uint64_t *)s; }
__device__ __forceinline__ uint64_t *empty_bar(char *s) { return (uint64_t *)s + kMaxStages; }
__device__ __forceinline__ uint64_t *ready_bar(char *s) { return (uint64_t *)s + 2 * kMaxStages; }
__device__ __forceinline__ uint64_t *idone_bar(char *s) { return (uint64_t *)s + 2 * kMaxStages + kSlots; }
__device__ __forceinline__ unsigned int *pubcnt(char *s) { return (unsigned int *)((uint64_t *)s + 2 * kMaxStages + 2 * kSlots); }
// {offset within the stage's part, width} of slice `sl` of part `pt` in stage `st`
__device__ __forceinline__ int2 *slice_info(char *s, int st, int pt) {
    return (int2 *)(s + 384) + (st * 2 + pt) * kTSF;
}
// per-stage unit descriptor written by the producer: physical 256-row tile
// (-1: an item without units), phase, flags
enum { U_FIRST = 1, U_LAST = 2, U_END = 4 };
struct UDesc {
    int tp;
    short j, flags;
};
__device__ __forceinline__ UDesc *udesc(char *s) { return (UDesc *)(s + 256); }
__device__ __forceinline__ char *stage_ptr(char *s, const SkewParams &p, int st) {
    return s + kHeader + (int64_t)st * p.stage_bytes;
}

// Which vector segments a unit stages (slot order): phase 0: dA, b, xin;
// phase j >= 1: dT (non-unit), rhs (given vector), x (last, x-update
// epilogue), dn (last, scaling epilogue).
struct VecSet {
    const double *v[kNVec];
    int n;
};
template <int PH0, bool UNIT>
__device__ __forceinline__ VecSet unit_vectors(const SkewParams &p, int j) {
    VecSet vs{};
    if (PH0 == SKEW_RESID && j == 0) {
        vs.v[0] = p.dA; vs.v[1] = p.b; vs.v[2] = p.xin; vs.n = 3;
        return vs;
    }
    const bool last = j == p.k;
    int n = 0;
    if (!UNIT) vs.v[n++] = p.dT;
    if (PH0 != SKEW_RESID) vs.v[n++] = p.rhs;
    if (last && (p.epi == SKEW_XADD || p.epi == SKEW_XADD_SCALE)) vs.v[n++] = p.x;
    if (last && (p.epi == SKEW_STORE2 || p.epi == SKEW_XADD_SCALE || p.epi == SKEW_STORE_SCALE)) vs.v[n++] = p.dn;
    vs.n = n;
    return vs;
}

struct GFull {
    const double *__restrict__ g;
    __device__ __forceinline__ double operator()(int32_t c) const { return __ldg(g + c); }
};
struct GScaled {
    const double *__restrict__ g;
    const double *__restrict__ d;
    __device__ __forceinline__ double operator()(int32_t c) const { return __ddiv_rn(__ldg(g + c), __ldg(d + c)); }
};
// Ring buffers are written by other CTAs during the launch: plain (L1-
// allocating) loads, made coherent by the acquire fence the sync warp issues
// before it releases each item (it invalidates the SM's L1; within the item
// neighbouring rows then share L1 lines).
struct GRing {
    const double *base;
    uint32_t mask;
    __device__ __forceinline__ double operator()(int32_t c) const { return base[(uint32_t)c & mask]; }
};

template <int CH>
struct Chunk {
    double v[CH];
    int32_t c[CH];
    const double *sv;
    const int32_t *sc;
    int w;
    __device__ __forceinline__ void load(const double *sv_, const int32_t *sc_, int off, int w_, int lane) {
        sv = sv_ + off + lane;
        sc = sc_ + off + lane;
        w = w_;
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) {
                v[j] = sv[j * kSlice];
                c[j] = sc[j * kSlice];
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
        for (int j = CH; j < w; ++j) acc = __dadd_rn(acc, __dmul_rn(sv[j * kSlice], g(sc[j * kSlice])));
        return acc;
    }
};

template <int CH, class G>
__device__ __forceinline__ double tri_sum(const double *sv, const int32_t *sc, int2 info, int lane, const G &g) {
    Chunk<CH> ch;
    ch.load(sv, sc, info.x, info.y, lane);
    ch.gather_mul(g);
    return ch.add(0.0, g);
}

// Completion is tracked per CTA: prog[c] = (epoch << 32) | items of CTA c
// done (CTA c owns items c, c + G, c + 2G, ... and finishes them in order).
// All items <= t are done iff t < F = min_c (c + done_c * G): the sync warp
// reads the G counters in one parallel sweep and keeps F until it no
// longer suffices.
__device__ __forceinline__ int64_t read_frontier(const SkewParams &p, unsigned int epoch, int lane) {
    const int64_t G = gridDim.x;
    int64_t f = INT64_MAX;
    for (int64_t c = lane; c < G; c += 32) {
        // relaxed: an acquire load would invalidate the SM's L1 on every
        // poll; the caller fences once when the condition holds
        const unsigned long long v = ptx::ld_relaxed_gpu_u64(p.prog + c);
        const int64_t cnt = (unsigned int)(v >> 32) == epoch ? (int64_t)(v & 0xffffffffull) : 0;
        f = min(f, c + cnt * G);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) f = min(f, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)f, o));
    return f;
}

// One unit: phase j of physical tile tp; consumer warp `warp` owns slices
// warp + 8h (h < kRPT), one row of each per thread: the rows' loads and
// gathers are issued together.  Row, slice and ring indices are 32-bit (a
// rank holds < 2^31 rows: columns are int32).  The stage is released (empty
// barrier) as soon as its shared-memory data is consumed, before the results
// are stored.
template <int PH0, bool UNIT, int CH>
__device__ __forceinline__ void run_unit(const SkewParams &p, char *sm, int st, int tp, int j, int warp,
                                         int lane) {
    char *stg = stage_ptr(sm, p, st);
    int i[kRPT], rl[kRPT];
    bool has[kRPT], row[kRPT];
#pragma unroll
    for (int h = 0; h < kRPT; ++h) {
        const int sl = warp + h * kWarpsC;   // slice within the tile
        const int s = tp * kTSF + sl;
        has[h] = s < (int)p.nslices;
        i[h] = s * kSlice + lane;
        row[h] = has[h] && i[h] < (int)p.n;
        rl[h] = sl * kSlice + lane;
    }
    // vectors from the stage (full tile, aligned) or from global memory
    const bool vs = p.vec_bulk && (int64_t)(tp + 1) * kRowsF <= p.n;
    const double *svec = (const double *)(stg + (p.cap0 + p.cap1) * 12);
    auto vec = [&](int slot, const double *g, int h) -> double {
        return vs ? svec[slot * kRowsF + rl[h]] : (row[h] ? __ldg(g + i[h]) : 0.0);
    };
    auto release_stage = [&]() {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(empty_bar(sm) + st);
    };
    const double *v0 = (const double *)stg;
    const int32_t *c0 = (const int32_t *)(stg + p.cap0 * 8);
    const uint32_t rmask = (uint32_t)p.rmask, gmask = (uint32_t)p.gmask;
    if (PH0 == SKEW_RESID && j == 0) {
        // phase 0: r = b - A x (A = L + D + U, ascending column order), g(0)
        const double *v1 = (const double *)(stg + p.cap0 * 12);
        const int32_t *c1 = (const int32_t *)(stg + p.cap0 * 12 + p.cap1 * 8);
        const GFull gx{p.xin};
        double di[kRPT], bi[kRPT], xi[kRPT], acc[kRPT];
#pragma unroll
        for (int h = 0; h < kRPT; ++h) {
            di[h] = row[h] ? vec(0, p.dA, h) : 1.0;
            bi[h] = vec(1, p.b, h);
            xi[h] = vec(2, p.xin, h);
            acc[h] = 0.0;
        }
#ifndef NSM_SKEW_SEQ_RESID
        constexpr bool both = CH <= 8;  // both triangles' gathers in flight together
#else
        constexpr bool both = false;    // experiment: one triangle at a time (fewer registers)
#endif
        if constexpr (both) {
            Chunk<CH> cl[kRPT], cu[kRPT];
#pragma unroll
            for (int h = 0; h < kRPT; ++h) {
                const int sl = warp + h * kWarpsC;
                const int2 il = slice_info(sm, st, 0)[sl], iu = slice_info(sm, st, 1)[sl];
                cl[h].load(v0, c0, il.x, has[h] ? il.y : 0, lane);
                cu[h].load(v1, c1, iu.x, has[h] ? iu.y : 0, lane);
            }
#pragma unroll
            for (int h = 0; h < kRPT; ++h) {
                cl[h].gather_mul(gx);
                cu[h].gather_mul(gx);
            }
#pragma unroll
            for (int h = 0; h < kRPT; ++h) {
                acc[h] = cl[h].add(acc[h], gx);
                acc[h] = __dadd_rn(acc[h], __dmul_rn(di[h], xi[h]));
                acc[h] = cu[h].add(acc[h], gx);
            }
        } else {
#pragma unroll
            for (int h = 0; h < kRPT; ++h) {
                const int sl = warp + h * kWarpsC;
                const int2 il = slice_info(sm, st, 0)[sl], iu = slice_info(sm, st, 1)[sl];
                Chunk<CH> c;
                c.load(v0, c0, il.x, has[h] ? il.y : 0, lane);
                c.gather_mul(gx);
                acc[h] = c.add(acc[h], gx);
                acc[h] = __dadd_rn(acc[h], __dmul_rn(di[h], xi[h]));
                c.load(v1, c1, iu.x, has[h] ? iu.y : 0, lane);
                c.gather_mul(gx);
                acc[h] = c.add(acc[h], gx);
            }
        }
        release_stage();
#pragma unroll
        for (int h = 0; h < kRPT; ++h)
            if (row[h]) {
                const double r = __dsub_rn(bi[h], acc[h]);
                p.ring_r[(uint32_t)i[h] & rmask] = r;
                if (!UNIT) p.ring_g[(uint32_t)i[h] & gmask] = __ddiv_rn(r, di[h]);  // eq:jr-initial-guess
            }
        return;
    }
    // phase j >= 1: v = (rhs - T g(j-1)) / dT   (eq:jacobi, eq:LUiterMat)
    // staged slots: [dT (non-unit)] [rhs (given)] [x (x update)] [dn (scaling)]
    const bool last = j == p.k;
    const bool xadd = last && (p.epi == SKEW_XADD || p.epi == SKEW_XADD_SCALE);
    const bool scale = last && (p.epi == SKEW_STORE2 || p.epi == SKEW_XADD_SCALE || p.epi == SKEW_STORE_SCALE);
    const int s_rhs = UNIT ? 0 : 1;
    const int s_x = s_rhs + (PH0 == SKEW_RESID ? 0 : 1);
    const int s_dn = s_x + (xadd ? 1 : 0);
    double di[kRPT], ri[kRPT], xi[kRPT], dn[kRPT], acc[kRPT];
#pragma unroll
    for (int h = 0; h < kRPT; ++h) {
        di[h] = UNIT ? 1.0 : (row[h] ? vec(0, p.dT, h) : 1.0);
        ri[h] = PH0 == SKEW_RESID ? (row[h] ? p.ring_r[(uint32_t)i[h] & rmask] : 0.0)
                                  : vec(s_rhs, p.rhs, h);
        xi[h] = xadd ? vec(s_x, p.x, h) : 0.0;
        dn[h] = scale ? vec(s_dn, p.dn, h) : 1.0;
    }
    auto sweep_sum = [&](const auto &g) {
        Chunk<CH> ct[kRPT];
#pragma unroll
        for (int h = 0; h < kRPT; ++h) {
            const int2 it = slice_info(sm, st, 0)[warp + h * kWarpsC];
            ct[h].load(v0, c0, it.x, has[h] ? it.y : 0, lane);
        }
#pragma unroll
        for (int h = 0; h < kRPT; ++h) ct[h].gather_mul(g);
#pragma unroll
        for (int h = 0; h < kRPT; ++h) acc[h] = ct[h].add(0.0, g);
    };
    if (PH0 == SKEW_NONE && j == 1) {
        if (p.scaled_g0) sweep_sum(GScaled{p.g0, p.dT});
        else sweep_sum(GFull{p.g0});
    } else if (PH0 == SKEW_RESID && UNIT && j == 1) {
        sweep_sum(GRing{p.ring_r, rmask});  // y(0) = r
    } else {
        sweep_sum(GRing{p.ring_g + (int64_t)(j - 1) * p.gstride, gmask});
    }
    release_stage();
#pragma unroll
    for (int h = 0; h < kRPT; ++h) {
        if (!row[h]) continue;
        double v = __dsub_rn(ri[h], acc[h]);
        if (!UNIT) v = __ddiv_rn(v, di[h]);
        if (!isfinite(v)) atomicMin(p.flag, (unsigned long long)(p.sweep_id0 + j - 1));
        if (!last) {
            p.ring_g[(int64_t)j * p.gstride + ((uint32_t)i[h] & gmask)] = v;
            continue;
        }
        switch (p.epi) {
            case SKEW_STORE: p.out1[i[h]] = v; break;
            case SKEW_XADD: p.x[i[h]] = __dadd_rn(xi[h], v); break;
            case SKEW_STORE2: p.out1[i[h]] = v; p.out2[i[h]] = __ddiv_rn(v, dn[h]); break;
            case SKEW_XADD_SCALE: p.x[i[h]] = __dadd_rn(xi[h], __ddiv_rn(v, dn[h])); break;
            default: p.out1[i[h]] = __ddiv_rn(v, dn[h]); break;  // SKEW_STORE_SCALE
        }
    }
}

// Unit sequence of a CTA: items w = blockIdx.x + m G in order, each with units
// q = qa..qb (phase j0 + q on logical tile w - qD), qa = max(0, ceil((w - T +
// 1) / D)), qb = min(floor(w / D), k - j0).  Division-free: the quotients
// are carried along as w grows by G.
struct UnitGen {
    int64_t w, T, D, G, nitems;
    int64_t quo, rem;     // w = quo D + rem
    int64_t x2, quo2, rem2; // x2 = w - T + D; floor(x2 / D) once x2 >= 0
    int nph;
    int64_t q, qa, qb;
    bool valid;
    // skip = true: position on the first unit (producer); false: on item
    // blockIdx.x whether or not it has units (consumers walk every item)
    __device__ __forceinline__ void init(const SkewParams &p, bool skip) {
        G = gridDim.x;
        w = blockIdx.x;
        T = p.nbig;
        D = p.D;
        nitems = p.nitems;
        nph = p.k - p.j0;
        quo = w / D;
        rem = w - quo * D;
        x2 = w - T + D;
        quo2 = x2 >= 0 ? x2 / D : 0;
        rem2 = x2 >= 0 ? x2 - quo2 * D : 0;
        item();
        if (skip) first_unit();
    }
    __device__ __forceinline__ void item() {
        qb = min(quo, (int64_t)nph);
        qa = x2 >= 0 ? quo2 : 0;
    }
    __device__ __forceinline__ void advance_item() {
        w += G;
        rem += G;
        while (rem >= D) { rem -= D; ++quo; }
        const bool was_neg = x2 < 0;
        x2 += G;
        if (x2 >= 0) {
            if (was_neg) {
                quo2 = x2 / D;  // once
                rem2 = x2 - quo2 * D;
            } else {
                rem2 += G;
                while (rem2 >= D) { rem2 -= D; ++quo2; }
            }
        }
        item();
    }
    // first unit of the current or a later item (skipping items without units)
    __device__ __forceinline__ void first_unit() {
        while (w < nitems && qa > qb) advance_item();
        valid = w < nitems;
        q = qa;
    }
    __device__ __forceinline__ void next() {
        if (++q <= qb) return;
        advance_item();
        first_unit();
    }
};

// Slice pointers of a unit's parts: lanes 0..8 part 0, lanes 16..24 part 1.
// Slice pointers of a unit's parts: lane l <= kTSF holds ptr[s0 + l] of part 0
// (.x) and, for phase 0, of part 1 (.y).
template <int PH0>
__device__ __forceinline__ longlong2 unit_ptrs(const SkewParams &p, int64_t tp, int j, int lane) {
    const int64_t s0 = tp * kTSF, s1 = min(s0 + kTSF, p.nslices);
    const bool ph0 = PH0 == SKEW_RESID && j == 0;
    longlong2 pv = make_longlong2(0, 0);
    if (lane <= kTSF) {
        pv.x = __ldg((ph0 ? p.A0.ptr : p.T.ptr) + min(s0 + lane, s1));
        if (ph0) pv.y = __ldg(p.A1.ptr + min(s0 + lane, s1));
    }
    return pv;
}

constexpr int kPre = 2;  // records whose slice pointers the producer has in flight

template <int PH0, bool UNIT>
__device__ __forceinline__ void stage_unit(const SkewParams &p, char *sm, int st, int64_t tp, int j, longlong2 pvv,
                                           uint64_t pol_first, uint64_t pol_keep, int lane) {
    const bool ph0 = PH0 == SKEW_RESID && j == 0;
    const SellView &P0 = ph0 ? p.A0 : p.T;
    const int64_t pv = pvv.x, pw = pvv.y;
    const int64_t pnext = __shfl_down_sync(0xffffffffu, pv, 1), wnext = __shfl_down_sync(0xffffffffu, pw, 1);
    const int64_t pbase0 = __shfl_sync(0xffffffffu, pv, 0), pend0 = __shfl_sync(0xffffffffu, pv, kTSF);
    const int64_t pbase1 = __shfl_sync(0xffffffffu, pw, 0), pend1 = __shfl_sync(0xffffffffu, pw, kTSF);
    if (lane < kTSF) {
        slice_info(sm, st, 0)[lane] = make_int2((int)(pv - pbase0), (int)((pnext - pv) / kSlice));
        if (ph0) slice_info(sm, st, 1)[lane] = make_int2((int)(pw - pbase1), (int)((wnext - pw) / kSlice));
    }
    __syncwarp();
    if (lane == 0) {
        char *sp = stage_ptr(sm, p, st);
        uint64_t *bar = full_bar(sm) + st;
        const VecSet V = unit_vectors<PH0, UNIT>(p, j);
        const bool vs = p.vec_bulk && (tp + 1) * kRowsF <= p.n;
        uint32_t bytes = (uint32_t)((pend0 - pbase0) * 12 + (ph0 ? (pend1 - pbase1) * 12 : 0));
        if (vs) bytes += (uint32_t)(V.n * kVecBytes);
        ptx::mbar_expect_tx(bar, bytes);
        const uint64_t pol0 = ph0 ? (p.keep0 ? pol_keep : pol_first) : (j < p.k ? pol_keep : pol_first);
        if (pend0 > pbase0) {
            ptx::bulk_g2s(sp, P0.val + pbase0, (uint32_t)((pend0 - pbase0) * 8), bar, pol0);
            ptx::bulk_g2s(sp + p.cap0 * 8, P0.col + pbase0, (uint32_t)((pend0 - pbase0) * 4), bar, pol0);
        }
        if (ph0 && pend1 > pbase1) {
            const uint64_t pol1 = p.keep1 ? pol_keep : pol_first;
            ptx::bulk_g2s(sp + p.cap0 * 12, p.A1.val + pbase1, (uint32_t)((pend1 - pbase1) * 8), bar, pol1);
            ptx::bulk_g2s(sp + p.cap0 * 12 + p.cap1 * 8, p.A1.col + pbase1, (uint32_t)((pend1 - pbase1) * 4), bar,
                          pol1);
        }
        if (vs) {
#pragma unroll
            for (int v = 0; v < kNVec; ++v)
                if (v < V.n)
                    ptx::bulk_g2s(sp + (p.cap0 + p.cap1) * 12 + v * kVecBytes, V.v[v] + tp * kRowsF,
                                  (uint32_t)kVecBytes, bar, pol_keep);
        }
    }
    __syncwarp();
}

// Record sequence of a CTA: for each of its items w = blockIdx.x + m G, the
// sub-units (unit (w, q) = big tile u = w - qD = 256-row tiles uB .. uB+B-1
// below ntiles, phase j0 + q), or one empty record for an item without units.
struct Seq {
    UnitGen g;
    int64_t q;
    int b;
    int64_t tp;
    int j, flags;
    bool valid;
    __device__ __forceinline__ void settle(const SkewParams &p) {
        valid = g.w < p.nitems;
        if (!valid) return;
        if (g.qa > g.qb) {
            tp = -1;
            j = 0;
            flags = U_FIRST | U_LAST;
            return;
        }
        const int64_t t = (g.w - q * p.D) * p.B + b;
        tp = p.desc ? p.ntiles - 1 - t : t;
        j = p.j0 + (int)q;
        const bool lastb = b + 1 >= p.B || t + 1 >= p.ntiles;
        flags = (q == g.qa && b == 0 ? U_FIRST : 0) | (q == g.qb && lastb ? U_LAST : 0);
    }
    __device__ __forceinline__ void init(const SkewParams &p) {
        g.init(p, false);
        q = g.qa;
        b = 0;
        settle(p);
    }
    __device__ __forceinline__ void next(const SkewParams &p) {
        if (tp >= 0) {
            const int64_t t = (g.w - q * p.D) * p.B + b;
            if (b + 1 < p.B && t + 1 < p.ntiles) {
                ++b;
                settle(p);
                return;
            }
            b = 0;
            if (q < g.qb) {
                ++q;
                settle(p);
                return;
            }
        }
        g.advance_item();
        q = g.qa;
        b = 0;
        settle(p);
    }
};

// Producer: walks the record sequence with the slice pointers of the next
// kPre records already loading (their latency would otherwise serialise
// every unit); writes each record's descriptor into its stage.
template <int PH0, bool UNIT>
__device__ __forceinline__ void produce(const SkewParams &p, char *sm, int lane) {
    const uint64_t pol_first = ptx::policy_evict_first(), pol_keep = ptx::policy_evict_normal();
    Seq seq;
    seq.init(p);
    int64_t ptp[kPre];
    longlong2 pv[kPre];
    int pj[kPre], pf[kPre];
    bool ok[kPre];
#pragma unroll
    for (int k = 0; k < kPre; ++k) {
        ok[k] = seq.valid;
        ptp[k] = seq.tp;
        pj[k] = seq.j;
        pf[k] = seq.flags;
        pv[k] = (ok[k] && seq.tp >= 0) ? unit_ptrs<PH0>(p, ptp[k], pj[k], lane) : make_longlong2(0, 0);
        if (seq.valid) seq.next(p);
    }
    int st = 0;
    uint32_t round = 0;
    auto next_stage = [&]() {
        if (++st == p.nst) { st = 0; ++round; }
    };
    auto wait_free = [&]() {
        if (round > 0) ptx::mbar_wait_sleep(empty_bar(sm) + st, (round - 1) & 1);
    };
    bool more = ok[0];
    while (more) {
#pragma unroll
        for (int k = 0; k < kPre; ++k) {
            if (!ok[k]) { more = false; break; }
            wait_free();
            if (lane == 0) udesc(sm)[st] = UDesc{(int)ptp[k], (short)pj[k], (short)pf[k]};
            if (ptp[k] >= 0) {
                stage_unit<PH0, UNIT>(p, sm, st, ptp[k], pj[k], pv[k], pol_first, pol_keep, lane);
            } else {
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(full_bar(sm) + st);
            }
            next_stage();
            ok[k] = seq.valid;
            ptp[k] = seq.tp;
            pj[k] = seq.j;
            pf[k] = seq.flags;
            pv[k] = (ok[k] && seq.tp >= 0) ? unit_ptrs<PH0>(p, ptp[k], pj[k], lane) : make_longlong2(0, 0);
            if (seq.valid) seq.next(p);
        }
    }
    // end of the sequence
    wait_free();
    if (lane == 0) {
        udesc(sm)[st] = UDesc{-1, 0, (short)U_END};
        ptx::mbar_arrive(full_bar(sm) + st);
    }
}

// Sync warp: signals "ready" for this CTA's items in order, once every item
// <= w - Dw is done and the item's barrier slot is free (the consumers
// finished item m - (kSlots-1)).  The progress counters are polled with
// relaxed loads, and not at all while the condition still includes this
// CTA's own unpublished item.  (Publication is done by the consumers: the
// last warp to finish an item.)
__device__ __forceinline__ void sync_role(const SkewParams &p, char *sm, unsigned int epoch, int lane) {
    const int64_t G = gridDim.x, c = blockIdx.x;
    const int64_t nmine = c < p.nitems ? (p.nitems - c + G - 1) / G : 0;
    int64_t F = 0;  // all items < F are known to be done
    for (int64_t m = 0; m < nmine; ++m) {
        if (m >= kSlots - 1) {
            const int64_t mo = m - (kSlots - 1);  // slot reuse: that item is finished here
            ptx::mbar_wait_sleep(idone_bar(sm) + (mo % kSlots), (uint32_t)(mo / kSlots) & 1);
        }
        const int64_t tgt = c + m * G - p.Dw;
        if (tgt >= F) {
            const uint64_t t0 = ptx::globaltimer_ns();
            while (true) {
                // own items before m are finished (the wait above) but maybe
                // not yet published: the frontier may lag by our own counter
                F = read_frontier(p, epoch, lane);
                if (tgt < F) break;
                if (ptx::globaltimer_ns() - t0 > p.timeout_ns) {
                    if (lane == 0) atomicOr(p.err, 2u);
                    F = INT64_MAX;  // give up: let the consumers drain
                    break;
                }
                __nanosleep(32);
            }
        }
        // acquire: the frontier was read with relaxed loads; one gpu-scope
        // fence per item (it also invalidates the SM's L1, so the consumers'
        // L1-cached ring reads of this item see what the counters published)
        __threadfence();
        if (lane == 0) {
            trace_at(p, 2, (int)m, 0);  // item made ready
            ptx::mbar_arrive(ready_bar(sm) + (m % kSlots));
        }
        __syncwarp();
    }
}

template <int PH0, bool UNIT, int CH>
#ifndef NSM_SKEW_MINB4
#define NSM_SKEW_MINB4 2  // CTAs per SM the CH = 4 variants are register-budgeted for
#endif
__global__ void __launch_bounds__(kThreadsF, CH <= 4 ? NSM_SKEW_MINB4 : (CH <= 8 ? 2 : 1)) k_skew(const __grid_constant__ SkewParams p) {
    extern __shared__ __align__(128) char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned int epoch = *(volatile unsigned int *)&p.sync->epoch;
    if (threadIdx.x == 0) {
        for (int st = 0; st < p.nst; ++st) {
            ptx::mbar_init(full_bar(sm) + st, 1);
            ptx::mbar_init(empty_bar(sm) + st, kWarpsC);
        }
        for (int sl = 0; sl < kSlots; ++sl) {
            ptx::mbar_init(ready_bar(sm) + sl, 1);
            ptx::mbar_init(idone_bar(sm) + sl, kWarpsC);
            pubcnt(sm)[sl] = 0;
        }
        ptx::mbar_init_fence();
    }
    __syncthreads();

    if (warp == kWarpP) {
        produce<PH0, UNIT>(p, sm, lane);
    } else if (warp == kWarpS) {
        sync_role(p, sm, epoch, lane);
    } else {
        // consumers: follow the producer's descriptors (stage and parity
        // tracked incrementally); item boundaries come with the flags
        int st = 0;
        uint32_t par = 0;
        int64_t m = -1;
        int it = 0;
        while (true) {
            if (warp == 0 && lane == 0) trace_at(p, 0, it, 0);
            ptx::mbar_wait_sleep(full_bar(sm) + st, par);
            if (warp == 0 && lane == 0) trace_at(p, 0, it, 1);
            const UDesc un = udesc(sm)[st];
            if (un.flags & U_END) break;
            if (un.flags & U_FIRST) {
                ++m;
                uint64_t *rb = ready_bar(sm) + (m % kSlots);
                const uint32_t rpar = (uint32_t)(m / kSlots) & 1;
                if (warp == 0 && !ptx::mbar_test(rb, rpar)) {  // statistics: consumers stalled on readiness
                    const uint64_t t0 = ptx::globaltimer_ns();
                    ptx::mbar_wait_sleep(rb, rpar);
                    if (lane == 0) {
                        atomicAdd(&p.sync->waits, 1ull);
                        atomicAdd(&p.sync->wait_ns, ptx::globaltimer_ns() - t0);
                    }
                }
                ptx::mbar_wait_sleep(rb, rpar);
            }
            if (un.tp >= 0) {
                run_unit<PH0, UNIT, CH>(p, sm, st, un.tp, un.j, warp, lane);  // releases the stage
            } else {
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(empty_bar(sm) + st);
            }
            if (warp == 0 && lane == 0) trace_at(p, 0, it, 2);
            if (un.flags & U_LAST) {
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(idone_bar(sm) + (m % kSlots));
                    if (warp == 0) trace_at(p, 2, (int)m, 2);
                    // the last warp to finish item m publishes "m + 1 items done";
                    // acq_rel at CTA scope makes the other warps' stores happen
                    // before this warp's release (cumulativity), max keeps the
                    // counter monotone if a later item's publication overtakes
                    const unsigned int prev = ptx::atom_add_acqrel_cta_shared(pubcnt(sm) + (m % kSlots), 1u);
                    if (prev == (unsigned int)((m / kSlots + 1) * kWarpsC - 1)) {
                        trace_at(p, 2, (int)m, 1);  // item published
                        ptx::red_max_release_gpu_u64(p.prog + blockIdx.x,
                                                     ((unsigned long long)epoch << 32) | (unsigned long long)(m + 1));
                    }
                }
            }
            if (++st == p.nst) { st = 0; par ^= 1; }
            ++it;
        }
    }
    // ---- the last CTA out resets the launch state for the next launch
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(&p.sync->exits, 1u);
        if (prev == gridDim.x - 1) {
            p.sync->wmark = 0;
            p.sync->exits = 0;
            p.sync->epoch = epoch + 1 == 0 ? 1 : epoch + 1;
            __threadfence();
        }
    }
}

// ---- host side -----------------------------------------------------------------
template <int PH0, bool UNIT, int CH>
const void *kernel_ptr() {
    return (const void *)k_skew<PH0, UNIT, CH>;
}

const void *pick(int ph0, bool unit, int ch) {
#define NSM_PK(P, U)                                                                               \
    (ch == 4 ? kernel_ptr<P, U, 4>() : ch == 8 ? kernel_ptr<P, U, 8>() : kernel_ptr<P, U, 16>())
    if (ph0 == SKEW_RESID) return unit ? NSM_PK(SKEW_RESID, true) : NSM_PK(SKEW_RESID, false);
    return unit ? NSM_PK(SKEW_NONE, true) : NSM_PK(SKEW_NONE, false);
#undef NSM_PK
}

int sm_count_f() {  // of the current device (launches happen with the handle's device current)
    static int n[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!n[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n[dev] = v > 0 ? v : 148;
    }
    return n[dev];
}

struct GeoF {
    int nst = 0, per_sm = 0;
    size_t smem = 0;
};

// stages: maximise resident consumer warps (<= 32 per SM, <= 4 CTAs), then depth
GeoF geometry_f(const void *k, int64_t stage_bytes) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, int64_t>, GeoF> cache;  // per device (opt-in attribute)
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    auto key = std::make_tuple(dev, k, stage_bytes);
    auto itc = cache.find(key);
    if (itc != cache.end()) return itc->second;
    GeoF g;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMaxF);
    // experiment knobs (tools/skew_exp.py): cap stages / CTAs per SM
    static const int max_nst = knob("NSM_DEBUG_SKEW_NST") ? atoi(knob("NSM_DEBUG_SKEW_NST")) : kMaxStages;
    static const int max_per = knob("NSM_DEBUG_SKEW_PERSM") ? atoi(knob("NSM_DEBUG_SKEW_PERSM")) : 4;
    int best = -1;
    for (int nst = 2; nst <= std::min(kMaxStages, max_nst); ++nst) {
        const int64_t smem = kHeader + nst * stage_bytes;
        if (smem > kSmemMaxF) break;
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kThreadsF, (size_t)smem);
        per = std::min(per, max_per);
        const int warps = std::min(per * kWarpsC, 32);
        if (per > 0 && warps >= best) {
            best = warps;
            g.nst = nst;
            g.per_sm = per;
            g.smem = (size_t)smem;
        }
    }
    cache[key] = g;
    return g;
}

int64_t pow2_at_least(int64_t v) {
    int64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

inline int chunk_for(int maxw) { return maxw <= 4 ? 4 : (maxw <= 8 ? 8 : 16); }

}  // namespace

int skew_tile_rows() { return kRowsF; }

// Shape of one launch (grid, stages, skew, rings); the same function sizes the
// handle's buffers at setup (upper bound over k <= kmax) and each launch.
SkewShape skew_shape(int ph0, bool unit, int maxw0, int maxw1, int maxwT, int k, int64_t n, int DT, int DA,
                     int dw_override) {
    SkewShape sh;
    const int64_t cap0 = (int64_t)kRowsF * std::max({ph0 == SKEW_RESID ? maxw0 : 0, maxwT, 1});
    const int64_t cap1 = ph0 == SKEW_RESID ? (int64_t)kRowsF * std::max(maxw1, 1) : 0;
    const int ch = chunk_for(std::max({ph0 == SKEW_RESID ? std::max(maxw0, maxw1) : 0, maxwT}));
    const void *kern = pick(ph0, unit, ch);
    // staged vector segments: phase 0 dA, b, x; later phases dT, rhs, x, dn
    const int nvec = ph0 == SKEW_RESID ? 3 : (unit ? 0 : 1) + 3;
    const int64_t stage_bytes = ((cap0 + cap1) * 12 + nvec * kVecBytes + 127) / 128 * 128;
    const GeoF g = geometry_f(kern, stage_bytes);
    if (!g.nst) return sh;
    sh.ok = true;
    sh.kernel = kern;
    sh.nst = g.nst;
    sh.smem = g.smem;
    sh.cap0 = cap0;
    sh.cap1 = cap1;
    sh.stage_bytes = stage_bytes;
    sh.ntiles = (n + kRowsF - 1) / kRowsF;
    // B consecutive 256-row tiles per scheduling tile: the per-item
    // synchronisation is paid once per B tiles of every phase
    static const int env_b = knob("NSM_DEBUG_SKEW_B") ? atoi(knob("NSM_DEBUG_SKEW_B")) : 0;
    int B = env_b > 0 ? env_b : 8;
    while (B > 1 && (B & (B - 1))) --B;  // power of two (ring masks)
    sh.B = B;
    sh.nbig = (sh.ntiles + B - 1) / B;
    sh.grid = (int)std::min<int64_t>((int64_t)sm_count_f() * g.per_sm, std::max<int64_t>(sh.nbig, 1));
    const int j0 = ph0 == SKEW_RESID ? 0 : 1;
    const int DTb = (DT + B - 1) / B, DAb = (DA + B - 1) / B;
    // wait distance: two rounds of the grid (CTAs run their items in
    // lockstep rounds; a wait blocks only on a CTA a full round behind)
    sh.Dw = dw_override > 0 ? dw_override : 2 * sh.grid;
    sh.D = sh.Dw + std::max(DTb, ph0 == SKEW_RESID ? DAb : 0);
    sh.nitems = sh.nbig + (int64_t)(k - j0) * sh.D;
    const int64_t big_pow2 = pow2_at_least(std::max<int64_t>(sh.nbig, 1));
    // ring lengths, reported in 256-row tiles
    sh.Mr = ph0 == SKEW_RESID ? std::min(pow2_at_least((int64_t)k * sh.D + sh.Dw), big_pow2) * B : 0;
    sh.Mg = std::min(pow2_at_least((int64_t)sh.D + DTb + sh.Dw), big_pow2) * B;
    return sh;
}

cudaError_t launch_skew(const SkewLaunch &L, cudaStream_t st) {
    const SkewShape &sh = L.shape;
    if (!sh.ok) return cudaErrorInvalidConfiguration;
    if (L.n == 0) return cudaSuccess;
    SkewParams p{};
    p.n = L.n;
    p.nslices = (L.n + kSlice - 1) / kSlice;
    p.ntiles = sh.ntiles;
    p.nitems = sh.nitems;
    p.nbig = sh.nbig;
    p.B = sh.B;
    p.desc = L.desc;
    p.k = L.k;
    p.j0 = L.ph0 == SKEW_RESID ? 0 : 1;
    p.D = sh.D;
    p.Dw = sh.Dw;
    p.epi = L.epi;
    p.scaled_g0 = L.scaled_g0;
    if (L.A0) p.A0 = view(*L.A0);
    if (L.A1) p.A1 = view(*L.A1);
    p.T = view(*L.T);
    p.dA = L.dA;
    p.b = L.b;
    p.xin = L.xin;
    p.dT = L.dT;
    p.rhs = L.rhs;
    p.g0 = L.g0;
    p.x = L.x;
    p.out1 = L.out1;
    p.out2 = L.out2;
    p.dn = L.dn;
    p.ring_r = L.ring_r;
    p.ring_g = L.ring_g;
    p.rmask = sh.Mr * kRowsF - 1;
    p.gmask = sh.Mg * kRowsF - 1;
    p.gstride = sh.Mg * kRowsF;
    p.flag = L.flag;
    p.sweep_id0 = L.sweep_id0;
    p.err = L.err;
    p.timeout_ns = L.timeout_ns;
    p.sync = L.sync;
    p.prog = L.prog;
    p.nst = sh.nst;
    p.keep0 = L.keep0;
    p.keep1 = L.keep1;
    p.cap0 = sh.cap0;
    p.cap1 = sh.cap1;
    p.stage_bytes = sh.stage_bytes;
    // vector segments go through the bulk-copy engine when 16-byte aligned
    auto al = [](const void *q) { return q == nullptr || ((uintptr_t)q & 15) == 0; };
    p.trace = L.trace;
    p.vec_bulk = al(p.dA) && al(p.b) && al(p.xin) && al(p.dT) && al(p.rhs) && al(p.x) && al(p.dn);
    static const bool novec = knob("NSM_DEBUG_SKEW_NOVEC") != nullptr;  // experiment knob
    if (novec) p.vec_bulk = 0;
    void *args[] = {&p};
    // cooperative: all CTAs co-resident (the item schedule relies on it)
    return cudaLaunchCooperativeKernel(sh.kernel, dim3((unsigned)sh.grid), dim3(kThreadsF), args, sh.smem, st);
}

void preload_fused_kernels() {
    cudaFuncAttributes a;
    for (int ph0 : {SKEW_RESID, SKEW_NONE})
        for (bool unit : {false, true})
            for (int ch : {4, 8, 16}) cudaFuncGetAttributes(&a, pick(ph0, unit, ch));
}

}  // namespace nsm
