// stream.cu — bulk-copy pipelined variants of the residual and sweep kernels
// (DESIGN.md §6 "Kernels").
//
// The SELL value/index streams of a contiguous range of slices are moved
// HBM -> shared memory by the bulk-copy (TMA) engine — cp.async.bulk with
// completion on an mbarrier — NST stages ahead of the consumers, so the DRAM
// stream does not stall while the consumers make their second round trip
// (the x / g gathers through L1/L2).  One producer warp (one elected lane)
// issues the copies; TS consumer warps each own one slice (one thread per
// row) of the tile, pull a register chunk of CH entries of their row from
// shared memory (lane-contiguous, conflict-free), issue all CH gathers
// together, and accumulate in stored order — the same arithmetic sequence as
// the plain kernels in kernels.cu and as the oracle, hence bit-identical
// results.
//
// Tiles of TS consecutive slices are dealt round-robin to a persistent grid
// (a multiple of the SM count), so at any moment all CTAs stream
// neighbouring tiles and the gathered vector windows stay L2-resident.  The
// number of stages is chosen per matrix to maximise resident consumer warps
// (occupancy from registers and shared memory), then pipeline depth.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <utility>

#include "nsm_internal.h"
#include "ptx.cuh"
#include "stream_dev.cuh"

namespace nsm {

namespace {

template <int OUT, int CH, bool OFS, bool WIN>
__device__ __forceinline__ void residual_tma_body(int64_t n, int64_t s_begin, int64_t s_end, SellView L, SellView U,
                                                  const double *__restrict__ d, const double *__restrict__ b,
                                                  const double *__restrict__ x, double *__restrict__ out,
                                                  double *__restrict__ out2, int nst, int64_t cap, WinView W) {
    extern __shared__ __align__(128) char sm[];
    constexpr bool ofs = OFS;
    static_assert(!WIN || OFS, "windowed kernels need the offset-aligned layout");
    const Layout Ly{nst, 2, cap, ofs ? 8 : 12, WIN ? (int64_t)W.wcap : 0};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (s_end - s_begin + kTS - 1) / kTS;
    init_barriers(Ly, sm);
    if (warp == kTS) {
        const SellView P[2] = {L, U};
        if constexpr (OFS) producer<2, WIN>(Ly, sm, P, s_begin, s_end, ntiles, lane, W, x, n);
        else if (lane == 0) producer_compact<2>(Ly, sm, P, s_begin, s_end, ntiles);
        return;
    }
    const GatherPlainT gx{x};
    pdl_wait();  // x, b of the previous kernel
    int it = 0;  // stage = it % nst (running stage/phase counters here measured 5-14 % slower on C3/C4)
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % nst;
        const uint32_t ph = (uint32_t)(it / nst) & 1;
        const int64_t s0 = s_begin + t * kTS, s = s0 + warp;
        const bool has = s < s_end;
        const int64_t i = s * kSlice + lane;
        const bool row = has && i < n;
        // per-row vectors and slice geometry: issued before waiting on the copy
        const double di = row ? __ldg(d + i) : 0.0, xi = row ? __ldg(x + i) : 0.0;
        const double bi = (OUT != OUT_AX && row) ? __ldg(b + i) : 0.0;
        int64_t lo = 0, uo = 0;
        int lw = 0, uw = 0;
        Offsets<CH> ol, ou;
        if (!OFS && has) {
            const int64_t l0 = __ldg(L.ptr + s0), ls = __ldg(L.ptr + s), ls1 = __ldg(L.ptr + s + 1);
            const int64_t u0 = __ldg(U.ptr + s0), us = __ldg(U.ptr + s), us1 = __ldg(U.ptr + s + 1);
            lo = ls - l0;
            lw = (int)((ls1 - ls) / kSlice);
            uo = us - u0;
            uw = (int)((us1 - us) / kSlice);
        }
        mbar_wait(Ly.full(sm) + st, ph);
        if constexpr (OFS) {  // slice geometry from the producer's header
            const int2 hl = *(const int2 *)(Ly.hdr(sm, st, 0) + 2 * warp);
            const int2 hu = *(const int2 *)(Ly.hdr(sm, st, 1) + 2 * warp);
            lo = hl.x; lw = hl.y;
            uo = hu.x; uw = hu.y;
            ol.at(Ly.col(sm, st, 0), lo);
            ou.at(Ly.col(sm, st, 1), uo);
        }
        double acc = 0.0;
        if constexpr (WIN) {
            if (has) {
                const double *ws = Ly.win(sm, st);
                if constexpr (CH <= 8) {
                    WinChunk<CH> cl, cu;
                    cl.load(Ly.val(sm, st, 0), Ly.col(sm, st, 0), ws, lo, lw, lane, row);
                    cu.load(Ly.val(sm, st, 1), Ly.col(sm, st, 1), ws, uo, uw, lane, row);
                    acc = cl.add(acc);
                    acc = __dadd_rn(acc, __dmul_rn(di, xi));
                    acc = cu.add(acc);
                } else {
                    WinChunk<CH> c;
                    c.load(Ly.val(sm, st, 0), Ly.col(sm, st, 0), ws, lo, lw, lane, row);
                    acc = c.add(acc);
                    acc = __dadd_rn(acc, __dmul_rn(di, xi));
                    c.load(Ly.val(sm, st, 1), Ly.col(sm, st, 1), ws, uo, uw, lane, row);
                    acc = c.add(acc);
                }
            }
        } else if (has) {
            if constexpr (CH <= 8) {  // both triangles' gathers in flight together
                StagedChunk<CH> cl, cu;
                if constexpr (OFS) {
                    cl.load_ofs(Ly.val(sm, st, 0), ol, lo, lw, lane, i, n);
                    cu.load_ofs(Ly.val(sm, st, 1), ou, uo, uw, lane, i, n);
                } else {
                    cl.load(Ly.val(sm, st, 0), Ly.col(sm, st, 0), lo, lw, lane);
                    cu.load(Ly.val(sm, st, 1), Ly.col(sm, st, 1), uo, uw, lane);
                }
                cl.gather_mul(gx);
                cu.gather_mul(gx);
                acc = cl.add(acc, gx);
                acc = __dadd_rn(acc, __dmul_rn(di, xi));
                acc = cu.add(acc, gx);
            } else {                  // wide rows: one triangle at a time (registers)
                StagedChunk<CH> c;
                if constexpr (OFS) c.load_ofs(Ly.val(sm, st, 0), ol, lo, lw, lane, i, n);
                else c.load(Ly.val(sm, st, 0), Ly.col(sm, st, 0), lo, lw, lane);
                c.gather_mul(gx);
#if NSM_RES_PREFETCH_U
                if constexpr (OFS) {  // U's gathers to L1 while L's are in flight (no registers held)
                    if (i < n) {
#pragma unroll
                        for (int j = 0; j < CH; ++j)
                            if (j < uw)
                                asm volatile("prefetch.global.L1 [%0];" ::"l"(x + Offsets<CH>::col(i, ou.so[j], n)));
                    }
                }
#endif
                acc = c.add(acc, gx);
                acc = __dadd_rn(acc, __dmul_rn(di, xi));
                if constexpr (OFS) c.load_ofs(Ly.val(sm, st, 1), ou, uo, uw, lane, i, n);
                else c.load(Ly.val(sm, st, 1), Ly.col(sm, st, 1), uo, uw, lane);
                c.gather_mul(gx);
                acc = c.add(acc, gx);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(Ly.empty(sm) + st);  // the stage may be refilled
        if (row) {
            if (OUT == OUT_AX) {
                out[i] = acc;
            } else {
                const double r = __dsub_rn(bi, acc);
                out[i] = r;
                if (OUT == OUT_RG) out2[i] = __ddiv_rn(r, di);
            }
        }
    }
}

template <int OUT, int CH, bool OFS>
__global__ void __launch_bounds__(kThreadsT) k_residual_tma(int64_t n, int64_t s_begin, int64_t s_end, SellView L,
                                                            SellView U, const double *__restrict__ d,
                                                            const double *__restrict__ b,
                                                            const double *__restrict__ x, double *__restrict__ out,
                                                            double *__restrict__ out2, int nst, int64_t cap,
                                                            WinView W) {
    residual_tma_body<OUT, CH, OFS, false>(n, s_begin, s_end, L, U, d, b, x, out, out2, nst, cap, W);
}

// Windowed variant: the producer's window bookkeeping must not cost the
// short-row kernels their third co-resident CTA (72 registers; without the
// bound ptxas takes 96 and the C2 / C5 residual lost a third of its warps).
template <int OUT, int CH>
__global__ void __launch_bounds__(kThreadsT, (CH <= 8 || CH == 14) ? 3 : 2)  // CH 14: 72 registers, 3 CTAs/SM
    k_residual_tma_w(int64_t n, int64_t s_begin, int64_t s_end, SellView L, SellView U, const double *__restrict__ d,
                     const double *__restrict__ b, const double *__restrict__ x, double *__restrict__ out,
                     double *__restrict__ out2, int nst, int64_t cap, WinView W) {
    residual_tma_body<OUT, CH, true, true>(n, s_begin, s_end, L, U, d, b, x, out, out2, nst, cap, W);
}

__device__ __forceinline__ const double *gathered(const GatherPlainT &g) { return g.g; }
__device__ __forceinline__ const double *gathered(const GatherScaledT &) { return nullptr; }

template <bool UNIT, int EPI, class G, int CH, bool OFS, bool WIN>
__device__ __forceinline__ void sweep_tma_body(int64_t n, int64_t s_begin, int64_t s_end, SellView T,
                                               const double *__restrict__ dT, const double *__restrict__ rhs, G gin,
                                               double *__restrict__ gout, double *__restrict__ x,
                                               const double *__restrict__ dnext, double *__restrict__ gout2,
                                               unsigned long long *flag, int64_t sweep_id, int nst, int64_t cap,
                                               WinView W) {
    extern __shared__ __align__(128) char sm[];
    constexpr bool ofs = OFS;
    static_assert(!WIN || OFS, "windowed kernels need the offset-aligned layout");
    const Layout Ly{nst, 1, cap, ofs ? 8 : 12, WIN ? (int64_t)W.wcap : 0};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (s_end - s_begin + kTS - 1) / kTS;
    init_barriers(Ly, sm);
    if (warp == kTS) {
        const SellView P[1] = {T};
        if constexpr (OFS) producer<1, WIN>(Ly, sm, P, s_begin, s_end, ntiles, lane, W, gathered(gin), n);
        else if (lane == 0) producer_compact<1>(Ly, sm, P, s_begin, s_end, ntiles);
        return;
    }
    pdl_wait();  // rhs, iterates, x of the previous kernels
    int it = 0;  // stage = it % nst (running stage/phase counters here measured 5-14 % slower on C3/C4)
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % nst;
        const uint32_t ph = (uint32_t)(it / nst) & 1;
        const int64_t s0 = s_begin + t * kTS, s = s0 + warp;
        const bool has = s < s_end;
        const int64_t i = s * kSlice + lane;
        const bool row = has && i < n;
        const double ri = row ? __ldg(rhs + i) : 0.0;
        const double di = (!UNIT && row) ? __ldg(dT + i) : 1.0;
        const double xi = ((EPI == EPI_XADD || EPI == EPI_XADD_SCALE) && row) ? x[i] : 0.0;
        const double dn = ((EPI == EPI_XADD_SCALE || EPI == EPI_STORE2) && row) ? __ldg(dnext + i) : 1.0;
        int64_t to = 0;
        int tw = 0;
        Offsets<CH> ot;
        if (!OFS && has) {
            const int64_t t0 = __ldg(T.ptr + s0), ts = __ldg(T.ptr + s), ts1 = __ldg(T.ptr + s + 1);
            to = ts - t0;
            tw = (int)((ts1 - ts) / kSlice);
        }
        mbar_wait(Ly.full(sm) + st, ph);
        if constexpr (OFS) {  // slice geometry from the producer's header
            const int2 h = *(const int2 *)(Ly.hdr(sm, st, 0) + 2 * warp);
            to = h.x; tw = h.y;
            ot.at(Ly.col(sm, st, 0), to);
        }
        double acc = 0.0;
        if constexpr (WIN && CH == 7) {   // chunks of 7 (fewer registers: four CTAs per SM)
            if (has) acc = win_sum_chunked<7>(Ly.val(sm, st, 0), Ly.col(sm, st, 0), Ly.win(sm, st), to, tw, lane, row, acc);
        } else if constexpr (WIN) {
            if (has) {
                WinChunk<CH> ct;
                ct.load(Ly.val(sm, st, 0), Ly.col(sm, st, 0), Ly.win(sm, st), to, tw, lane, row);
                acc = ct.add(acc);
            }
        } else if (has) {
            StagedChunk<CH> ct;
            if constexpr (OFS) ct.load_ofs(Ly.val(sm, st, 0), ot, to, tw, lane, i, n);
            else ct.load(Ly.val(sm, st, 0), Ly.col(sm, st, 0), to, tw, lane);
            ct.gather_mul(gin);
            acc = ct.add(acc, gin);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(Ly.empty(sm) + st);
        if (row) {
            double v = __dsub_rn(ri, acc);
            if (!UNIT) v = __ddiv_rn(v, di);
            if (!isfinite(v)) atomicMin(flag, (unsigned long long)sweep_id);
            if (EPI == EPI_STORE) gout[i] = v;
            if (EPI == EPI_XADD) x[i] = __dadd_rn(xi, v);
            if (EPI == EPI_STORE2) { gout[i] = v; gout2[i] = __ddiv_rn(v, dn); }
            if (EPI == EPI_XADD_SCALE) x[i] = __dadd_rn(xi, __ddiv_rn(v, dn));
        }
    }
}

template <bool UNIT, int EPI, class G, int CH, bool OFS>
__global__ void __launch_bounds__(kThreadsT) k_sweep_tma(int64_t n, int64_t s_begin, int64_t s_end, SellView T,
                                                         const double *__restrict__ dT,
                                                         const double *__restrict__ rhs, G gin,
                                                         double *__restrict__ gout, double *__restrict__ x,
                                                         const double *__restrict__ dnext, double *__restrict__ gout2,
                                                         unsigned long long *flag, int64_t sweep_id, int nst,
                                                         int64_t cap, WinView W) {
    sweep_tma_body<UNIT, EPI, G, CH, OFS, false>(n, s_begin, s_end, T, dT, rhs, gin, gout, x, dnext, gout2, flag,
                                                 sweep_id, nst, cap, W);
}

template <bool UNIT, int EPI, int CH>
__global__ void __launch_bounds__(kThreadsT, CH == 7 ? 4 : 3)
    k_sweep_tma_w(int64_t n, int64_t s_begin, int64_t s_end, SellView T, const double *__restrict__ dT,
                  const double *__restrict__ rhs, GatherPlainT gin, double *__restrict__ gout, double *__restrict__ x,
                  const double *__restrict__ dnext, double *__restrict__ gout2, unsigned long long *flag,
                  int64_t sweep_id, int nst, int64_t cap, WinView W) {
    sweep_tma_body<UNIT, EPI, GatherPlainT, CH, true, true>(n, s_begin, s_end, T, dT, rhs, gin, gout, x, dnext, gout2,
                                                           flag, sweep_id, nst, cap, W);
}

// ---- launch geometry ---------------------------------------------------------
constexpr int64_t kSmemMax = 220 * 1024;  // per CTA (opt-in max 227 KB)

int sm_count() {  // of the current device (launches happen with the handle's device current)
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

inline int chunk_for_t(int maxw) { return maxw <= 4 ? 4 : (maxw <= 8 ? 8 : 16); }

struct Geo {
    int nst = 0;
    int64_t cap = 0;
    size_t smem = 0;
    int per_sm = 0;
};

// Stages per CTA: maximise resident consumer warps (capped at 32 per SM),
// then the pipeline depth.  Cached per kernel and stage size.
template <class K>
Geo geometry(K kernel, int np, int maxw, int eb = 12, int64_t win_bytes = 0) {
    static std::mutex mu;
    // keyed by device too: the shared-memory opt-in attribute is per device
    static std::map<std::tuple<int, const void *, int64_t>, Geo> cache;
    Geo g;
    g.cap = (int64_t)kTS * kSlice * std::max(maxw, 1);
    const int64_t stage = np * Layout::part_bytes(g.cap, eb) + win_bytes;
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    auto key = std::make_tuple(dev, (const void *)kernel, stage);
    auto itc = cache.find(key);
    if (itc != cache.end()) return itc->second;
    int best_warps = -1;
    // the attribute is per kernel and device (shared by all handles): allow
    // the maximum once per device; each launch passes its own dynamic size
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
    for (int nst = 1; nst <= 6; ++nst) {  // nst = 1: overlap comes from co-resident CTAs
        const int64_t smem = 128 + nst * stage;
        if (smem > kSmemMax) break;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreadsT, (size_t)smem);
        const int warps = std::min(per_sm * kTS, 32);
        if (per_sm > 0 && warps >= best_warps) {  // ties: deeper pipeline
            best_warps = warps;
            g.nst = nst;
            g.smem = (size_t)smem;
            g.per_sm = per_sm;
        }
    }
    cache[key] = g;
    return g;
}

template <class K>
int grid_of(const Geo &g, int64_t ntiles) {
    return (int)std::min<int64_t>(ntiles, (int64_t)sm_count() * std::max(g.per_sm, 1));
}

template <class K, class... Args>
cudaError_t launch_pdl(bool pdl, K kernel, int grid, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreadsT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Kernel view of a gather window; capacity = its largest tile window rounded
// up to 32 doubles (256 bytes).
WinView win_view(const Window *w) {
    if (!w) return WinView{};
    return WinView{w->tseg, w->glo, w->len, w->sbase, {w->wpos[0], w->wpos[1]}, (w->wmax + 31) / 32 * 32};
}

template <int OUT, int CH, bool OFS, bool WIN>
cudaError_t residual_tma_ofs(const Window *w, int64_t n, int64_t s_begin, int64_t s_end, const Sell &L, const Sell &U,
                             const double *d, const double *b, const double *x, double *out, double *out2,
                             bool pdl, cudaStream_t st) {
    auto k = WIN ? k_residual_tma_w<OUT, CH> : k_residual_tma<OUT, CH, OFS>;
    const WinView W = win_view(WIN ? w : nullptr);
    Geo g = geometry(k, 2, std::max(L.maxw, U.maxw), OFS ? 8 : 12, (int64_t)W.wcap * 8);
    if (!g.nst) return cudaErrorInvalidConfiguration;
    if (const char *v = knob("NSM_RES_NST")) {  // experiment: force the stage count (occupancy follows)
        const int nst = atoi(v);
        const int64_t stage = 2 * Layout::part_bytes(g.cap, OFS ? 8 : 12) + (int64_t)W.wcap * 8;
        g.nst = nst;
        g.smem = (size_t)(128 + nst * stage);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreadsT, g.smem);
        g.per_sm = per_sm;
    }
    const int64_t ntiles = (s_end - s_begin + kTS - 1) / kTS;
    return launch_pdl(pdl, k, grid_of<decltype(k)>(g, ntiles), g.smem, st, n, s_begin, s_end, view(L), view(U), d, b, x,
                      out, out2, g.nst, g.cap, W);
}

template <int OUT, int CH>
cudaError_t residual_tma_ch(const Window *w, int64_t n, int64_t s_begin, int64_t s_end, const Sell &L, const Sell &U,
                            const double *d, const double *b, const double *x, double *out, double *out2,
                            bool pdl, cudaStream_t st) {
    // offset-aligned layout (both triangles): stage values only, columns = row + offset;
    // with a gather window over the whole range: gathers from shared memory
    if (L.off && U.off && w && s_begin % kTS == 0)
        return residual_tma_ofs<OUT, CH, true, true>(w, n, s_begin, s_end, L, U, d, b, x, out, out2, pdl, st);
    if (L.off && U.off)
        return residual_tma_ofs<OUT, CH, true, false>(w, n, s_begin, s_end, L, U, d, b, x, out, out2, pdl, st);
    return residual_tma_ofs<OUT, CH, false, false>(w, n, s_begin, s_end, L, U, d, b, x, out, out2, pdl, st);
}

template <bool UNIT, int EPI, class G, int CH, bool OFS, bool WIN>
cudaError_t sweep_tma_ofs(const SweepArgs &a, int64_t s_begin, int64_t s_end, G gin, cudaStream_t st) {
    const WinView W = win_view(WIN ? a.win : nullptr);
    auto k = k_sweep_tma<UNIT, EPI, G, CH, OFS>;
    if constexpr (WIN) k = k_sweep_tma_w<UNIT, EPI, CH>;
    Geo g = geometry(k, 1, a.T->maxw, OFS ? 8 : 12, (int64_t)W.wcap * 8);
    if (!g.nst) return cudaErrorInvalidConfiguration;
    if (const char *v = knob("NSM_SWEEP_NST")) {  // experiment: force the stage count (occupancy follows)
        const int nst = atoi(v);
        const int64_t stage = Layout::part_bytes(g.cap, OFS ? 8 : 12) + (int64_t)W.wcap * 8;
        g.nst = nst;
        g.smem = (size_t)(128 + nst * stage);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreadsT, g.smem);
        g.per_sm = per_sm;
    }
    const int64_t ntiles = (s_end - s_begin + kTS - 1) / kTS;
    return launch_pdl(a.pdl, k, grid_of<decltype(k)>(g, ntiles), g.smem, st, a.n, s_begin, s_end, view(*a.T), a.dT, a.rhs,
                      gin, a.gout, a.x, a.dnext, a.gout2, a.flag, a.sweep_id, g.nst, g.cap, W);
}

template <bool UNIT, int EPI, class G, int CH>
cudaError_t sweep_tma_launch(const SweepArgs &a, int64_t s_begin, int64_t s_end, G gin, cudaStream_t st) {
    // offset-aligned layout: stage values only, columns = row + offset; with a
    // gather window of the plain iterate over the whole range: gathers from
    // shared memory
    if constexpr (std::is_same<G, GatherPlainT>::value) {
        // windowed sweeps over rows wider than 8 entries: the window sum in
        // chunks of 7 fits 56 registers, so four CTAs share an SM instead of
        // three at CH = 16 (C3 sweeps 0.95 -> 0.98 of peak, 1.384 -> 1.360 ms
        // per application; tools/experiments/README.md)
        if constexpr (CH == 16) {
            if (a.T->off && a.win && s_begin % kTS == 0)
                return sweep_tma_ofs<UNIT, EPI, G, 7, true, true>(a, s_begin, s_end, gin, st);
        }
        if (a.T->off && a.win && s_begin % kTS == 0)
            return sweep_tma_ofs<UNIT, EPI, G, CH, true, true>(a, s_begin, s_end, gin, st);
    }
    if (a.T->off) return sweep_tma_ofs<UNIT, EPI, G, CH, true, false>(a, s_begin, s_end, gin, st);
    return sweep_tma_ofs<UNIT, EPI, G, CH, false, false>(a, s_begin, s_end, gin, st);
}

template <bool UNIT, int EPI, int CH>
cudaError_t sweep_tma_g(const SweepArgs &a, int64_t s_begin, int64_t s_end, cudaStream_t st) {
    if constexpr (!UNIT) {
        if (a.gin_scaled)
            return sweep_tma_launch<UNIT, EPI, GatherScaledT, CH>(a, s_begin, s_end, GatherScaledT{a.rhs, a.dT}, st);
    }
    return sweep_tma_launch<UNIT, EPI, GatherPlainT, CH>(a, s_begin, s_end,
                                                          GatherPlainT{a.gin_scaled ? a.rhs : a.gin}, st);
}

template <bool UNIT, int EPI>
cudaError_t sweep_tma_epi(const SweepArgs &a, int64_t s_begin, int64_t s_end, cudaStream_t st) {
    switch (chunk_for_t(a.T->maxw)) {
        case 4: return sweep_tma_g<UNIT, EPI, 4>(a, s_begin, s_end, st);
        case 8: return sweep_tma_g<UNIT, EPI, 8>(a, s_begin, s_end, st);
        default: return sweep_tma_g<UNIT, EPI, 16>(a, s_begin, s_end, st);
    }
}

}  // namespace

// Shared memory of one stage must fit (two stages at least).
bool tma_ok(int np, int maxw) {
    const int64_t stage = np * (int64_t)kTS * kSlice * std::max(maxw, 1) * 12;
    return 128 + stage <= kSmemMax;
}

cudaError_t launch_residual_tma(const Window *w, int out_mode, int64_t n, int64_t s_begin, int64_t s_end, const Sell &L,
                                const Sell &U, const double *d, const double *b, const double *x, double *out,
                                double *out2, bool pdl, cudaStream_t st) {
    if (s_end <= s_begin) return cudaSuccess;
    const int ch = chunk_for_t(std::max(L.maxw, U.maxw));
    // windowed rows of 9..14 entries per triangle (27-point stencils: 13): a
    // 14-entry register chunk fits 72 registers, so three CTAs share an SM
    // instead of two at CH = 16 (C3 residual 0.93 -> 0.99 of the measured
    // peak in the step, 1.428 -> 1.383 ms per application)
    if (ch == 16 && std::max(L.maxw, U.maxw) <= 14 && L.off && U.off && w && s_begin % kTS == 0) {
        if (out_mode == OUT_AX)
            return residual_tma_ofs<OUT_AX, 14, true, true>(w, n, s_begin, s_end, L, U, d, b, x, out, out2, pdl, st);
        if (out_mode == OUT_RG)
            return residual_tma_ofs<OUT_RG, 14, true, true>(w, n, s_begin, s_end, L, U, d, b, x, out, out2, pdl, st);
        return residual_tma_ofs<OUT_R, 14, true, true>(w, n, s_begin, s_end, L, U, d, b, x, out, out2, pdl, st);
    }
#define NSM_RT(OUT)                                                                                  \
    (ch == 4 ? residual_tma_ch<OUT, 4>(w, n, s_begin, s_end, L, U, d, b, x, out, out2, pdl, st)           \
             : ch == 8 ? residual_tma_ch<OUT, 8>(w, n, s_begin, s_end, L, U, d, b, x, out, out2, pdl, st) \
                       : residual_tma_ch<OUT, 16>(w, n, s_begin, s_end, L, U, d, b, x, out, out2, pdl, st))
    return out_mode == OUT_AX ? NSM_RT(OUT_AX) : (out_mode == OUT_RG ? NSM_RT(OUT_RG) : NSM_RT(OUT_R));
#undef NSM_RT
}

cudaError_t launch_sweep_tma(const SweepArgs &a, int64_t s_begin, int64_t s_end, cudaStream_t st) {
    if (s_end <= s_begin) return cudaSuccess;
    if (a.unit) {
        switch (a.epi) {
            case EPI_STORE: return sweep_tma_epi<true, EPI_STORE>(a, s_begin, s_end, st);
            case EPI_XADD: return sweep_tma_epi<true, EPI_XADD>(a, s_begin, s_end, st);
            case EPI_STORE2: return sweep_tma_epi<true, EPI_STORE2>(a, s_begin, s_end, st);
            default: return sweep_tma_epi<true, EPI_XADD_SCALE>(a, s_begin, s_end, st);
        }
    }
    switch (a.epi) {
        case EPI_STORE: return sweep_tma_epi<false, EPI_STORE>(a, s_begin, s_end, st);
        case EPI_XADD: return sweep_tma_epi<false, EPI_XADD>(a, s_begin, s_end, st);
        case EPI_STORE2: return sweep_tma_epi<false, EPI_STORE2>(a, s_begin, s_end, st);
        default: return sweep_tma_epi<false, EPI_XADD_SCALE>(a, s_begin, s_end, st);
    }
}

// ---- eager loading (see kernels.cu) --------------------------------------------
namespace {
template <class K>
void touch_t(K k) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k);
}
template <int CH>
void touch_tma_win() {
    touch_t(k_residual_tma_w<OUT_R, CH>);
    touch_t(k_residual_tma_w<OUT_AX, CH>);
    touch_t(k_residual_tma_w<OUT_RG, CH>);
    touch_t(k_sweep_tma_w<true, EPI_STORE2, CH>);
    touch_t(k_sweep_tma_w<false, EPI_STORE2, CH>);
    touch_t(k_sweep_tma_w<true, EPI_STORE, CH>);
    touch_t(k_sweep_tma_w<true, EPI_XADD, CH>);
    touch_t(k_sweep_tma_w<true, EPI_XADD_SCALE, CH>);
    touch_t(k_sweep_tma_w<false, EPI_STORE, CH>);
    touch_t(k_sweep_tma_w<false, EPI_XADD, CH>);
    touch_t(k_sweep_tma_w<false, EPI_XADD_SCALE, CH>);
}
template <int CH, bool OFS>
void touch_tma_ch() {
    touch_t(k_residual_tma<OUT_R, CH, OFS>);
    touch_t(k_residual_tma<OUT_AX, CH, OFS>);
    touch_t(k_residual_tma<OUT_RG, CH, OFS>);
    touch_t(k_sweep_tma<true, EPI_STORE2, GatherPlainT, CH, OFS>);
    touch_t(k_sweep_tma<false, EPI_STORE2, GatherPlainT, CH, OFS>);
    touch_t(k_sweep_tma<false, EPI_STORE2, GatherScaledT, CH, OFS>);
    touch_t(k_sweep_tma<true, EPI_STORE, GatherPlainT, CH, OFS>);
    touch_t(k_sweep_tma<true, EPI_XADD, GatherPlainT, CH, OFS>);
    touch_t(k_sweep_tma<true, EPI_XADD_SCALE, GatherPlainT, CH, OFS>);
    touch_t(k_sweep_tma<false, EPI_STORE, GatherPlainT, CH, OFS>);
    touch_t(k_sweep_tma<false, EPI_XADD, GatherPlainT, CH, OFS>);
    touch_t(k_sweep_tma<false, EPI_XADD_SCALE, GatherPlainT, CH, OFS>);
    touch_t(k_sweep_tma<false, EPI_STORE, GatherScaledT, CH, OFS>);
    touch_t(k_sweep_tma<false, EPI_XADD, GatherScaledT, CH, OFS>);
    touch_t(k_sweep_tma<false, EPI_XADD_SCALE, GatherScaledT, CH, OFS>);
}
}  // namespace

void preload_tma_kernels() {
    touch_t(k_sweep_tma_w<true, EPI_STORE2, 7>);   // the chunk-7 windowed sweeps
    touch_t(k_sweep_tma_w<false, EPI_STORE2, 7>);
    touch_t(k_sweep_tma_w<true, EPI_STORE, 7>);
    touch_t(k_sweep_tma_w<true, EPI_XADD, 7>);
    touch_t(k_sweep_tma_w<true, EPI_XADD_SCALE, 7>);
    touch_t(k_sweep_tma_w<false, EPI_STORE, 7>);
    touch_t(k_sweep_tma_w<false, EPI_XADD, 7>);
    touch_t(k_sweep_tma_w<false, EPI_XADD_SCALE, 7>);
    touch_t(k_residual_tma_w<OUT_R, 14>);
    touch_t(k_residual_tma_w<OUT_AX, 14>);
    touch_t(k_residual_tma_w<OUT_RG, 14>);
    touch_tma_ch<4, false>();
    touch_tma_ch<8, false>();
    touch_tma_ch<16, false>();
    touch_tma_ch<4, true>();
    touch_tma_ch<8, true>();
    touch_tma_ch<16, true>();
    touch_tma_win<4>();
    touch_tma_win<8>();
    touch_tma_win<16>();
}

}  // namespace nsm
