// kernels.cu — sm_100a kernels of the Neumann-series smoothers
// (DESIGN.md §6 "Kernels").
//
// The hot path is a streaming sparse gather-reduce in fp64 (≈0.17 flop/B): it
// is HBM-bound, so there is no tensor-core work (tcgen05/TMEM do not apply).
// What matters is moving the SELL-32 value/index streams at full HBM
// bandwidth (coalesced 256 B / 128 B warp loads, no L1 allocation, L2
// evict-first), keeping the small gathered vectors (x, r, g, d) in L1/L2, and
// enough independent loads in flight per thread.
//
// Numerics: one thread owns one row and accumulates its sum sequentially in
// ascending column order with explicit round-to-nearest multiply and add
// (no FMA contraction), and D^{-1} is an IEEE division — the exact rounding
// sequence of the oracle (reading R10), so GPU and oracle agree
// bit for bit on the same inputs.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "nsm_internal.h"

namespace nsm {

namespace {

constexpr int kThreads = 256;                 // 8 warps = 8 slices per CTA
constexpr int kSlicesPerCta = kThreads / kSlice;

// ---- memory access helpers -------------------------------------------------
// Matrix streams are read exactly once per pass: no L1 allocation, and mark
// them evict-first in L2 so they do not push out the gathered vectors.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_stream(const double *a, uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t *a, uint64_t pol) {
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}

// Gather source of a sweep: either a stored iterate g[c], or (for the first
// sweep, eq:jr-initial-guess g^(0) = D^{-1} r) the scaled right-hand side
// rhs[c] / d[c] recomputed on the fly, which saves writing and re-reading g^(0).
struct GatherPlain {
    const double *__restrict__ g;
    __device__ __forceinline__ double operator()(int32_t c) const { return __ldg(g + c); }
};
struct GatherScaled {
    const double *__restrict__ rhs;
    const double *__restrict__ d;
    __device__ __forceinline__ double operator()(int32_t c) const { return __ddiv_rn(__ldg(rhs + c), __ldg(d + c)); }
};

// acc += sum over the slice-s entries of this lane's row, in stored order
// (= ascending columns).  Entries past the row's length are padding (val 0).
template <class G>
__device__ __forceinline__ double accum(const SellView P, int64_t s, int lane, const G &gather, double acc,
                                        uint64_t pol) {
    const int64_t b = __ldg(P.ptr + s) + lane, e = __ldg(P.ptr + s + 1);
#pragma unroll 4
    for (int64_t p = b; p < e; p += kSlice) {
        const double v = ld_stream(P.val + p, pol);
        const int32_t c = ld_stream(P.col + p, pol);
        acc = __dadd_rn(acc, __dmul_rn(v, gather(c)));
    }
    return acc;
}

// Register-blocked form of accum for the hot loops: the first CH entries of
// the row are loaded by CH independent, predicated loads issued back to back
// (memory-level parallelism: all value/index requests of a row are in
// flight together), multiplied by their gathered operands as they arrive,
// then summed in stored order.  Entries beyond CH (rows wider than the
// chunk: coarse AMG levels) follow in further chunks of CH — their gathers
// again issued together, their products again added one by one in stored
// order — so the summation order (and every rounding) is unchanged.
template <int CH>
struct Chunk {
    double v[CH];
    int32_t c[CH];
    int w;
    int64_t base;
    __device__ __forceinline__ void load(const SellView P, int64_t s, int lane, uint64_t pol) {
        const int64_t b = __ldg(P.ptr + s), e = __ldg(P.ptr + s + 1);
        w = (int)((e - b) / kSlice);
        base = b + lane;
#pragma unroll
        for (int j = 0; j < CH; ++j) {
            if (j < w) {
                v[j] = ld_stream(P.val + base + (int64_t)j * kSlice, pol);
                c[j] = ld_stream(P.col + base + (int64_t)j * kSlice, pol);
            }
        }
    }
    template <class G>
    __device__ __forceinline__ void gather_mul(const G &g) {
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) v[j] = __dmul_rn(v[j], g(c[j]));
    }
    template <class G>
    __device__ __forceinline__ double add(double acc, const SellView P, const G &g, uint64_t pol) const {
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j < w) acc = __dadd_rn(acc, v[j]);
        for (int j0 = CH; j0 < w; j0 += CH) {
            double pr[CH];
#pragma unroll
            for (int t = 0; t < CH; ++t)
                if (j0 + t < w) {
                    const int64_t p = base + (int64_t)(j0 + t) * kSlice;
                    pr[t] = __dmul_rn(ld_stream(P.val + p, pol), g(ld_stream(P.col + p, pol)));
                }
#pragma unroll
            for (int t = 0; t < CH; ++t)
                if (j0 + t < w) acc = __dadd_rn(acc, pr[t]);
        }
        return acc;
    }
};

__device__ __forceinline__ void flag_nonfinite(double v, unsigned long long *flag, int64_t sweep_id) {
    if (!isfinite(v)) atomicMin(flag, (unsigned long long)sweep_id);
}

__device__ __forceinline__ bool slice_of(int nslices, const int32_t *list, int64_t *s, int *lane) {
    const int64_t w = (int64_t)blockIdx.x * kSlicesPerCta + (threadIdx.x >> 5);
    if (w >= nslices) return false;
    *s = list ? (int64_t)list[w] : w;
    *lane = threadIdx.x & 31;
    return true;
}

// Programmatic dependent launch (launches with pdl = true): a kernel may be
// scheduled while its predecessor drains; it waits for the predecessor's
// completion (and memory) before touching ANY memory, then lets its own
// dependents be scheduled.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

// ---- residual / SpMV (row a2) ------------------------------------------------
// acc_i = sum_{j ascending} a_ij x_j over LG (ghosts below), L, D, U, UG
// (ghosts above); then  OUT_R: r = b - acc;  OUT_AX: y = acc;  OUT_RG: r and
// g^(0) = r / d (eq:jr-initial-guess) so the first sweep gathers g^(0)
// instead of recomputing one division per gathered entry.

template <int OUT, int CH>
__global__ void __launch_bounds__(kThreads) k_residual(int64_t n, int nslices, const int32_t *__restrict__ list,
                                                       SellView LG, SellView L, SellView U, SellView UG, int has_ghost,
                                                       const double *__restrict__ d, const double *__restrict__ b,
                                                       const double *__restrict__ x, const double *__restrict__ ghost,
                                                       double *__restrict__ out, double *__restrict__ out2) {
    pdl_enter();
    int64_t s;
    int lane;
    if (!slice_of(nslices, list, &s, &lane)) return;
    const uint64_t pol = policy_evict_first();
    const int64_t i = s * kSlice + lane;
    const bool row = i < n;
    const GatherPlain gx{x};
    // issue every independent load of the row first
    Chunk<CH> cl, cu;
    cl.load(L, s, lane, pol);
    cu.load(U, s, lane, pol);
    const double di = row ? __ldg(d + i) : 0.0, xi = row ? __ldg(x + i) : 0.0;
    const double bi = (OUT != OUT_AX && row) ? __ldg(b + i) : 0.0;
    cl.gather_mul(gx);
    cu.gather_mul(gx);
    // then sum in ascending column order: LG, L, D, U, UG
    double acc = 0.0;
    if (has_ghost) acc = accum(LG, s, lane, GatherPlain{ghost}, acc, pol);
    acc = cl.add(acc, L, gx, pol);
    acc = __dadd_rn(acc, __dmul_rn(di, xi));
    acc = cu.add(acc, U, gx, pol);
    if (has_ghost) acc = accum(UG, s, lane, GatherPlain{ghost}, acc, pol);
    if (!row) return;
    if (OUT == OUT_AX) {
        out[i] = acc;
    } else {
        const double r = __dsub_rn(bi, acc);
        out[i] = r;
        if (OUT == OUT_RG) out2[i] = __ddiv_rn(r, di);
    }
}

// ---- inner Jacobi sweep (rows a3, a4, a5) -----------------------------------
//   v_i = (rhs_i - sum_{j in T(i)} t_ij gin_j) / dT_i      (UNIT: no division)
// eq:jacobi for pGS (T = L, dT = D); the unit-lower ILU factor
// (G_L = I - L) and the row-scaled U factor (G_U = I - D_U^{-1}U,
// P:L829) with the same kernel.  Epilogues:
//   EPI_STORE      gout_i = v
//   EPI_XADD       x_i += v                     (last sweep)
//   EPI_STORE2     gout_i = v ; gout2_i = v / dnext_i   (last L sweep of ILU:
//                  y and the U-solve start z^(0) = D_U^{-1} y in one pass)
//   EPI_XADD_SCALE x_i += v / dnext_i            (ILU with k_u = 0)

template <bool UNIT, int EPI, class G, int CH>
__global__ void __launch_bounds__(kThreads) k_sweep(int64_t n, int nslices, const int32_t *__restrict__ list,
                                                    SellView T, SellView TG, int has_ghost,
                                                    const double *__restrict__ dT, const double *__restrict__ rhs,
                                                    G gin, const double *__restrict__ ghost,
                                                    double *__restrict__ gout, double *__restrict__ x,
                                                    const double *__restrict__ dnext, double *__restrict__ gout2,
                                                    unsigned long long *flag, int64_t sweep_id) {
    pdl_enter();
    int64_t s;
    int lane;
    if (!slice_of(nslices, list, &s, &lane)) return;
    const uint64_t pol = policy_evict_first();
    const int64_t i = s * kSlice + lane;
    const bool row = i < n;
    Chunk<CH> ct;
    ct.load(T, s, lane, pol);
    const double ri = row ? __ldg(rhs + i) : 0.0;
    const double di = (!UNIT && row) ? __ldg(dT + i) : 1.0;
    const double xi = ((EPI == EPI_XADD || EPI == EPI_XADD_SCALE) && row) ? x[i] : 0.0;
    const double dn = ((EPI == EPI_STORE2 || EPI == EPI_XADD_SCALE) && row) ? __ldg(dnext + i) : 1.0;
    ct.gather_mul(gin);
    double acc = 0.0;
    // ghost couplings lie below the block for a lower triangle (has_ghost 1)
    // and above it for an upper one (2): keep the ascending column order
    if (has_ghost == 1) acc = accum(TG, s, lane, GatherPlain{ghost}, acc, pol);
    acc = ct.add(acc, T, gin, pol);
    if (has_ghost == 2) acc = accum(TG, s, lane, GatherPlain{ghost}, acc, pol);
    if (!row) return;
    double v = __dsub_rn(ri, acc);
    if (!UNIT) v = __ddiv_rn(v, di);
    flag_nonfinite(v, flag, sweep_id);
    if (EPI == EPI_STORE) gout[i] = v;
    if (EPI == EPI_XADD) x[i] = __dadd_rn(xi, v);
    if (EPI == EPI_STORE2) { gout[i] = v; gout2[i] = __ddiv_rn(v, dn); }
    if (EPI == EPI_XADD_SCALE) x[i] = __dadd_rn(xi, __ddiv_rn(v, dn));
}

// ---- wide rows (coarse AMG levels): one warp per row --------------------------
// Galerkin rows have 50-100+ entries while the levels are small (a few to a
// few hundred slices), so one thread per row leaves the SMs idle and each
// thread walks a long dependent chain.  Here the 32 lanes form the products of
// 32 consecutive entries of ONE row at once (their gathers in flight
// together) and every lane then adds them in stored order through shuffles —
// the same sequence of IEEE operations as the thread-per-row kernels, so the
// results are bit-identical.  Padding entries (val 0) take part exactly as
// there.
template <class G>
__device__ __forceinline__ double accum_row_warp(const SellView P, int64_t s, int rr, int lane, const G &g,
                                                 double acc) {
    const int64_t b = __ldg(P.ptr + s), e = __ldg(P.ptr + s + 1);
    const int w = (int)((e - b) / kSlice);
    for (int j0 = 0; j0 < w; j0 += 32) {
        const int j = j0 + lane;
        double pr = 0.0;
        if (j < w) {
            const int64_t p = b + (int64_t)j * kSlice + rr;
            pr = __dmul_rn(__ldg(P.val + p), g(__ldg(P.col + p)));
        }
        const int m = min(32, w - j0);
        for (int t = 0; t < m; ++t) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, pr, t));
    }
    return acc;
}

__device__ __forceinline__ bool row_of(int nslices, const int32_t *list, int64_t *s, int *rr) {
    const int64_t gw = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    if (gw >= (int64_t)nslices * kSlice) return false;
    const int64_t k = gw / kSlice;
    *s = list ? (int64_t)list[k] : k;
    *rr = (int)(gw - k * kSlice);
    return true;
}

template <int OUT>
__global__ void __launch_bounds__(kThreads) k_residual_wide(int64_t n, int nslices, const int32_t *__restrict__ list,
                                                            SellView LG, SellView L, SellView U, SellView UG,
                                                            int has_ghost, const double *__restrict__ d,
                                                            const double *__restrict__ b,
                                                            const double *__restrict__ x,
                                                            const double *__restrict__ ghost,
                                                            double *__restrict__ out, double *__restrict__ out2) {
    pdl_enter();
    int64_t s;
    int rr;
    if (!row_of(nslices, list, &s, &rr)) return;
    const int lane = threadIdx.x & 31;
    const int64_t i = s * kSlice + rr;
    if (i >= n) return;  // whole warp
    const GatherPlain gx{x};
    double acc = 0.0;
    if (has_ghost) acc = accum_row_warp(LG, s, rr, lane, GatherPlain{ghost}, acc);
    acc = accum_row_warp(L, s, rr, lane, gx, acc);
    const double di = __ldg(d + i);
    acc = __dadd_rn(acc, __dmul_rn(di, __ldg(x + i)));
    acc = accum_row_warp(U, s, rr, lane, gx, acc);
    if (has_ghost) acc = accum_row_warp(UG, s, rr, lane, GatherPlain{ghost}, acc);
    if (lane != 0) return;
    if (OUT == OUT_AX) {
        out[i] = acc;
    } else {
        const double r = __dsub_rn(__ldg(b + i), acc);
        out[i] = r;
        if (OUT == OUT_RG) out2[i] = __ddiv_rn(r, di);
    }
}

template <bool UNIT, int EPI, class G>
__global__ void __launch_bounds__(kThreads) k_sweep_wide(int64_t n, int nslices, const int32_t *__restrict__ list,
                                                         SellView T, SellView TG, int has_ghost,
                                                         const double *__restrict__ dT,
                                                         const double *__restrict__ rhs, G gin,
                                                         const double *__restrict__ ghost, double *__restrict__ gout,
                                                         double *__restrict__ x, const double *__restrict__ dnext,
                                                         double *__restrict__ gout2, unsigned long long *flag,
                                                         int64_t sweep_id) {
    pdl_enter();
    int64_t s;
    int rr;
    if (!row_of(nslices, list, &s, &rr)) return;
    const int lane = threadIdx.x & 31;
    const int64_t i = s * kSlice + rr;
    if (i >= n) return;
    double acc = 0.0;
    if (has_ghost == 1) acc = accum_row_warp(TG, s, rr, lane, GatherPlain{ghost}, acc);
    acc = accum_row_warp(T, s, rr, lane, gin, acc);
    if (has_ghost == 2) acc = accum_row_warp(TG, s, rr, lane, GatherPlain{ghost}, acc);
    if (lane != 0) return;
    double v = __dsub_rn(__ldg(rhs + i), acc);
    if (!UNIT) v = __ddiv_rn(v, __ldg(dT + i));
    flag_nonfinite(v, flag, sweep_id);
    if (EPI == EPI_STORE) gout[i] = v;
    if (EPI == EPI_XADD) x[i] = __dadd_rn(x[i], v);
    if (EPI == EPI_STORE2) { gout[i] = v; gout2[i] = __ddiv_rn(v, __ldg(dnext + i)); }
    if (EPI == EPI_XADD_SCALE) x[i] = __dadd_rn(x[i], __ddiv_rn(v, __ldg(dnext + i)));
}

inline unsigned grid_wide(int nslices) {
    return (unsigned)(((int64_t)nslices * kSlice + (kThreads / 32) - 1) / (kThreads / 32));
}

// ---- diagonal scaling:  out = rhs / d  or  x += rhs / d  (k = 0 cases) -------
template <bool XADD>
__global__ void __launch_bounds__(kThreads) k_scale(int64_t n, const double *__restrict__ rhs,
                                                    const double *__restrict__ d, double *__restrict__ out,
                                                    unsigned long long *flag, int64_t sweep_id) {
    pdl_enter();
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (i >= n) return;
    const double v = d ? __ddiv_rn(__ldg(rhs + i), __ldg(d + i)) : __ldg(rhs + i);
    flag_nonfinite(v, flag, sweep_id);
    out[i] = XADD ? __dadd_rn(out[i], v) : v;
}

inline unsigned grid_for(int nslices) { return (unsigned)((nslices + kSlicesPerCta - 1) / kSlicesPerCta); }

template <class K, class... Args>
void launch_k(bool pdl, K kernel, unsigned grid, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace

// ---------------------------------------------------------------- launchers --
// Rows wider than 24 entries on a small level (<= 4096 rows: too few slices
// to fill the GPU one thread per row): warp per row.
bool wide_rows(int maxw, int64_t nslices) { return maxw > 24 && nslices * kSlice <= 4096; }

// Register chunk CH: the smallest of 4 / 8 / 16 covering the widest slice
// (wider rows continue in the plain loop).
static inline int chunk_for(int maxw) { return maxw <= 4 ? 4 : (maxw <= 8 ? 8 : 16); }

template <int OUT, int CH>
static void residual_ch(int64_t n, int nslices, const int32_t *list, const Sell &LG, const Sell &L, const Sell &U,
                        const Sell &UG, bool has_ghost, const double *d, const double *b, const double *x,
                        const double *ghost, double *out, double *out2, bool pdl, cudaStream_t st) {
    launch_k(pdl, k_residual<OUT, CH>, grid_for(nslices), st, n, nslices, list, view(LG), view(L), view(U),
             view(UG), (int)has_ghost, d, b, x, ghost, out, out2);
}

cudaError_t launch_residual(int out_mode, int64_t n, int nslices, const int32_t *list, const Sell &LG,
                            const Sell &L, const Sell &U, const Sell &UG, bool has_ghost, const double *d,
                            const double *b, const double *x, const double *ghost, double *out, double *out2,
                            bool pdl, cudaStream_t st) {
    if (nslices <= 0) return cudaSuccess;
    if (wide_rows(std::max(L.maxw, U.maxw), nslices)) {
        const SellView lg = view(LG), l = view(L), u = view(U), ug = view(UG);
        const int hg = has_ghost;
        if (out_mode == OUT_AX)
            launch_k(pdl, k_residual_wide<OUT_AX>, grid_wide(nslices), st, n, nslices, list, lg, l, u, ug, hg, d, b, x, ghost, out, out2);
        else if (out_mode == OUT_RG)
            launch_k(pdl, k_residual_wide<OUT_RG>, grid_wide(nslices), st, n, nslices, list, lg, l, u, ug, hg, d, b, x, ghost, out, out2);
        else
            launch_k(pdl, k_residual_wide<OUT_R>, grid_wide(nslices), st, n, nslices, list, lg, l, u, ug, hg, d, b, x, ghost, out, out2);
        return cudaGetLastError();
    }
    const int ch = chunk_for(std::max(L.maxw, U.maxw));
#define NSM_RES(OUT)                                                                                              \
    (ch == 4 ? residual_ch<OUT, 4>(n, nslices, list, LG, L, U, UG, has_ghost, d, b, x, ghost, out, out2, pdl, st)      \
             : ch == 8 ? residual_ch<OUT, 8>(n, nslices, list, LG, L, U, UG, has_ghost, d, b, x, ghost, out, out2, pdl, st) \
                       : residual_ch<OUT, 16>(n, nslices, list, LG, L, U, UG, has_ghost, d, b, x, ghost, out, out2, pdl, st))
    if (out_mode == OUT_AX) NSM_RES(OUT_AX);
    else if (out_mode == OUT_RG) NSM_RES(OUT_RG);
    else NSM_RES(OUT_R);
#undef NSM_RES
    return cudaGetLastError();
}

template <bool UNIT, int EPI, int CH>
static void sweep_ch(const SweepArgs &a, cudaStream_t st) {
    dim3 g(grid_for(a.nslices));
    SellView TG = a.TG ? view(*a.TG) : SellView{nullptr, nullptr, nullptr};
    if constexpr (!UNIT) {
        if (a.gin_scaled) {
            launch_k(a.pdl, k_sweep<UNIT, EPI, GatherScaled, CH>, g.x, st,
                a.n, a.nslices, a.list, view(*a.T), TG, a.has_ghost, a.dT, a.rhs, GatherScaled{a.rhs, a.dT}, a.ghost,
                a.gout, a.x, a.dnext, a.gout2, a.flag, a.sweep_id);
            return;
        }
    }
    // unit diagonal: g^(0) = rhs itself
    launch_k(a.pdl, k_sweep<UNIT, EPI, GatherPlain, CH>, g.x, st,
        a.n, a.nslices, a.list, view(*a.T), TG, a.has_ghost, a.dT, a.rhs, GatherPlain{a.gin_scaled ? a.rhs : a.gin},
        a.ghost, a.gout, a.x, a.dnext, a.gout2, a.flag, a.sweep_id);
}

template <bool UNIT, int EPI>
static void sweep_wide(const SweepArgs &a, cudaStream_t st) {
    const dim3 g(grid_wide(a.nslices));
    const SellView TG = a.TG ? view(*a.TG) : SellView{nullptr, nullptr, nullptr};
    if constexpr (!UNIT) {
        if (a.gin_scaled) {
            launch_k(a.pdl, k_sweep_wide<UNIT, EPI, GatherScaled>, g.x, st,
                a.n, a.nslices, a.list, view(*a.T), TG, a.has_ghost, a.dT, a.rhs, GatherScaled{a.rhs, a.dT}, a.ghost,
                a.gout, a.x, a.dnext, a.gout2, a.flag, a.sweep_id);
            return;
        }
    }
    launch_k(a.pdl, k_sweep_wide<UNIT, EPI, GatherPlain>, g.x, st,
        a.n, a.nslices, a.list, view(*a.T), TG, a.has_ghost, a.dT, a.rhs, GatherPlain{a.gin_scaled ? a.rhs : a.gin},
        a.ghost, a.gout, a.x, a.dnext, a.gout2, a.flag, a.sweep_id);
}

template <bool UNIT, int EPI>
static void sweep_epi(const SweepArgs &a, cudaStream_t st) {
    if (wide_rows(a.T->maxw, a.nslices)) {
        sweep_wide<UNIT, EPI>(a, st);
        return;
    }
    switch (chunk_for(a.T->maxw)) {
        case 4: sweep_ch<UNIT, EPI, 4>(a, st); break;
        case 8: sweep_ch<UNIT, EPI, 8>(a, st); break;
        default: sweep_ch<UNIT, EPI, 16>(a, st); break;
    }
}

template <bool UNIT>
static void sweep_unit(const SweepArgs &a, cudaStream_t st) {
    switch (a.epi) {
        case EPI_STORE: sweep_epi<UNIT, EPI_STORE>(a, st); break;
        case EPI_XADD: sweep_epi<UNIT, EPI_XADD>(a, st); break;
        case EPI_STORE2: sweep_epi<UNIT, EPI_STORE2>(a, st); break;
        default: sweep_epi<UNIT, EPI_XADD_SCALE>(a, st); break;
    }
}

cudaError_t launch_sweep(const SweepArgs &a, cudaStream_t st) {
    if (a.nslices <= 0) return cudaSuccess;
    if (a.unit) sweep_unit<true>(a, st);
    else sweep_unit<false>(a, st);
    return cudaGetLastError();
}

cudaError_t launch_scale(bool xadd, int64_t n, const double *rhs, const double *d, double *out,
                         unsigned long long *flag, int64_t sweep_id, bool pdl, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    unsigned g = (unsigned)((n + kThreads - 1) / kThreads);
    if (xadd) launch_k(pdl, k_scale<true>, g, st, n, rhs, d, out, flag, sweep_id);
    else launch_k(pdl, k_scale<false>, g, st, n, rhs, d, out, flag, sweep_id);
    return cudaGetLastError();
}

}  // namespace nsm

// ---- eager loading ------------------------------------------------------------
// CUDA loads kernels lazily on first launch, and a lazy load may wait for the
// device to go idle.  A halo-wait kernel spinning on a neighbour's flag while
// the host launches a not-yet-loaded kernel would then stall until the wait
// times out, so multi-rank handles load every kernel up front.
namespace nsm {
namespace {
template <class K>
void touch(K k) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k);
}
void touch_wide() {
    touch(k_residual_wide<OUT_R>);
    touch(k_residual_wide<OUT_AX>);
    touch(k_residual_wide<OUT_RG>);
    touch(k_sweep_wide<true, EPI_STORE, GatherPlain>);
    touch(k_sweep_wide<true, EPI_XADD, GatherPlain>);
    touch(k_sweep_wide<true, EPI_XADD_SCALE, GatherPlain>);
    touch(k_sweep_wide<true, EPI_STORE2, GatherPlain>);
    touch(k_sweep_wide<false, EPI_STORE2, GatherPlain>);
    touch(k_sweep_wide<false, EPI_STORE2, GatherScaled>);
    touch(k_sweep_wide<false, EPI_STORE, GatherPlain>);
    touch(k_sweep_wide<false, EPI_XADD, GatherPlain>);
    touch(k_sweep_wide<false, EPI_XADD_SCALE, GatherPlain>);
    touch(k_sweep_wide<false, EPI_STORE, GatherScaled>);
    touch(k_sweep_wide<false, EPI_XADD, GatherScaled>);
    touch(k_sweep_wide<false, EPI_XADD_SCALE, GatherScaled>);
}
template <int CH>
void touch_ch() {
    touch(k_residual<OUT_R, CH>);
    touch(k_residual<OUT_AX, CH>);
    touch(k_residual<OUT_RG, CH>);
    touch(k_sweep<true, EPI_STORE, GatherPlain, CH>);
    touch(k_sweep<true, EPI_XADD, GatherPlain, CH>);
    touch(k_sweep<true, EPI_XADD_SCALE, GatherPlain, CH>);
    touch(k_sweep<true, EPI_STORE2, GatherPlain, CH>);
    touch(k_sweep<false, EPI_STORE2, GatherPlain, CH>);
    touch(k_sweep<false, EPI_STORE2, GatherScaled, CH>);
    touch(k_sweep<false, EPI_STORE, GatherPlain, CH>);
    touch(k_sweep<false, EPI_XADD, GatherPlain, CH>);
    touch(k_sweep<false, EPI_XADD_SCALE, GatherPlain, CH>);
    touch(k_sweep<false, EPI_STORE, GatherScaled, CH>);
    touch(k_sweep<false, EPI_XADD, GatherScaled, CH>);
    touch(k_sweep<false, EPI_XADD_SCALE, GatherScaled, CH>);
}
}  // namespace

void preload_plain_kernels() {
    touch_wide();
    touch_ch<4>();
    touch_ch<8>();
    touch_ch<16>();
    touch(k_scale<true>);
    touch(k_scale<false>);
}
}  // namespace nsm
