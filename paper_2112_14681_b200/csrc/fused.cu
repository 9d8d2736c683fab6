// fused.cu — one-pass ("wavefront") polynomial Gauss-Seidel application
// (DESIGN.md §6 "Fused wavefront kernel").
//
// One launch computes  r = b - A x,  g^(0) = D^{-1} r,  k sweeps
// g^(j) = D^{-1}(r - L g^(j-1))  and  x <- x + g^(k) while
// reading the split matrix ONCE from HBM: tile t (256 rows) runs all k+1
// phases back to back with its L and U slices held in shared memory (one
// bulk copy), r and D in registers, and the inner iterates g^(j) published to
// small L2-resident ring buffers.  Phase j of tile t needs g^(j-1) of the
// rows within the lower bandwidth, i.e. of tiles [t - DL, t], so tiles are
// dispatched IN ORDER to a persistent grid (atomic tile counter) and a tile
// waits only for LOWER tiles' progress flags — the standard argument of
// decoupled look-back: the lowest unfinished tile always progresses, so
// there is no deadlock.
//
// The new x of tile t cannot overwrite the old x while tiles up to t + DL
// (whose residual reads it through L) or from t - DU (through U) have not
// finished phase 0.  It goes to a ring buffer, and the CTA that processes
// tile t + DL + 1 writes it back after checking those (lower) tiles' flags;
// the last DL + 1 tiles are written back by a small tail kernel.
//
// Every row is summed in the same order with the same IEEE operations as
// the per-pass kernels and the oracle: the result is bit-identical.
// All spin-waits are bounded (NSM_OPT_HALO_TIMEOUT_MS); a timeout sets an
// error flag reported by nsm_check (NSM_ERR_DIST) instead of hanging.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "nsm_internal.h"
#include "ptx.cuh"

namespace nsm {

namespace {

constexpr int kTSF = 8;                     // slices (consumer warps) per tile
constexpr int kRowsF = kTSF * kSlice;       // 256 rows per tile
constexpr int kThreadsF = (kTSF + 1) * 32;  // + 1 producer warp
constexpr int kConsumers = kTSF * 32;

struct FusedParams {
    int64_t n, nslices, ntiles;
    SellView L, U;
    const double *d, *b;
    double *x;
    int k;
    int DL, DU;              // dependency distances in tiles
    int64_t M;               // ring length in tiles
    double *ring;            // k + 1 rings of M * 256 doubles: g^(0..k-1), new x
    unsigned int *counter;   // tile dispenser
    int *prog;               // [ntiles]: number of finished phases of the tile
    int *wb;                 // [ntiles]: new x written back
    unsigned long long *flag;
    int64_t sweep_id0;
    unsigned int *err;
    unsigned long long timeout_ns;
    int nst;
    int64_t capL, capU;      // staged entries per stage per part
};

struct FLayout {
    int nst;
    int64_t capL, capU;
    __device__ __forceinline__ uint64_t *full(char *s) const { return (uint64_t *)s; }
    __device__ __forceinline__ uint64_t *empty(char *s) const { return (uint64_t *)s + nst; }
    __device__ __forceinline__ int *tile_id(char *s) const { return (int *)(s + 16 * nst); }
    __device__ __forceinline__ char *stage(char *s, int st) const {
        return s + 256 + (int64_t)st * (capL + capU) * 12;
    }
    __device__ __forceinline__ double *lval(char *s, int st) const { return (double *)stage(s, st); }
    __device__ __forceinline__ int32_t *lcol(char *s, int st) const { return (int32_t *)(stage(s, st) + capL * 8); }
    __device__ __forceinline__ double *uval(char *s, int st) const { return (double *)(stage(s, st) + capL * 12); }
    __device__ __forceinline__ int32_t *ucol(char *s, int st) const {
        return (int32_t *)(stage(s, st) + capL * 12 + capU * 8);
    }
};

// Warp-wide: wait until flags[v] >= need for every v in [lo, hi] (clamped to
// [0, ...]).  Loads are issued in batches so one check costs about one L2
// round trip; acquire ordering by a fence afterwards.  Bounded by a timeout.
__device__ __forceinline__ void wait_flags(const int *flags, int64_t lo, int64_t hi, int need, const FusedParams &p,
                                           int lane) {
    lo = lo < 0 ? 0 : lo;
    if (hi < lo) return;
    const uint64_t t0 = ptx::globaltimer_ns();
    for (int64_t base = lo; base <= hi; base += 32 * 8) {
        while (true) {
            int mn = INT_MAX;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t v = base + (int64_t)u * 32 + lane;
                if (v <= hi) mn = min(mn, __ldcv(flags + v));
            }
            if (__all_sync(0xffffffffu, mn >= need)) break;
            if (ptx::globaltimer_ns() - t0 > p.timeout_ns) {
                if (lane == 0) atomicOr(p.err, 2u);
                return;
            }
            __nanosleep(100);
        }
    }
    __threadfence();
}

__device__ __forceinline__ double *ring_at(const FusedParams &p, int which, int64_t tile) {
    return p.ring + ((int64_t)which * p.M + tile % p.M) * kRowsF;
}

template <int CH>
struct FChunk {
    double v[CH];
    int32_t c[CH];
    const double *sv;
    const int32_t *sc;
    int w;
    __device__ __forceinline__ void load(const double *sv_, const int32_t *sc_, int64_t off, int w_, int lane) {
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
};

// sum of v_j * g(c_j) over the row, in stored order (products first)
template <int CH, class G>
__device__ __forceinline__ double row_sum(const double *sv, const int32_t *sc, int64_t off, int w, int lane,
                                          const G &g, double acc) {
    FChunk<CH> ch;
    ch.load(sv, sc, off, w, lane);
#pragma unroll
    for (int j = 0; j < CH; ++j)
        if (j < w) ch.v[j] = __dmul_rn(ch.v[j], g(ch.c[j]));
#pragma unroll
    for (int j = 0; j < CH; ++j)
        if (j < w) acc = __dadd_rn(acc, ch.v[j]);
    for (int j = CH; j < w; ++j) acc = __dadd_rn(acc, __dmul_rn(ch.sv[j * kSlice], g(ch.sc[j * kSlice])));
    return acc;
}

template <int CH>
__global__ void __launch_bounds__(kThreadsF, 2) k_pgs_fused(FusedParams p) {
    extern __shared__ __align__(128) char sm[];
    const FLayout Ly{p.nst, p.capL, p.capU};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int st = 0; st < p.nst; ++st) {
            ptx::mbar_init(Ly.full(sm) + st, 1);
            ptx::mbar_init(Ly.empty(sm) + st, kTSF);
        }
        ptx::mbar_init_fence();
    }
    __syncthreads();

    if (warp == kTSF) {  // ---- producer: claim tiles in order, stream their L and U slices
        if (lane != 0) return;
        const uint64_t pol = ptx::policy_evict_first();
        for (int it = 0;; ++it) {
            const int st = it % p.nst;
            const uint32_t use = (uint32_t)(it / p.nst);
            if (it >= p.nst) ptx::mbar_wait(Ly.empty(sm) + st, (use - 1) & 1);
            const int64_t t = atomicAdd(p.counter, 1u);
            Ly.tile_id(sm)[st] = (int)t;
            if (t >= p.ntiles) {
                ptx::mbar_arrive(Ly.full(sm) + st);
                return;
            }
            const int64_t s0 = t * kTSF, s1 = min(s0 + kTSF, p.nslices);
            const int64_t lb = __ldg(p.L.ptr + s0), le = __ldg(p.L.ptr + s1);
            const int64_t ub = __ldg(p.U.ptr + s0), ue = __ldg(p.U.ptr + s1);
            ptx::mbar_expect_tx(Ly.full(sm) + st, (uint32_t)((le - lb + ue - ub) * 12));
            if (le > lb) {
                ptx::bulk_g2s(Ly.lval(sm, st), p.L.val + lb, (uint32_t)((le - lb) * 8), Ly.full(sm) + st, pol);
                ptx::bulk_g2s(Ly.lcol(sm, st), p.L.col + lb, (uint32_t)((le - lb) * 4), Ly.full(sm) + st, pol);
            }
            if (ue > ub) {
                ptx::bulk_g2s(Ly.uval(sm, st), p.U.val + ub, (uint32_t)((ue - ub) * 8), Ly.full(sm) + st, pol);
                ptx::bulk_g2s(Ly.ucol(sm, st), p.U.col + ub, (uint32_t)((ue - ub) * 4), Ly.full(sm) + st, pol);
            }
        }
    }

    // ---- consumers: one slice (32 rows) per warp, one row per thread
    for (int it = 0;; ++it) {
        const int st = it % p.nst;
        const uint32_t use = (uint32_t)(it / p.nst);
        ptx::mbar_wait(Ly.full(sm) + st, use & 1);
        const int64_t t = Ly.tile_id(sm)[st];
        if (t >= p.ntiles) return;
        const int64_t s0 = t * kTSF, s = s0 + warp;
        const bool has = s < p.nslices;
        const int64_t i = s * kSlice + lane;
        const bool row = has && i < p.n;
        const double di = row ? __ldg(p.d + i) : 1.0;
        const double bi = row ? __ldg(p.b + i) : 0.0;
        const double xi = row ? __ldg(p.x + i) : 0.0;
        int64_t lo = 0, uo = 0;
        int lw = 0, uw = 0;
        if (has) {
            const int64_t l0 = __ldg(p.L.ptr + s0), ls = __ldg(p.L.ptr + s), ls1 = __ldg(p.L.ptr + s + 1);
            const int64_t u0 = __ldg(p.U.ptr + s0), us = __ldg(p.U.ptr + s), us1 = __ldg(p.U.ptr + s + 1);
            lo = ls - l0;
            lw = (int)((ls1 - ls) / kSlice);
            uo = us - u0;
            uw = (int)((us1 - us) / kSlice);
        }
        // ring slots of tile t may be reused once tile t - M is fully done
        // and written back (tiles below t: no deadlock)
        if (warp == 0 && t >= p.M) {
            wait_flags(p.prog, t - p.M, t - p.M + p.DL, p.k + 1, p, lane);
            wait_flags(p.wb, t - p.M, t - p.M, 1, p, lane);
        }
        // phase 0: residual r = b - A x (x is the input: its overwrite is deferred)
        const double *lv = Ly.lval(sm, st), *uv = Ly.uval(sm, st);
        const int32_t *lc = Ly.lcol(sm, st), *uc = Ly.ucol(sm, st);
        const double *x = p.x;
        auto gx = [x](int32_t c) { return __ldg(x + c); };
        double acc = 0.0;
        if (has) {
            acc = row_sum<CH>(lv, lc, lo, lw, lane, gx, acc);
            acc = __dadd_rn(acc, __dmul_rn(di, xi));
            acc = row_sum<CH>(uv, uc, uo, uw, lane, gx, acc);
        }
        const double ri = __dsub_rn(bi, acc);
        double g = __ddiv_rn(ri, di);
        if (row && !isfinite(g)) atomicMin(p.flag, (unsigned long long)p.sweep_id0);
        ptx::bar_sync(1, kConsumers);  // ring-reuse wait (warp 0) done; U slices no longer needed
        if (row) ring_at(p, 0, t)[i - t * kRowsF] = g;
        for (int ph = 1; ph <= p.k; ++ph) {
            ptx::bar_sync(1, kConsumers);
            if (threadIdx.x == 0) {
                __threadfence();
                ptx::st_release_gpu(p.prog + t, ph);  // phase ph-1 of tile t done
            }
            if (warp == 0) wait_flags(p.prog, t - p.DL, t - 1, ph, p, lane);
            ptx::bar_sync(1, kConsumers);
            const double *gp = p.ring + (int64_t)(ph - 1) * p.M * kRowsF;
            const int64_t M = p.M;
            auto gg = [gp, M](int32_t c) {
                const int64_t tc = c / kRowsF;
                return __ldcg(gp + (tc % M) * kRowsF + (c - tc * kRowsF));
            };
            double a2 = 0.0;
            if (has) a2 = row_sum<CH>(lv, lc, lo, lw, lane, gg, a2);
            g = __ddiv_rn(__dsub_rn(ri, a2), di);
            if (row && !isfinite(g)) atomicMin(p.flag, (unsigned long long)(p.sweep_id0 + ph));
            if (ph < p.k) {
                if (row) ring_at(p, ph, t)[i - t * kRowsF] = g;
            } else if (row) {
                ring_at(p, p.k, t)[i - t * kRowsF] = __dadd_rn(xi, g);  // new x, written back later
            }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(Ly.empty(sm) + st);  // L/U slices consumed
        ptx::bar_sync(1, kConsumers);
        if (threadIdx.x == 0) {
            __threadfence();
            ptx::st_release_gpu(p.prog + t, p.k + 1);
        }
        // deferred write-back of tile w = t - DL - 1: every tile reading old
        // x[w] in its residual (w - DU .. w + DL = t - 1) has finished phase 0
        const int64_t w = t - p.DL - 1;
        if (w >= 0) {
            if (warp == 0) {
                wait_flags(p.prog, w - p.DU, t - 1, 1, p, lane);
                wait_flags(p.prog, w, w, p.k + 1, p, lane);
            }
            ptx::bar_sync(1, kConsumers);
            const int64_t iw = w * kRowsF + threadIdx.x;
            if (iw < p.n) p.x[iw] = __ldcg(ring_at(p, p.k, w) + threadIdx.x);
            ptx::bar_sync(1, kConsumers);
            if (threadIdx.x == 0) {
                __threadfence();
                ptx::st_release_gpu(p.wb + w, 1);
            }
        }
    }
}

// write back the new x of the last tiles (nobody above them to do it)
__global__ void k_fused_tail(int64_t n, int64_t w0, int64_t ntiles, int64_t M, const double *xring, double *x) {
    const int64_t i = w0 * kRowsF + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || i >= ntiles * kRowsF) return;
    const int64_t tl = i / kRowsF;
    x[i] = xring[(tl % M) * kRowsF + (i - tl * kRowsF)];
}

template <int CH>
cudaError_t fused_launch(const FusedParams &p, size_t smem, int grid, cudaStream_t st) {
    k_pgs_fused<CH><<<grid, kThreadsF, smem, st>>>(p);
    return cudaGetLastError();
}

int occupancy_fused(int ch, size_t smem) {
    int per = 0;
    auto f = [&](auto k) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kThreadsF, smem);
    };
    if (ch == 4) f(k_pgs_fused<4>);
    else if (ch == 8) f(k_pgs_fused<8>);
    else f(k_pgs_fused<16>);
    return per;
}

}  // namespace

// ---- host side -----------------------------------------------------------------
int fused_tile_rows() { return kRowsF; }

size_t fused_smem(int maxwL, int maxwU, int nst) {
    const int64_t capL = (int64_t)kRowsF * std::max(maxwL, 1), capU = (int64_t)kRowsF * std::max(maxwU, 1);
    return 256 + (size_t)nst * (capL + capU) * 12;
}

bool fused_ok(int maxwL, int maxwU) { return fused_smem(maxwL, maxwU, 2) <= 220 * 1024; }

// Grid size (resident CTAs) for the persistent launch.
int fused_grid(int maxwL, int maxwU) {
    const int ch = std::max(maxwL, maxwU) <= 4 ? 4 : (std::max(maxwL, maxwU) <= 8 ? 8 : 16);
    const size_t smem = fused_smem(maxwL, maxwU, 2);
    int per = std::max(occupancy_fused(ch, smem), 1);
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms * per;
}

cudaError_t launch_pgs_fused(const FusedLaunch &f, cudaStream_t st) {
    FusedParams p{};
    p.n = f.n;
    p.nslices = (f.n + kSlice - 1) / kSlice;
    p.ntiles = (f.n + kRowsF - 1) / kRowsF;
    if (p.ntiles == 0) return cudaSuccess;
    p.L = view(*f.L);
    p.U = view(*f.U);
    p.d = f.d;
    p.b = f.b;
    p.x = f.x;
    p.k = f.k;
    p.DL = f.DL;
    p.DU = f.DU;
    p.M = f.M;
    p.ring = f.ring;
    p.counter = f.sync;
    p.prog = (int *)(f.sync + 64);
    p.wb = p.prog + p.ntiles;
    p.flag = f.flag;
    p.sweep_id0 = f.sweep_id0;
    p.err = f.err;
    p.timeout_ns = f.timeout_ns;
    p.nst = 2;
    if (const char *e = getenv("NSM_FUSED_NST")) p.nst = std::max(1, atoi(e));  // DEBUG experiment
    p.capL = (int64_t)kRowsF * std::max(f.L->maxw, 1);
    p.capU = (int64_t)kRowsF * std::max(f.U->maxw, 1);
    // reset the dispenser and the progress flags
    cudaError_t e = cudaMemsetAsync(f.sync, 0, (64 + 2 * (size_t)p.ntiles) * sizeof(int), st);
    if (e != cudaSuccess) return e;
    const size_t smem = fused_smem(f.L->maxw, f.U->maxw, p.nst);
    int grid = (int)std::min<int64_t>(f.grid, p.ntiles);
    if (const char *e = getenv("NSM_FUSED_GRID_DIV")) grid = std::max(1, grid / std::max(1, atoi(e)));  // DEBUG
    const int mw = std::max(f.L->maxw, f.U->maxw);
    e = mw <= 4 ? fused_launch<4>(p, smem, grid, st)
                : (mw <= 8 ? fused_launch<8>(p, smem, grid, st) : fused_launch<16>(p, smem, grid, st));
    if (e != cudaSuccess) return e;
    const int64_t w0 = std::max<int64_t>(0, p.ntiles - p.DL - 1);
    const int64_t rows = std::min<int64_t>(f.n - w0 * kRowsF, (p.ntiles - w0) * kRowsF);
    if (rows > 0)
        k_fused_tail<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(f.n, w0, p.ntiles, p.M,
                                                                     f.ring + (int64_t)p.k * p.M * kRowsF, f.x);
    return cudaGetLastError();
}

void preload_fused_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_pgs_fused<4>);
    cudaFuncGetAttributes(&a, k_pgs_fused<8>);
    cudaFuncGetAttributes(&a, k_pgs_fused<16>);
    cudaFuncGetAttributes(&a, k_fused_tail);
}

}  // namespace nsm
