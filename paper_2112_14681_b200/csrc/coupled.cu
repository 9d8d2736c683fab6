// coupled.cu — one forward pGS application (residual, k Jacobi sweeps, x
// update; the pGS application of P:L743-785 with g(0) = D^{-1} r,
// eq:jr-initial-guess) as CONCURRENT WARP GROUPS of one persistent kernel,
// so the matrix rows the sweeps re-read come from L2 instead of HBM
// (DESIGN.md §6 "Coupled passes").
//
// The per-pass schedule (stream.cu) reads L three times from HBM for k = 2:
// once in the residual, once per sweep.  Here every CTA (one per SM) holds
// k + 1 warp groups, each an instance of the per-pass pipeline — a producer
// warp staging tiles by bulk copy (values, window positions, slice header,
// gather window) and consumer warps with one row per thread:
//
//   group 0      8 consumer warps   r = b - A x, g(0) = r / d         tile t
//   group j      4 consumer warps   g(j) = (r - L g(j-1)) / d         tile t - lag_j
//   (j = 1..k)   (two slices each)  the last one x += g(k)
//
// All groups walk the same tiles (t = CTA, CTA + G, ...), so tile t's L values
// are streamed from HBM by group 0 and re-read shortly after by groups 1..k
// of the same CTA while they are still in L2 (group 0 copies L with the
// evict_normal policy, U and the last sweep's L with evict_first).
//
// Dependencies (256-row tiles; "phase q done through t" = every CTA's group q
// has completed all of its tiles <= t, read from per-CTA progress counters
// like fused_w.cu's frontiers):
//   group j >= 1, tile t:  phase j-1 done through t       (its gather window
//                          of g(j-1) covers rows below and inside tile t; r of
//                          tile t follows by causality)
//   group k, tile t:       phase 0 done through t + DA     (x of tile t: every
//                          residual window reading it has been consumed)
//   group 0, tile t:       phase k done through t - lag    (throttle: keeps the
//                          L rows group 0 streamed L2-resident until re-read)
// Each condition refers to tiles strictly earlier in the chain (lag > DA), so
// the lowest unfinished tile can always proceed; a cooperative launch makes
// all CTAs resident, so the kernel is deadlock-free.  A wait longer than the
// handle's timeout sets the error word (nsm_check: NSM_ERR_DIST) instead of
// hanging.
//
// Arithmetic: the consumers run the per-pass kernels' code on the same staged
// operands — the same products and stored-order additions, the same division
// — so results are bit-identical to the per-pass path and to the oracle.
// The r rows a sweep needs are bulk-copied into its stage by the producer
// (after the dependency wait), never read through L1.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <map>
#include <mutex>
#include <tuple>

#include "nsm_internal.h"
#include "ptx.cuh"
#include "stream_dev.cuh"

namespace nsm {

namespace {

constexpr int kRW = kTS;      // residual consumer warps: one slice each
constexpr int kSW = 4;        // consumer warps per sweep group: slices w and w + 4
constexpr int kMaxK = 2;
constexpr int kPubBytes = 256;  // per-group, per-stage publication counters
constexpr int64_t kSmemMaxC = 227 * 1024;
template <int K>
constexpr int threads_c() { return (kRW + K * kSW + K + 1) * 32; }

struct CoupledParams {
    int64_t n, nslices, ntiles;
    SellView L, U;
    WinView WR, WL;              // residual window (L and U), sweep window (L)
    const double *d, *b;
    double *x, *r;
    double *g[kMaxK];            // g[j] = g(j), j = 0 .. k-1
    unsigned long long *prog;    // [k + 1][pstride] per-CTA progress (epoch << 32 | tiles done)
    int64_t pstride;
    unsigned int *sync;          // [0] epoch, [1] CTAs finished
    unsigned long long *flag;
    int64_t sweep_id0;
    unsigned int *err;
    unsigned long long timeout_ns;
    int64_t DA, lag;
    int nst_r, nst_s;
    int64_t cap_r, cap_s, goff_s;   // goff_s: bytes from group 1's base to group 2's
};

__device__ __forceinline__ unsigned int *pubc(char *sm, int g, int st) { return (unsigned int *)sm + g * 8 + st; }

// frontier of one phase: all tiles < F are complete (acquire reads of the
// per-CTA progress counters, refreshed only when a wait needs more)
__device__ __forceinline__ void need(const CoupledParams &p, int64_t &F, bool &dirty, int q, int64_t t,
                                     unsigned int epoch, int lane) {
    t = min(t, p.ntiles - 1);
    if (t < F) return;
    const int64_t G = gridDim.x;
    const unsigned long long *pr = p.prog + (int64_t)q * p.pstride;
    const uint64_t t0 = ptx::globaltimer_ns();
    while (true) {
        int64_t f = INT64_MAX;
        for (int64_t c = lane; c < G; c += 32) {
            const unsigned long long v = ptx::ld_acquire_gpu_u64(pr + c);
            const int64_t cnt = (unsigned int)(v >> 32) == epoch ? (int64_t)(v & 0xffffffffull) : 0;
            f = min(f, c + cnt * G);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) f = min(f, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)f, o));
        F = max(F, f);
        if (t < F) break;
        if (ptx::globaltimer_ns() - t0 > p.timeout_ns) {
            if (lane == 0) atomicOr(p.err, 2u);
            F = INT64_MAX;
            break;
        }
        __nanosleep(128);
    }
    dirty = true;
}

// Producer hooks (stream_dev.cuh): dependency waits before a tile is staged,
// then a proxy fence (the bulk copies read vectors other SMs wrote through
// the generic proxy); sweeps also stage the tile's r rows.
template <int K>
struct CoupledHook {
    const CoupledParams *p;
    int g;                 // 0: residual, j >= 1: sweep j
    unsigned int epoch;
    double *rslot0;        // sweeps: r rows of stage 0 (256 doubles per stage)
    int64_t Fa, Fb;        // frontiers: Fa of the phase this group waits on (k for group 0, g - 1 for
                           // group g), Fb of phase 0 (group k)
    bool dirty;
    uint64_t pol_keep, pol_first;
    __device__ __forceinline__ int64_t first() const { return blockIdx.x; }
    __device__ __forceinline__ int64_t stride() const { return gridDim.x; }
    __device__ __forceinline__ int64_t rows(int64_t t) const { return min((int64_t)kTS * kSlice, p->n - t * kTS * kSlice); }
    __device__ __forceinline__ void before(int64_t t, int st, int lane) {
        if (g == 0) {
            if (t - p->lag >= 0) need(*p, Fa, dirty, K, t - p->lag, epoch, lane);
        } else {
            need(*p, Fa, dirty, g - 1, t, epoch, lane);
            if (g == K) need(*p, Fb, dirty, 0, t + p->DA, epoch, lane);
        }
        if (dirty) {
            __syncwarp();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            dirty = false;
        }
        if (g > 0 && lane == 0) {
            const int64_t m = rows(t);
            if (m & 1) rslot0[st * kTS * kSlice + m - 1] = __ldcg(p->r + t * kTS * kSlice + m - 1);  // odd n: last row
        }
    }
    __device__ __forceinline__ uint32_t extra_bytes(int64_t t) const {
        return g > 0 ? (uint32_t)((rows(t) & ~(int64_t)1) * 8) : 0u;
    }
    __device__ __forceinline__ void extra_copy(int64_t t, int st, uint64_t *bar) const {
        const uint32_t bytes = extra_bytes(t);
        if (bytes) ptx::bulk_g2s(rslot0 + st * kTS * kSlice, p->r + t * kTS * kSlice, bytes, bar, pol_keep);
    }
    __device__ __forceinline__ uint64_t val_policy(int part, uint64_t) const {
        if (g == 0) return part == 0 ? pol_keep : pol_first;  // L is re-read by the sweeps, U is not
        return g == K ? pol_first : pol_keep;
    }
};

// publish "this CTA's group g has completed its tiles 0..m" once every
// consumer warp of the group has counted tile m (CTA-scope acq_rel count,
// then a gpu-scope release); the stage is released after the count, so no
// warp counts the stage's next tile before every warp has counted this one
__device__ __forceinline__ void publish_and_release(const CoupledParams &p, char *sm, int g, int st, int nwarps,
                                                    uint64_t *empty, int64_t m, unsigned int epoch, int lane) {
    __syncwarp();
    if (lane == 0) {
        const unsigned int prev = ptx::atom_add_acqrel_cta_shared(pubc(sm, g, st), 1u);
        if ((prev + 1) % (unsigned)nwarps == 0)
            ptx::red_max_release_gpu_u64(p.prog + (int64_t)g * p.pstride + blockIdx.x,
                                         ((unsigned long long)epoch << 32) | (unsigned long long)(m + 1));
        ptx::mbar_arrive(empty);
    }
}

template <int CH, int K>
__global__ void __launch_bounds__(threads_c<K>(), 1) k_pgs_coupled(const __grid_constant__ CoupledParams p) {
    extern __shared__ __align__(128) char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned int epoch = *(volatile unsigned int *)&p.sync[0];
    // group bases: [0, 256) publication counters, then group 0, group 1, group 2
    const Layout LyR{p.nst_r, 2, p.cap_r, 8, (int64_t)p.WR.wcap};
    const Layout LyS{p.nst_s, 1, p.cap_s, 8, (int64_t)p.WL.wcap};
    char *gb0 = sm + kPubBytes;
    char *gb1 = gb0 + 128 + (int64_t)p.nst_r * (2 * Layout::part_bytes(p.cap_r, 8) + (int64_t)p.WR.wcap * 8);
    auto gbase = [&](int g) { return g == 0 ? gb0 : gb1 + (int64_t)(g - 1) * p.goff_s; };
    // sweeps: r rows after the stages' windows
    auto rslot = [&](int g) { return LyS.win(gbase(g), 0) + (int64_t)p.nst_s * p.WL.wcap; };
    if (threadIdx.x == 0) {
        for (int st = 0; st < p.nst_r; ++st) {
            ptx::mbar_init(LyR.full(gb0) + st, 1);
            ptx::mbar_init(LyR.empty(gb0) + st, kRW);
        }
        for (int g = 1; g <= K; ++g)
            for (int st = 0; st < p.nst_s; ++st) {
                ptx::mbar_init(LyS.full(gbase(g)) + st, 1);
                ptx::mbar_init(LyS.empty(gbase(g)) + st, kSW);
            }
        for (int q = 0; q < kPubBytes / 4; ++q) ((unsigned int *)sm)[q] = 0;
        ptx::mbar_init_fence();
    }
    __syncthreads();
    const int64_t ntiles = p.ntiles, G = gridDim.x, c = blockIdx.x;
    constexpr int kProd0 = kRW + K * kSW;

    if (warp >= kProd0) {
        // ------------------------------------------------------------ producers
        const int g = warp - kProd0;
        CoupledHook<K> hk;
        hk.p = &p;
        hk.g = g;
        hk.epoch = epoch;
        hk.rslot0 = g > 0 ? rslot(g) : nullptr;
        hk.Fa = hk.Fb = 0;
        hk.dirty = false;
        hk.pol_keep = ptx::policy_evict_normal();
        hk.pol_first = ptx::policy_evict_first();
        if (g == 0) {
            const SellView P[2] = {p.L, p.U};
            producer<2, true, CoupledHook<K>>(LyR, gb0, P, 0, p.nslices, ntiles, lane, p.WR, p.x, p.n, hk);
        } else {
            const SellView P[1] = {p.L};
            producer<1, true, CoupledHook<K>>(LyS, gbase(g), P, 0, p.nslices, ntiles, lane, p.WL, p.g[g - 1], p.n, hk);
        }
    } else if (warp < kRW) {
        // ------------------------------------ group 0: r = b - A x, g(0) = r / d
        int st = 0;
        uint32_t ph = 0;
        for (int64_t t = c, m = 0; t < ntiles; t += G, ++m) {
            const int64_t s = t * kTS + warp;
            const bool has = s < p.nslices;
            const int64_t i = s * kSlice + lane;
            const bool row = has && i < p.n;
            // own-row vectors: immutable (d, b), or x of tile t, which group k
            // rewrites only after this tile is published
            const double di = row ? __ldg(p.d + i) : 0.0, xi = row ? __ldg(p.x + i) : 0.0;
            const double bi = row ? __ldg(p.b + i) : 0.0;
            ptx::mbar_wait(LyR.full(gb0) + st, ph);
            double acc = 0.0;
            if (has) {
                const int2 hl = *(const int2 *)(LyR.hdr(gb0, st, 0) + 2 * warp);
                const int2 hu = *(const int2 *)(LyR.hdr(gb0, st, 1) + 2 * warp);
                const double *ws = LyR.win(gb0, st);
                if constexpr (CH <= 8) {
                    WinChunk<CH> cl, cu;
                    cl.load(LyR.val(gb0, st, 0), LyR.col(gb0, st, 0), ws, hl.x, hl.y, lane, row);
                    cu.load(LyR.val(gb0, st, 1), LyR.col(gb0, st, 1), ws, hu.x, hu.y, lane, row);
                    acc = cl.add(acc);
                    acc = __dadd_rn(acc, __dmul_rn(di, xi));
                    acc = cu.add(acc);
                } else {
                    WinChunk<CH> cw;
                    cw.load(LyR.val(gb0, st, 0), LyR.col(gb0, st, 0), ws, hl.x, hl.y, lane, row);
                    acc = cw.add(acc);
                    acc = __dadd_rn(acc, __dmul_rn(di, xi));
                    cw.load(LyR.val(gb0, st, 1), LyR.col(gb0, st, 1), ws, hu.x, hu.y, lane, row);
                    acc = cw.add(acc);
                }
            }
            if (row) {
                const double r = __dsub_rn(bi, acc);
                p.r[i] = r;
                p.g[0][i] = __ddiv_rn(r, di);
            }
            publish_and_release(p, sm, 0, st, kRW, LyR.empty(gb0) + st, m, epoch, lane);
            if (++st == p.nst_r) { st = 0; ph ^= 1; }
        }
    } else {
        // -------------------- group j: g(j) = (r - L g(j-1)) / d; j = k: x += g(k)
        const int g = 1 + (warp - kRW) / kSW, wl = (warp - kRW) % kSW;
        char *gb = gbase(g);
        const double *rs0 = rslot(g);
        double *gout = g < K ? p.g[g] : nullptr;
        const unsigned long long sid = (unsigned long long)(p.sweep_id0 + g - 1);
        int st = 0;
        uint32_t ph = 0;
        for (int64_t t = c, m = 0; t < ntiles; t += G, ++m) {
            double di[2], xi[2], v[2];
            bool row[2], has[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t s = t * kTS + wl + h * kSW;
                const int64_t i = s * kSlice + lane;
                has[h] = s < p.nslices;
                row[h] = has[h] && i < p.n;
                di[h] = row[h] ? __ldg(p.d + i) : 1.0;
                xi[h] = (g == K && row[h]) ? p.x[i] : 0.0;  // x of tile t: written only by this group, below
            }
            ptx::mbar_wait(LyS.full(gb) + st, ph);
            const double *ws = LyS.win(gb, st);
            const double *rs = rs0 + st * kTS * kSlice;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int sl = wl + h * kSW;
                double acc = 0.0;
                if (has[h]) {
                    const int2 hd = *(const int2 *)(LyS.hdr(gb, st, 0) + 2 * sl);
                    WinChunk<CH> ct;
                    ct.load(LyS.val(gb, st, 0), LyS.col(gb, st, 0), ws, hd.x, hd.y, lane, row[h]);
                    acc = ct.add(acc);
                }
                const double ri = row[h] ? rs[sl * kSlice + lane] : 0.0;
                v[h] = __ddiv_rn(__dsub_rn(ri, acc), di[h]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (!row[h]) continue;
                const int64_t i = (t * kTS + wl + h * kSW) * kSlice + lane;
                if (!isfinite(v[h])) atomicMin(p.flag, sid);
                if (g < K) gout[i] = v[h];
                else p.x[i] = __dadd_rn(xi[h], v[h]);
            }
            publish_and_release(p, sm, g, st, kSW, LyS.empty(gb) + st, m, epoch, lane);
            if (++st == p.nst_s) { st = 0; ph ^= 1; }
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

WinView wview(const Window *w) {
    return WinView{w->tseg, w->glo, w->len, w->sbase, {w->wpos[0], w->wpos[1]}, (w->wmax + 31) / 32 * 32};
}

template <int CH, int K>
const void *kernel_of() { return (const void *)k_pgs_coupled<CH, K>; }

const void *coupled_kernel(int ch, int k) {
    if (ch <= 8) return k == 1 ? kernel_of<8, 1>() : kernel_of<8, 2>();
    return k == 1 ? kernel_of<16, 1>() : kernel_of<16, 2>();
}
int coupled_threads(int k) { return k == 1 ? threads_c<1>() : threads_c<2>(); }

}  // namespace

CoupledShape coupled_shape(int maxw_a, int maxw_l, int64_t wcap_r, int64_t wcap_s, int k, int64_t n) {
    CoupledShape sh;
    if (k < 1 || k > kMaxK || n <= 0 || maxw_a > 16 || maxw_l > 16) return sh;
    const int ch = maxw_a <= 8 ? 8 : 16;
    sh.cap_r = (int64_t)kTS * kSlice * std::max(maxw_a, 1);
    sh.cap_s = (int64_t)kTS * kSlice * std::max(maxw_l, 1);
    wcap_r = (wcap_r + 31) / 32 * 32;
    wcap_s = (wcap_s + 31) / 32 * 32;
    const int64_t stage_r = 2 * Layout::part_bytes(sh.cap_r, 8) + wcap_r * 8;
    const int64_t stage_s = Layout::part_bytes(sh.cap_s, 8) + wcap_s * 8 + (int64_t)kTS * kSlice * 8;
    // deepest residual pipeline first (it streams from HBM), then the sweeps'
    for (int nr = 3; nr >= 1 && !sh.ok; --nr)
        for (int ns = 3; ns >= 1 && !sh.ok; --ns) {
            const int64_t goff = 128 + ns * stage_s;
            const int64_t smem = kPubBytes + 128 + nr * stage_r + k * goff;
            if (smem <= kSmemMaxC) {
                sh.ok = true;
                sh.nst_r = nr;
                sh.nst_s = ns;
                sh.goff_s = goff;
                sh.smem = (size_t)smem;
            }
        }
    if (!sh.ok) return sh;
    sh.kernel = coupled_kernel(ch, k);
    sh.threads = coupled_threads(k);
    sh.wcap_r = wcap_r;
    sh.wcap_s = wcap_s;
    return sh;
}

cudaError_t launch_coupled(const CoupledLaunch &L, cudaStream_t st) {
    const CoupledShape &sh = L.shape;
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, int> per_sm;  // device, kernel
    int dev = 0;
    cudaGetDevice(&dev);
    int occ = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto key = std::make_pair(dev, sh.kernel);
        auto it = per_sm.find(key);
        if (it == per_sm.end()) {
            cudaFuncSetAttribute(sh.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMaxC);
            it = per_sm.emplace(key, -1).first;
        }
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sh.kernel, sh.threads, sh.smem);
        if (e != cudaSuccess) return e;
    }
    if (occ < 1) return cudaErrorInvalidConfiguration;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ntiles = (L.n + kTS * kSlice - 1) / (kTS * kSlice);
    const int grid = (int)std::min<int64_t>({(int64_t)nsm, ntiles, L.pstride});
    CoupledParams p{};
    p.n = L.n;
    p.nslices = (L.n + kSlice - 1) / kSlice;
    p.ntiles = ntiles;
    p.L = view(*L.Lp);
    p.U = view(*L.Up);
    p.WR = wview(L.wr);
    p.WL = wview(L.wl);
    p.WR.wcap = (int32_t)sh.wcap_r;
    p.WL.wcap = (int32_t)sh.wcap_s;
    p.d = L.d;
    p.b = L.b;
    p.x = L.x;
    p.r = L.r;
    p.g[0] = L.g0;
    p.g[1] = L.g1;
    p.prog = L.prog;
    p.pstride = L.pstride;
    p.sync = L.sync;
    p.flag = L.flag;
    p.sweep_id0 = L.sweep_id0;
    p.err = L.err;
    p.timeout_ns = L.timeout_ns;
    p.DA = L.DA;
    // throttle distance: the dependency distance plus a few rounds of tiles
    p.lag = L.lag > 0 ? std::max<int64_t>(L.lag, L.DA + 1) : L.DA + 1 + 4 * (int64_t)grid;
    p.nst_r = sh.nst_r;
    p.nst_s = sh.nst_s;
    p.cap_r = sh.cap_r;
    p.cap_s = sh.cap_s;
    p.goff_s = sh.goff_s;
    void *args[] = {&p};
    return cudaLaunchCooperativeKernel(sh.kernel, dim3((unsigned)grid), dim3((unsigned)sh.threads), args, sh.smem, st);
}

void preload_coupled_kernels() {
    cudaFuncAttributes a;
    for (int ch : {8, 16})
        for (int k = 1; k <= kMaxK; ++k) cudaFuncGetAttributes(&a, coupled_kernel(ch, k));
}

}  // namespace nsm
