// pair.cu — the two Jacobi sweeps of a forward pGS application with k = 2
// (eq:jacobi; the second fused with x += g(2)) in ONE persistent
// cooperative kernel in which every CTA runs BOTH sweeps on its own tiles,
// keeping each tile's staged L values in shared memory between the two
// (DESIGN.md §6 "Paired sweeps").  L is read from HBM once per application.
//
// The residual pass runs before it (k_residual_tma_w: r and g(0) = r / d).
// CTA c owns tiles t_m = c + m G.  Iteration m of a CTA:
//   sweep 1 on t_m:      g(1) = (r - L g(0)) / d       (L, r, window of g(0): ring slot m mod 2)
//   sweep 2 on t_{m-1}:  x += (r - L g(1)) / d         (L, r from ring slot (m-1) mod 2, window of g(1))
// Sweep 2 of tile t needs g(1) of the rows its L couples to (rows <= t's last
// row), i.e. sweep 1 done through t by every CTA: per-CTA progress counters
// as in coupled.cu (the last consumer warp of a tile publishes it), read by
// the producer before it stages the g(1) window (acquire, proxy fence).  A CTA
// is at most one iteration ahead in sweep 2 of the slowest CTA's sweep 1, so
// the lowest unfinished step can always proceed (cooperative launch: all CTAs
// resident; a wait longer than the handle's timeout sets the error word).
//
// Shared memory per CTA: two ring slots (L values, window positions, slice
// header, r rows, the g(0) window, segment metadata) and two g(1) window
// buffers, about 100 KB for 27-point rows: two CTAs per SM.
//
// Arithmetic: the per-pass sweep's products and stored-order additions on the
// same staged operands, the same division: bit-identical.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <map>
#include <mutex>

#include "nsm_internal.h"
#include "ptx.cuh"
#include "stream_dev.cuh"

namespace nsm {

namespace {

constexpr int kPW = kTS;                     // consumer warps
constexpr int kThreadsP = (kPW + 1) * 32;    // + producer
constexpr int kSlotsP = 4;                   // publication count slots
constexpr int kPVp = 10;                     // frontier counters per lane (<= 320 CTAs)
constexpr int64_t kSmemMaxP = 227 * 1024;
constexpr int kRowsT = kTS * kSlice;

struct PairParams {
    int64_t n, nslices, ntiles;
    SellView L;
    WinView W;                 // L's gather window
    const double *d, *r, *g0;
    double *g1, *x;
    unsigned int *prog;        // per-CTA progress of sweep 1: tag | tiles done
    unsigned int *sync;        // [0] epoch, [1] CTAs finished
    unsigned long long *flag;
    int64_t sweep_id0;
    unsigned int *err;
    unsigned long long timeout_ns;
    int64_t cap, wcap;         // entries per tile part, window doubles
    int64_t slot_bytes;
};

__device__ __forceinline__ unsigned int ptag(unsigned int epoch) { return (epoch & 0x7ffu) << 21; }

// ring slot layout: values | positions | header | r rows | window A | segment metadata (32 x int4 + count)
struct Slot {
    char *base;
    int64_t cap, wcap;
    __device__ __forceinline__ double *val() const { return (double *)base; }
    __device__ __forceinline__ int32_t *pos() const { return (int32_t *)(base + cap * 8); }
    __device__ __forceinline__ int32_t *hdr() const { return (int32_t *)(base + cap * 8 + Layout::ofs_bytes(cap)); }
    __device__ __forceinline__ double *rrow() const { return (double *)(base + cap * 8 + Layout::ofs_bytes(cap) + 64); }
    __device__ __forceinline__ double *win() const { return rrow() + kRowsT; }
    __device__ __forceinline__ int4 *seg() const { return (int4 *)(win() + wcap); }
};
__host__ __device__ inline int64_t slot_bytes_p(int64_t cap, int64_t wcap) {
    return cap * 8 + Layout::ofs_bytes(cap) + 64 + (int64_t)kRowsT * 8 + wcap * 8 + 33 * 16;
}

// stage a window of `vec` for a tile into `ws` from its segments (lane k:
// segment k = {lo low, lo high, len, base}); returns this lane's bulk bytes
__device__ __forceinline__ uint32_t stage_window(double *wsb, const double *vec, int64_t n, int nseg, int4 sg,
                                                 int lane, uint64_t *bar, uint64_t pol, bool issue) {
    uint32_t wbytes = 0;
    int64_t wa = 0, lo = 0;
    int sbase = 0;
    if (lane < nseg) {
        lo = (int64_t)(((uint64_t)(uint32_t)sg.y << 32) | (uint32_t)sg.x);
        const int len = sg.z;
        sbase = sg.w;
        double *ws = wsb + sbase - lo;
        const int64_t hi = lo + len;
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
    if (issue && wbytes) ptx::bulk_g2s(wsb + sbase + (wa - lo), vec + wa, wbytes, bar, pol);
    return wbytes;
}

__global__ void __launch_bounds__(kThreadsP, 2) k_sweeps_pair(const __grid_constant__ PairParams p) {
    extern __shared__ __align__(128) char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned int epoch = *(volatile unsigned int *)&p.sync[0];
    const int64_t G = gridDim.x, c = blockIdx.x, ntiles = p.ntiles;
    const int64_t mine = c < ntiles ? (ntiles - 1 - c) / G + 1 : 0;
    uint64_t *fullA = (uint64_t *)sm, *emptyA = fullA + 2, *fullB = fullA + 4, *emptyB = fullA + 6;
    unsigned int *cnt = (unsigned int *)(sm + 64);
    auto slot = [&](int s) { return Slot{sm + 256 + s * p.slot_bytes, p.cap, p.wcap}; };
    double *winB0 = (double *)(sm + 256 + 2 * p.slot_bytes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(fullA + s, 1);
            ptx::mbar_init(emptyA + s, kPW);
            ptx::mbar_init(fullB + s, 1);
            ptx::mbar_init(emptyB + s, kPW);
        }
        for (int q = 0; q < kSlotsP; ++q) cnt[q] = 0;
        ptx::mbar_init_fence();
    }
    __syncthreads();

    if (warp == kPW) {
        // ------------------------------------------------------------ producer
        const uint64_t pol_first = ptx::policy_evict_first(), pol_keep = ptx::policy_evict_normal();
        const SellView P[1] = {p.L};
        const Layout Ly{1, 1, p.cap, 8, p.wcap};
        int64_t Fs = 0, Ff = 0;  // sweep-1 frontier: seen (relaxed), fenced
        unsigned int rv[kPVp];
        bool pending = false;
        auto issue = [&]() {
#pragma unroll
            for (int q = 0; q < kPVp; ++q) {
                const int64_t cc = lane + 32 * q;
                rv[q] = cc < G ? ptx::ld_relaxed_gpu_u32(p.prog + cc) : 0u;
            }
            pending = true;
        };
        auto reduce = [&]() {
            int64_t f = INT64_MAX;
#pragma unroll
            for (int q = 0; q < kPVp; ++q) {
                const int64_t cc = lane + 32 * q;
                if (cc < G) {
                    const int64_t k = (rv[q] & 0xffe00000u) == ptag(epoch) ? (int64_t)(rv[q] & 0x1fffffu) : 0;
                    f = min(f, cc + k * G);
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) f = min(f, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)f, o));
            Fs = max(Fs, f);
            pending = false;
        };
        TileRefs<1> cur, nxt;
        if (c < ntiles) tile_refs<1>(Ly, P, 0, p.nslices, c, lane, cur, p.W, true);
        for (int64_t m = 0; m <= mine; ++m) {
            if (m < mine) {
                // ---- stage A: tile t_m into ring slot m & 1
                const int64_t t = c + m * G;
                if (m + 1 < mine) tile_refs<1>(Ly, P, 0, p.nslices, t + G, lane, nxt, p.W, true);
                const int s = (int)(m & 1);
                if (m >= 2) ptx::mbar_wait(emptyA + s, (uint32_t)((m / 2 - 1) & 1));
                const Slot S = slot(s);
                const int4 sg = lane < cur.nseg ? make_int4((int)(uint32_t)cur.sg_lo, (int)((uint64_t)cur.sg_lo >> 32),
                                                            cur.sg_len, cur.sg_base)
                                                : make_int4(0, 0, 0, 0);
                S.seg()[lane] = sg;
                if (lane == 0) S.seg()[32] = make_int4(cur.nseg, 0, 0, 0);   // segment count for stage B
                // window positions, header
                int32_t *so = S.pos();
                const int64_t no = (cur.e[0] - cur.b[0]) / kSlice;
#pragma unroll
                for (int q = 0; q < kOfsPerLane; ++q) {
                    const int64_t k = lane + 32 * q;
                    if (k < no) so[k] = cur.o[0][q];
                }
                const int32_t *go = p.W.wpos[0] + cur.b[0] / kSlice;
                for (int64_t k = lane + 32 * kOfsPerLane; k < no; k += 32) so[k] = __ldg(go + k);
                const int64_t nsp = __shfl_down_sync(0xffffffffu, cur.sp[0], 1);
                int32_t *h = S.hdr();
                if (lane < kTS) {
                    h[2 * lane] = (int32_t)(cur.sp[0] - cur.b[0]);
                    h[2 * lane + 1] = (int32_t)((nsp - cur.sp[0]) / kSlice);
                }
                const int64_t r0 = t * kRowsT, rows = min((int64_t)kRowsT, p.n - r0);
                if (lane == 0 && (rows & 1)) S.rrow()[rows - 1] = p.r[r0 + rows - 1];
                uint32_t wb = stage_window(S.win(), p.g0, p.n, cur.nseg, sg, lane, fullA + s, pol_keep, false);
#pragma unroll
                for (int o = 16; o; o >>= 1) wb += __shfl_xor_sync(0xffffffffu, wb, o);
                const uint32_t rb = (uint32_t)((rows & ~(int64_t)1) * 8);
                const uint32_t vb = (uint32_t)((cur.e[0] - cur.b[0]) * 8);
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_expect_tx(fullA + s, vb + rb + wb);
                    if (vb) ptx::bulk_g2s(S.val(), p.L.val + cur.b[0], vb, fullA + s, pol_keep);
                    if (rb) ptx::bulk_g2s(S.rrow(), p.r + r0, rb, fullA + s, pol_keep);
                }
                __syncwarp();
                stage_window(S.win(), p.g0, p.n, cur.nseg, sg, lane, fullA + s, pol_keep, true);
                __syncwarp();
                cur = nxt;
            }
            if (m >= 1) {
                // ---- stage B: the g(1) window of tile t_{m-1} (after sweep 1 is done through it)
                const int64_t mb = m - 1, tb = c + mb * G;
                const int s = (int)(mb & 1);
                if (mb >= 2) ptx::mbar_wait(emptyB + s, (uint32_t)((mb / 2 - 1) & 1));
                if (pending) reduce();
                if (tb >= Ff) {
                    if (tb >= Fs) {
                        const uint64_t t0 = ptx::globaltimer_ns();
                        while (true) {
                            issue();
                            reduce();
                            if (tb < Fs) break;
                            if (ptx::globaltimer_ns() - t0 > p.timeout_ns) {
                                if (lane == 0) atomicOr(p.err, 2u);
                                Fs = INT64_MAX;
                                break;
                            }
                            __nanosleep(64);
                        }
                    }
                    ptx::fence_acq_rel_gpu();
                    Ff = Fs;
                    __syncwarp();
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                const Slot S = slot(s);
                const int nseg = S.seg()[32].x;
                const int4 sg = lane < nseg ? S.seg()[lane] : make_int4(0, 0, 0, 0);
                double *wbuf = winB0 + s * p.wcap;
                uint32_t wb = stage_window(wbuf, p.g1, p.n, nseg, sg, lane, fullB + s, pol_first, false);
#pragma unroll
                for (int o = 16; o; o >>= 1) wb += __shfl_xor_sync(0xffffffffu, wb, o);
                __syncwarp();
                if (lane == 0) ptx::mbar_expect_tx(fullB + s, wb);
                __syncwarp();
                stage_window(wbuf, p.g1, p.n, nseg, sg, lane, fullB + s, pol_first, true);
                __syncwarp();
                if (!pending && Fs < ntiles && tb + G + 2 * G >= Fs) issue();   // the next view, in flight
            }
        }
    } else {
        // ------------------------------------------------------------ consumers
        const unsigned long long sid = (unsigned long long)p.sweep_id0;
        for (int64_t m = 0; m <= mine; ++m) {
            if (m < mine) {   // sweep 1 on t_m: g(1) = (r - L g(0)) / d
                const int64_t t = c + m * G;
                const int s = (int)(m & 1);
                const int64_t sl = t * kTS + warp, i = sl * kSlice + lane;
                const bool has = sl < p.nslices, row = has && i < p.n;
                const double di = row ? __ldg(p.d + i) : 1.0;
                ptx::mbar_wait(fullA + s, (uint32_t)((m / 2) & 1));
                const Slot S = slot(s);
                double acc = 0.0;
                if (has) {
                    const int2 hd = *(const int2 *)(S.hdr() + 2 * warp);
                    acc = win_sum_chunked<16>(S.val(), S.pos(), S.win(), hd.x, hd.y, lane, row, acc);
                }
                if (row) {
                    const double v = __ddiv_rn(__dsub_rn(S.rrow()[warp * kSlice + lane], acc), di);
                    if (!isfinite(v)) atomicMin(p.flag, sid);
                    p.g1[i] = v;
                }
                __syncwarp();
                if (lane == 0) {   // the last warp to count tile m publishes tiles 0..m of this CTA
                    const unsigned int prev = ptx::atom_add_acqrel_cta_shared(cnt + m % kSlotsP, 1u);
                    if (prev + 1 == (unsigned int)((m / kSlotsP + 1) * kPW))
                        ptx::red_max_release_gpu_u32(p.prog + c, ptag(epoch) | (unsigned int)(m + 1));
                }
            }
            if (m >= 1) {    // sweep 2 on t_{m-1}: x += (r - L g(1)) / d
                const int64_t mb = m - 1, t = c + mb * G;
                const int s = (int)(mb & 1);
                const int64_t sl = t * kTS + warp, i = sl * kSlice + lane;
                const bool has = sl < p.nslices, row = has && i < p.n;
                const double di = row ? __ldg(p.d + i) : 1.0;
                const double xi = row ? p.x[i] : 0.0;
                ptx::mbar_wait(fullB + s, (uint32_t)((mb / 2) & 1));
                const Slot S = slot(s);
                double acc = 0.0;
                if (has) {
                    const int2 hd = *(const int2 *)(S.hdr() + 2 * warp);
                    acc = win_sum_chunked<16>(S.val(), S.pos(), winB0 + s * p.wcap, hd.x, hd.y, lane, row, acc);
                }
                const double ri = row ? S.rrow()[warp * kSlice + lane] : 0.0;
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(emptyA + s);   // the ring slot and the window buffer may be refilled
                    ptx::mbar_arrive(emptyB + s);
                }
                if (row) {
                    const double v = __ddiv_rn(__dsub_rn(ri, acc), di);
                    if (!isfinite(v)) atomicMin(p.flag, sid + 1);
                    p.x[i] = __dadd_rn(xi, v);
                }
            }
        }
    }
    // ---- the last CTA out advances the epoch (clearing the words before the tag wraps)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(&p.sync[1], 1u);
        if (prev == gridDim.x - 1) {
            const unsigned int next = epoch + 1 == 0 ? 1 : epoch + 1;
            if (ptag(next) == 0)
                for (int64_t q = 0; q < G; ++q) p.prog[q] = 0u;
            p.sync[1] = 0;
            p.sync[0] = next;
            __threadfence();
        }
    }
}

WinView wview_p(const Window *w) {
    return WinView{w->tseg, w->glo, w->len, w->sbase, {w->wpos[0], w->wpos[1]}, (w->wmax + 31) / 32 * 32};
}

}  // namespace

bool pair_possible(int maxw_l, int64_t wmax, int maxseg) {
    if (maxw_l < 1 || maxw_l > 16 || wmax <= 0 || maxseg > 32) return false;
    const int64_t cap = (int64_t)kTS * kSlice * maxw_l, wcap = (wmax + 31) / 32 * 32;
    return 256 + 2 * slot_bytes_p(cap, wcap) + 2 * wcap * 8 <= kSmemMaxP;
}

cudaError_t launch_pair(const PairLaunch &L, cudaStream_t st) {
    static std::mutex mu;
    static std::map<int, bool> attr;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!attr[dev]) {
            cudaFuncSetAttribute(k_sweeps_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMaxP);
            attr[dev] = true;
        }
    }
    PairParams p{};
    p.n = L.n;
    p.nslices = (L.n + kSlice - 1) / kSlice;
    p.ntiles = (L.n + kRowsT - 1) / kRowsT;
    p.L = view(*L.Lp);
    p.W = wview_p(L.wl);
    p.cap = (int64_t)kTS * kSlice * std::max(L.Lp->maxw, 1);
    p.wcap = p.W.wcap;
    p.slot_bytes = slot_bytes_p(p.cap, p.wcap);
    const size_t smem = (size_t)(256 + 2 * p.slot_bytes + 2 * p.wcap * 8);
    int occ = 0, nsm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweeps_pair, kThreadsP, smem);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>({(int64_t)nsm * occ, p.ntiles, (int64_t)32 * kPVp, L.pstride});
    if (grid < 1) return cudaErrorInvalidConfiguration;
    p.d = L.d;
    p.r = L.r;
    p.g0 = L.g0;
    p.g1 = L.g1;
    p.x = L.x;
    p.prog = L.prog;
    p.sync = L.sync;
    p.flag = L.flag;
    p.sweep_id0 = L.sweep_id0;
    p.err = L.err;
    p.timeout_ns = L.timeout_ns;
    void *args[] = {&p};
    return cudaLaunchCooperativeKernel((const void *)k_sweeps_pair, dim3((unsigned)grid), dim3(kThreadsP), args, smem,
                                       st);
}

void preload_pair_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_sweeps_pair);
}

}  // namespace nsm
