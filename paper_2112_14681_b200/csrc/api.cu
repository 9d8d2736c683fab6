// api.cu — the C-ABI of libnsm.so (include/nsm.h).
//
// Owns the handle (device copies of the split storage, workspace, halo
// mailbox) and turns each nsm_* call into a fixed sequence of kernel launches
// on the caller's stream: no allocation and no host synchronisation on the
// hot calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nsm_internal.h"

using namespace nsm;

namespace {

struct Peer {
    int q = -1;
    std::vector<int32_t> send_rows;   // local rows rank q needs from us
    bool send_set = false;
    int32_t *d_send_rows = nullptr;
    double *remote_data = nullptr;    // q's ghost data base + q's offset for our block
    int64_t remote_stride = 0;        // q's n_ghost (parity stride)
    unsigned long long *remote_flags = nullptr;
    void *ipc_base = nullptr;         // opened IPC mapping to close at destroy
    bool connected = false;
};

}  // namespace

struct nsm_handle {
    int device = 0;
    uint64_t uid = 0;  // unique per setup (caches keyed by handle must not confuse a reused address)
    uint64_t cfg_gen = 0;  // bumped by nsm_set_option / nsm_set_ruiz (captured graphs compare it)
    nsm_comm *comm = nullptr;  // borrowed cross-rank reduction (nsm_set_comm), distributed solver layer
    Window res_win;            // gather window of the residual (L and U together), single rank
    // one-pass windowed pGS (fused_w.cu): rings, per-phase progress, launch state
    bool fw_ready = false;
    double *fw_ring_r = nullptr, *fw_ring_g = nullptr;
    int64_t fw_Mr = 0, fw_Mg = 0;
    unsigned long long *fw_prog = nullptr;
    unsigned int *fw_sync = nullptr;
    int32_t *fw_tpos[2] = {nullptr, nullptr}, *fw_nseg[2] = {nullptr, nullptr};
    int4 *fw_tseg[2] = {nullptr, nullptr};
    int fw_pst = 0;
    int64_t plane_tiles = 0;   // NSM_OPT_PLANE_ROWS / 256 when the plane-wavefront check passed
    // coupled passes (coupled.cu): progress counters and launch state, single rank
    int coupled = 0;           // NSM_OPT_COUPLED: 0 off (default), 1 on, > 1: on with this throttle lag (tiles)
    unsigned long long *cp_prog = nullptr, *cp_stats = nullptr;
    unsigned int *cp_sync = nullptr;
    bool window = true;        // NSM_OPT_WINDOW: windowed pipelined kernels where a window exists
    bool chunked_host = true;  // NSM_OPT_HOST_CHUNKS: nsm_smooth_host overlaps copies and passes
    int64_t n = 0, row_begin = 0, n_ghost = 0, nnz_off = 0, device_bytes = 0;
    int nslices = 0;
    // A = L + D + U (+ ghost couplings LG / UG)
    double *d = nullptr, *dl1 = nullptr;  // diagonal; l1-Jacobi diagonal
    Sell L, U, LG, UG;
    // ILU(0) factors: unit-lower L = I + Ls, U = D_U (I + D_U^{-1} Us)
    bool has_ilu = false;
    double *dU = nullptr;
    // nsm_smooth_host staging vectors (allocated by its first call)
    double *hb_dev = nullptr, *hx_dev = nullptr;
    // chunked nsm_smooth_host (copies overlapped with the passes): streams, events
    cudaStream_t hs_in = nullptr, hs_out = nullptr;
    std::vector<cudaEvent_t> hev;          // 2 per chunk + 2
    // Ruiz-scaled U factor (Alg. 2 / NEXT-3): U~ = diag(1/s_r) U diag(1/s_c), unit diagonal
    bool ruiz = false;
    double *s_r = nullptr, *s_c = nullptr;
    Sell Ls, Us, LsG, UsG;
    // workspace: four n-vectors (residual, ping-pong iterates, g^(0)), divergence flag
    double *w[4] = {nullptr, nullptr, nullptr, nullptr};
    unsigned long long *flag = nullptr;
    int64_t sweep_counter = 0;
    int64_t launches = 0, exchanges = 0;
    // ---- distribution (row-block partition)
    int rank = 0, nranks = 1;
    nsm_dist_mode mode = NSM_DIST_HYBRID;
    std::vector<int64_t> row_offsets, ghost_gid, recv_off;  // recv_off[q]: first ghost owned by q
    int32_t *interior = nullptr, *boundary = nullptr;       // slice lists
    int n_interior = 0, n_boundary = 0;
    int64_t interior_begin = -1, interior_end = -1;          // set if the interior list is one range
    bool pipeline = true;                                    // bulk-copy pipelined kernels (stream.cu)
    bool pdl = true;                                         // programmatic dependent launch for them
    // in-stream pass timing (NSM_OPT_PROFILE): event pool and records
    bool profile = false;
    std::vector<cudaEvent_t> ev;
    std::vector<int> ev_kind;                                // kind of record i (events 2i, 2i+1)
    int ev_used = 0;
    // phase-skewed fused passes (fused.cu), single rank
    int fused_mode = 0;                      // NSM_OPT_FUSED: 0 off (default), 1 on, 2 auto (large problems)
    bool fused_ready = false, fused_possible = false;  // rings allocated / single rank
    int skew_dw = 0;                         // NSM_OPT_FUSED_WINDOW (0 = automatic)
    int DLA = 0, DUA = 0, DLs = 0, DUs = 0;  // bandwidths in tiles of A and of the factors
    static constexpr int kFusedKmax = 8;
    double *ring_r = nullptr, *ring_g = nullptr;
    int64_t ring_r_tiles = 0, ring_g_tiles = 0;
    SkewSync *skew_sync = nullptr;
    unsigned long long *skew_prog = nullptr;  // per-CTA progress counters
    void *mailbox = nullptr;           // [flags: nranks u64, padded][data: 2 x n_ghost f64]
    size_t mailbox_bytes = 0, flags_bytes = 0;
    unsigned long long *mb_flags = nullptr;
    double *mb_data = nullptr;
    std::vector<Peer> peers;           // symmetric neighbour set, ascending q
    PutDesc *d_put = nullptr;
    int *d_peer_ids = nullptr;
    unsigned int *d_counters = nullptr, *d_dist_err = nullptr;
    int put_grid = 0;
    bool committed = false;
    unsigned long long exch_seq = 0;
    cudaStream_t side = nullptr;           // the halo put runs here, concurrently with the interior kernel
    cudaEvent_t ev_fork = nullptr, ev_put = nullptr;
    unsigned long long timeout_ns = 20ull * 1000 * 1000 * 1000;
    double *ghost_null = nullptr;      // 1-element dummy ghost buffer (single rank)
    std::string err;
};

namespace {

thread_local std::string g_setup_err;

struct DevAlloc {
    nsm_handle *h;
    template <class T>
    bool get(T **p, int64_t count) {
        *p = nullptr;
        if (count <= 0) return true;
        size_t bytes = (size_t)count * sizeof(T);
        if (cudaMalloc((void **)p, bytes) != cudaSuccess) { *p = nullptr; return false; }
        h->device_bytes += (int64_t)bytes;
        return true;
    }
};

// progress counters and launch state of the coupled passes (coupled.cu):
// [3][kCpProgStride] per-CTA counters, zero once; sync[0] = epoch 1
constexpr int64_t kCpProgStride = 1024;
bool coupled_alloc(DevAlloc &a, nsm_handle *h) {
    const unsigned int init[4] = {1u, 0u, 0u, 0u};
    return a.get(&h->cp_prog, 3 * kCpProgStride) && a.get(&h->cp_sync, 4) && a.get(&h->cp_stats, 16) &&
           cudaMemset(h->cp_stats, 0, 16 * sizeof(unsigned long long)) == cudaSuccess &&
           cudaMemset(h->cp_prog, 0, 3 * kCpProgStride * sizeof(unsigned long long)) == cudaSuccess &&
           cudaMemcpy(h->cp_sync, init, sizeof(init), cudaMemcpyHostToDevice) == cudaSuccess;
}

template <class T>
bool upload(T *dst, const T *src, int64_t count) {
    if (count <= 0) return true;
    return cudaMemcpy(dst, src, (size_t)count * sizeof(T), cudaMemcpyHostToDevice) == cudaSuccess;
}

bool upload_sell(DevAlloc &a, const SellHost &hs, Sell *s) {
    s->padded = (int64_t)hs.col.size();
    s->nnz = hs.nnz;
    s->maxw = hs.maxw;
    if (!a.get(&s->ptr, (int64_t)hs.ptr.size())) return false;
    if (!upload(s->ptr, hs.ptr.data(), (int64_t)hs.ptr.size())) return false;
    if (!a.get(&s->col, s->padded) || !a.get(&s->val, s->padded)) return false;
    if (!hs.off.empty() && (!a.get(&s->off, (int64_t)hs.off.size()) || !upload(s->off, hs.off.data(), (int64_t)hs.off.size())))
        return false;
    return upload(s->col, hs.col.data(), s->padded) && upload(s->val, hs.val.data(), s->padded);
}

void free_window(Window &w) {
    cudaFree(w.tseg);
    cudaFree(w.glo);
    cudaFree(w.len);
    cudaFree(w.sbase);
    cudaFree(w.wpos[0]);
    cudaFree(w.wpos[1]);
    w = Window();
}

void free_sell(Sell &s) {
    cudaFree(s.ptr);
    cudaFree(s.col);
    cudaFree(s.val);
    cudaFree(s.off);
    free_window(s.win);
    s = Sell();
}

// Gather window of a group of offset-aligned parts (stream.cu windowed
// kernels).  Not built (wmax = 0) when a part is compact or a tile's window
// would exceed kWinCap doubles; failure to allocate is an error.
constexpr int32_t kWinCap = 8192;
bool make_window(DevAlloc &a, int64_t n, const std::vector<const SellHost *> &parts, Window *w) {
    WindowHost wh;
    if (n <= 0 || !build_window(n, parts, kWinCap, &wh)) return true;
    if (!a.get(&w->tseg, (int64_t)wh.tseg.size()) || !upload(w->tseg, wh.tseg.data(), (int64_t)wh.tseg.size()) ||
        !a.get(&w->glo, (int64_t)wh.glo.size()) || !upload(w->glo, wh.glo.data(), (int64_t)wh.glo.size()) ||
        !a.get(&w->len, (int64_t)wh.len.size()) || !upload(w->len, wh.len.data(), (int64_t)wh.len.size()) ||
        !a.get(&w->sbase, (int64_t)wh.sbase.size()) || !upload(w->sbase, wh.sbase.data(), (int64_t)wh.sbase.size()))
        return false;
    for (size_t p = 0; p < parts.size(); ++p)
        if (!a.get(&w->wpos[p], (int64_t)wh.wpos[p].size()) ||
            !upload(w->wpos[p], wh.wpos[p].data(), (int64_t)wh.wpos[p].size()))
            return false;
    w->wmax = wh.wmax;
    w->maxseg = wh.maxseg;
    return true;
}

void free_handle(nsm_handle *h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    for (Sell *s : {&h->L, &h->U, &h->LG, &h->UG, &h->Ls, &h->Us, &h->LsG, &h->UsG}) free_sell(*s);
    free_window(h->res_win);
    cudaFree(h->d);
    cudaFree(h->dl1);
    cudaFree(h->dU);
    cudaFree(h->s_r);
    cudaFree(h->s_c);
    for (double *&p : h->w) cudaFree(p);
    cudaFree(h->flag);
    cudaFree(h->interior);
    cudaFree(h->boundary);
    for (Peer &p : h->peers) {
        cudaFree(p.d_send_rows);
        if (p.ipc_base) cudaIpcCloseMemHandle(p.ipc_base);
    }
    if (h->side) cudaStreamDestroy(h->side);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_put) cudaEventDestroy(h->ev_put);
    cudaFree(h->mailbox);
    cudaFree(h->d_put);
    cudaFree(h->d_peer_ids);
    cudaFree(h->d_counters);
    cudaFree(h->d_dist_err);
    cudaFree(h->ghost_null);
    for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
    cudaFree(h->ring_r);
    cudaFree(h->ring_g);
    cudaFree(h->fw_ring_r);
    cudaFree(h->fw_ring_g);
    cudaFree(h->fw_prog);
    cudaFree(h->fw_sync);
    cudaFree(h->cp_prog);
    cudaFree(h->cp_stats);
    cudaFree(h->cp_sync);
    for (int q = 0; q < 2; ++q) {
        cudaFree(h->fw_tpos[q]);
        cudaFree(h->fw_nseg[q]);
        cudaFree(h->fw_tseg[q]);
    }
    cudaFree(h->skew_sync);
    cudaFree(h->skew_prog);
    cudaFree(h->hb_dev);
    cudaFree(h->hx_dev);
    if (h->hs_in) cudaStreamDestroy(h->hs_in);
    if (h->hs_out) cudaStreamDestroy(h->hs_out);
    for (cudaEvent_t e : h->hev) cudaEventDestroy(e);
    delete h;
}

nsm_status cuda_fail(nsm_handle *h, cudaError_t e, const char *where) {
    h->err = std::string(where) + ": " + cudaGetErrorString(e);
    return NSM_ERR_CUDA;
}

inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

bool overlap(const double *a, const double *b, int64_t n) { return a && b && a < b + n && b < a + n; }

bool distributed(const nsm_handle *h) { return h->nranks > 1; }

Peer *find_peer(nsm_handle *h, int q) {
    for (Peer &p : h->peers)
        if (p.q == q) return &p;
    return nullptr;
}

// ---- one pass over the slices, with or without a halo exchange --------------
// A set of slices: an explicit list, and (if it is one contiguous range)
// its bounds, which lets the bulk-copy pipelined kernels stream it.
struct Slices {
    const int32_t *list;
    int count;
    int64_t begin, end;  // begin < 0: not a single range
};

// launch(slices, with_ghost, ghost): run the kernel on a set of slices.
// With an exchange of `src` (scaled by 1/scale if given): put -> interior
// slices (overlap with the NVLink transfer) -> wait -> boundary slices.
// Optional in-stream timing of each pass (NSM_OPT_PROFILE): an event pair
// around the pass, accumulated per kind by nsm_profile().
struct ProfScope {
    nsm_handle *h;
    int kind;
    cudaStream_t s;
    int slot = -1;
    ProfScope(nsm_handle *h_, int kind_, cudaStream_t s_) : h(h_), kind(kind_), s(s_) {
        if (!h->profile || h->ev_used >= (int)h->ev_kind.size()) return;
        slot = h->ev_used++;
        h->ev_kind[slot] = kind;
        cudaEventRecord(h->ev[2 * slot], s);
    }
    ~ProfScope() {
        if (slot >= 0) cudaEventRecord(h->ev[2 * slot + 1], s);
    }
};

template <class F>
nsm_status pass(nsm_handle *h, bool exchange, const double *src, const double *scale, cudaStream_t s, F launch,
                int prof_kind) {
    ProfScope prof(h, prof_kind, s);
    if (!exchange || !distributed(h)) {
        cudaError_t e = launch(Slices{nullptr, h->nslices, 0, h->nslices}, false, (const double *)h->ghost_null);
        if (h->n > 0) ++h->launches;
        return e == cudaSuccess ? NSM_OK : cuda_fail(h, e, "kernel launch");
    }
    if (!h->committed) {
        h->err = "halo exchange requested before nsm_halo_commit";
        return NSM_ERR_STATE;
    }
    const unsigned long long seq = ++h->exch_seq;
    const int parity = (int)(seq & 1);
    const double *ghost = h->mb_data + (int64_t)parity * h->n_ghost;
    // the put (gather of the boundary entries + peer stores over NVLink) runs
    // on the side stream, concurrently with the interior slices on `s`; the
    // wait kernel is ordered after both
    const bool fork = h->side && h->n_interior > 0;
    cudaError_t e = cudaSuccess;
    if (fork) {
        e = cudaEventRecord(h->ev_fork, s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(h->side, h->ev_fork, 0);
        if (e != cudaSuccess) return cuda_fail(h, e, "halo fork");
    }
    e = launch_halo_put(h->d_put, (int)h->peers.size(), h->put_grid, src, scale, parity, seq, h->d_counters,
                        fork ? h->side : s);
    if (e != cudaSuccess) return cuda_fail(h, e, "halo put");
    if (fork) {
        e = cudaEventRecord(h->ev_put, h->side);
        if (e != cudaSuccess) return cuda_fail(h, e, "halo put event");
    }
    if (h->n_interior > 0) {
        e = launch(Slices{h->interior, h->n_interior, h->interior_begin, h->interior_end}, false, ghost);
        ++h->launches;
        if (e != cudaSuccess) return cuda_fail(h, e, "kernel launch (interior)");
    }
    if (fork && (e = cudaStreamWaitEvent(s, h->ev_put, 0)) != cudaSuccess) return cuda_fail(h, e, "halo join");
    e = launch_halo_wait(h->mb_flags, h->d_peer_ids, (int)h->peers.size(), seq, h->timeout_ns, h->d_dist_err, s);
    if (e != cudaSuccess) return cuda_fail(h, e, "halo wait");
    if (h->n_boundary > 0) {
        e = launch(Slices{h->boundary, h->n_boundary, -1, -1}, true, ghost);
        ++h->launches;
        if (e != cudaSuccess) return cuda_fail(h, e, "kernel launch (boundary)");
    }
    h->launches += h->peers.empty() ? 0 : 2;
    ++h->exchanges;
    return NSM_OK;
}

// Bulk-copy pipelined kernels for contiguous slice ranges, unless the rows
// are too wide to stage or the level is small with wide rows (warp-per-row
// kernels).  (Plain kernels on mid-sized AMG levels, 50K-300K rows, were
// measured 15-40 % slower: profiles/r01_solver_solve_timing.md.)
bool use_pipelined(const nsm_handle *h, const Slices &sl, bool with_ghost, int np, int maxw) {
    return h->pipeline && sl.begin >= 0 && !with_ghost && tma_ok(np, maxw) && !wide_rows(maxw, h->nslices);
}

// One stage of a Jacobi-iterated triangular solve: k >= 1 sweeps on T from
// g^(0) = rhs / dT (recomputed in the first sweep's gather), the final
// iterate written with epilogue last_epi.  bufA/bufB: ping-pong scratch.
// TG: ghost couplings of T, used in GLOBAL mode (exchange before each sweep).
struct Stage {
    const Sell *T;
    const Sell *TG;
    const double *dT;    // nullptr = unit diagonal
    const double *rhs;
    int k;
    const double *g0 = nullptr;  // materialised g^(0) (else recomputed as rhs / dT)
};

nsm_status run_sweeps(nsm_handle *h, const Stage &st, double *bufA, double *bufB, int last_epi, double *last_out,
                      double *x, const double *dnext, cudaStream_t s, double *gout2 = nullptr) {
    const bool global = distributed(h) && h->mode == NSM_DIST_GLOBAL;
    const double *gin = st.g0;
    for (int j = 1; j <= st.k; ++j) {
        const bool last = j == st.k;
        double *out = last ? last_out : ((j & 1) ? bufA : bufB);
        const int64_t sid = ++h->sweep_counter;
        const bool scaled = j == 1 && !st.g0;
        // the ghost values a GLOBAL sweep needs are those of its input iterate:
        // g^(0) (materialised, or rhs / dT) for the first sweep, then the
        // previous output
        const double *xsrc = scaled ? st.rhs : gin;
        const double *xscale = scaled ? st.dT : nullptr;
        nsm_status r = pass(h, global, xsrc, xscale, s,
                            [&](const Slices &sl, bool with_ghost, const double *ghost) {
                                SweepArgs a{};
                                a.n = h->n;
                                a.nslices = sl.count;
                                a.list = sl.list;
                                a.T = st.T;
                                a.TG = st.TG;
                                // upper-triangle ghosts follow the local entries
                                a.has_ghost = !with_ghost ? 0 : ((st.TG == &h->UG || st.TG == &h->UsG) ? 2 : 1);
                                a.unit = st.dT == nullptr;
                                a.epi = last ? last_epi : EPI_STORE;
                                a.gin_scaled = scaled;
                                a.dT = st.dT;
                                a.rhs = st.rhs;
                                a.gin = gin;
                                a.ghost = ghost;
                                a.gout = out;
                                a.x = x;
                                a.dnext = dnext;
                                a.gout2 = last ? gout2 : nullptr;
                                a.flag = h->flag;
                                a.sweep_id = sid;
                                a.pdl = h->pdl;
                                // windows of the local parts are planned on tiles of the full
                                // local range: usable for any tile-aligned contiguous range (the
                                // interior slices of a slab partition too)
                                a.win = (h->window && st.T->win.wmax && !scaled && sl.begin >= 0 &&
                                         sl.begin % kTileSlices == 0) ? &st.T->win : nullptr;
                                if (use_pipelined(h, sl, with_ghost, 1, st.T->maxw))
                                    return launch_sweep_tma(a, sl.begin, sl.end, s);
                                return launch_sweep(a, s);
                            },
                            1);
        if (r != NSM_OK) return r;
        gin = out;
    }
    return NSM_OK;
}

// mode OUT_R: out = b - A x; OUT_AX: out = A x; OUT_RG: also out2 = out / d.
nsm_status residual_into(nsm_handle *h, const double *b, const double *x, double *out, int mode, cudaStream_t s,
                         double *out2 = nullptr) {
    return pass(h, true, x, nullptr, s, [&](const Slices &sl, bool with_ghost, const double *ghost) {
        if (use_pipelined(h, sl, with_ghost, 2, std::max(h->L.maxw, h->U.maxw)))
            return launch_residual_tma((h->window && h->res_win.wmax && sl.begin >= 0 && sl.begin % kTileSlices == 0)
                                           ? &h->res_win : nullptr,
                                       mode, h->n, sl.begin, sl.end, h->L, h->U, h->d, b, x, out, out2, h->pdl, s);
        return launch_residual(mode, h->n, sl.count, sl.list, h->LG, h->L, h->U, h->UG, with_ghost, h->d, b, x, ghost,
                               out, out2, h->pdl, s);
    }, 0);
}

nsm_status scale_into(nsm_handle *h, bool xadd, const double *rhs, const double *d, double *out, cudaStream_t s) {
    cudaError_t e = launch_scale(xadd, h->n, rhs, d, out, h->flag, ++h->sweep_counter, h->pdl, s);
    if (h->n > 0) ++h->launches;
    return e == cudaSuccess ? NSM_OK : cuda_fail(h, e, "scale launch");
}

uint64_t next_handle_uid() {
    static std::atomic<uint64_t> next_uid{1};
    return next_uid++;
}

size_t flags_bytes_for(int nranks) { return (((size_t)nranks * 8 + 255) / 256) * 256; }

}  // namespace

// Rings, progress counters and launch state of the fused passes, sized for
// the largest shape any k <= kFusedKmax can need (single rank; once).
// Rings and counters of the one-pass windowed pGS (fused_w.cu), sized for
// k <= kMaxPhW - 1: single rank, offset-aligned L and U with gather windows.
constexpr int64_t kFwProgStride = 1024;
static bool fw_possible(const nsm_handle *h) {
    return h->fused_possible && h->L.off && h->U.off && h->U.win.wmax && h->L.win.wmax;
}
static FusedWShape fw_shape(const nsm_handle *h, int k, bool planes) {
    return fused_w_shape(std::max(h->L.maxw, h->U.maxw), std::max(h->U.win.wmax, h->L.win.wmax), k, h->n, h->DLA,
                         std::max(h->DLA, h->DUA), h->skew_dw, planes ? h->plane_tiles : 0);
}

// NSM_OPT_PLANE_ROWS: the plane-wavefront schedule (fused_w.cu
// k_fused_pgs_planes) is valid when every coupling of a tile lies within two
// lines (tile index mod tpp) in the same or a neighbouring plane (checked on
// the device over the stored entries; pads are free: they multiply by 0).
static bool planes_ok(nsm_handle *h, int64_t tpp) {
    const int64_t nt = (h->n + 255) / 256;
    if (tpp < 1 || nt < 2 * tpp) return false;
    return fused_w_plane_check(h->n, tpp, h->L, h->U);
}
static nsm_status fw_alloc(nsm_handle *h) {
    if (h->fw_ready || !fw_possible(h)) return NSM_OK;
    FusedWShape sh = fw_shape(h, kMaxPhW - 1, false);
    if (!sh.ok || sh.grid > kFwProgStride) return NSM_OK;
    const FusedWShape shp = fw_shape(h, kMaxPhW - 1, true);   // rings large enough for both schedules
    if (shp.ok) {
        sh.Mr = std::max(sh.Mr, shp.Mr);
        sh.Mg = std::max(sh.Mg, shp.Mg);
    }
    DevAlloc a{h};
    const unsigned int init[16] = {1u};
    const bool ok = a.get(&h->fw_ring_r, sh.Mr * 256) && a.get(&h->fw_ring_g, (int64_t)(kMaxPhW - 1) * sh.Mg * 256) &&
                    a.get(&h->fw_prog, kMaxPhW * kFwProgStride) && a.get(&h->fw_sync, 16) &&
                    cudaMemset(h->fw_prog, 0, kMaxPhW * kFwProgStride * sizeof(unsigned long long)) == cudaSuccess &&
                    cudaMemcpy(h->fw_sync, init, sizeof(init), cudaMemcpyHostToDevice) == cudaSuccess;
    const int64_t nt = (h->n + 255) / 256;
    const int pst = 8 * std::max(h->L.maxw, h->U.maxw);
    bool tok = ok;
    tok = tok && cudaMemset(h->fw_ring_r, 0, sh.Mr * 256 * sizeof(double)) == cudaSuccess &&
          cudaMemset(h->fw_ring_g, 0, (int64_t)(kMaxPhW - 1) * sh.Mg * 256 * sizeof(double)) == cudaSuccess;
    for (int q = 0; tok && q < 2; ++q)
        tok = a.get(&h->fw_tpos[q], nt * pst) && a.get(&h->fw_nseg[q], nt) && a.get(&h->fw_tseg[q], nt * 32) &&
              fused_w_tables(h->n, q == 0 ? h->L : h->U, q == 0 ? h->L.win : h->U.win, pst, h->fw_tpos[q],
                             h->fw_nseg[q], h->fw_tseg[q]) == cudaSuccess;
    if (!tok) {
        cudaGetLastError();
        h->err = "NSM_OPT_FUSED: device allocation of the one-pass rings failed";
        return NSM_ERR_OOM;
    }
    h->fw_pst = pst;
    h->fw_Mr = sh.Mr;
    h->fw_Mg = sh.Mg;
    h->fw_ready = true;
    return NSM_OK;
}

static nsm_status fused_alloc(nsm_handle *h) {
    const nsm_status fst = fw_alloc(h);
    if (fst != NSM_OK) return fst;
    if (h->fused_ready || !h->fused_possible) return NSM_OK;
    cudaSetDevice(h->device);
    const int64_t tr = skew_tile_rows();
    int64_t mr = 0, mg = 0;
    bool all = true;
    auto need = [&](const SkewShape &sh) {
        all = all && sh.ok;
        mr = std::max(mr, sh.Mr);
        mg = std::max(mg, sh.Mg);
    };
    const int K = nsm_handle::kFusedKmax;
    const int mw = std::max(h->L.maxw, h->U.maxw);
    need(skew_shape(SKEW_RESID, false, h->L.maxw, h->U.maxw, mw, K, h->n, std::max(h->DLA, h->DUA),
                    std::max(h->DLA, h->DUA), 0));
    need(skew_shape(SKEW_NONE, false, 0, 0, mw, K, h->n, std::max(h->DLA, h->DUA), 0, 0));
    if (h->has_ilu) {
        const int mwf = std::max(h->Ls.maxw, h->Us.maxw);
        need(skew_shape(SKEW_RESID, true, h->L.maxw, h->U.maxw, h->Ls.maxw, K, h->n, h->DLs, h->DLA, 0));
        need(skew_shape(SKEW_NONE, true, 0, 0, mwf, K, h->n, std::max(h->DLs, h->DUs), 0, 0));
        need(skew_shape(SKEW_NONE, false, 0, 0, mwf, K, h->n, std::max(h->DLs, h->DUs), 0, 0));
    }
    if (!all) return NSM_OK;  // shapes that do not fit shared memory: per-pass kernels
    if (knob("NSM_DEBUG_FULL_RINGS")) {  // window experiments (tools/skew_exp.py) only
        int64_t t = 1;
        while (t * tr < h->n) t <<= 1;
        mr = mg = t;
    }
    h->ring_r_tiles = std::max<int64_t>(mr, 1);
    h->ring_g_tiles = std::max<int64_t>(mg, 1);
    SkewSync init{};
    init.epoch = 1;
    DevAlloc a{h};
    const bool ok = a.get(&h->ring_r, h->ring_r_tiles * tr) && a.get(&h->ring_g, (int64_t)K * h->ring_g_tiles * tr) &&
                    a.get(&h->skew_sync, 1) && a.get(&h->skew_prog, 4096) &&
                    cudaMemcpy(h->skew_sync, &init, sizeof(init), cudaMemcpyHostToDevice) == cudaSuccess &&
                    cudaMemset(h->skew_prog, 0, 4096 * sizeof(unsigned long long)) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        h->err = "NSM_OPT_FUSED: device allocation of the fused-pass rings failed";
        return NSM_ERR_OOM;
    }
    h->fused_ready = true;
    return NSM_OK;
}

bool nsm::nsm_is_distributed(const nsm_handle *h) { return h && h->nranks > 1; }
uint64_t nsm::nsm_handle_uid(const nsm_handle *h) { return h ? h->uid : 0; }
uint64_t nsm::nsm_handle_cfg_gen(const nsm_handle *h) { return h ? h->cfg_gen : 0; }
int nsm::nsm_handle_device(const nsm_handle *h) { return h ? h->device : 0; }
nsm_comm *nsm::nsm_handle_comm(const nsm_handle *h) { return h ? h->comm : nullptr; }

extern "C" {

const char *nsm_last_error(const nsm_handle *h) { return h ? h->err.c_str() : g_setup_err.c_str(); }

nsm_status nsm_ilu0(const nsm_csr *A, int64_t row_begin, double *fval) {
    if (!A || !fval) { g_setup_err = "nsm_ilu0: NULL argument"; return NSM_ERR_ARG; }
    return ilu0_host(A, row_begin, fval, &g_setup_err);
}

nsm_status nsm_ilu0_fixed_point(const nsm_csr *A, int64_t row_begin, int sweeps, double *fval, int device) {
    if (!A || !fval) { g_setup_err = "nsm_ilu0_fixed_point: NULL argument"; return NSM_ERR_ARG; }
    return ilu0_fixed_point_device(A, row_begin, sweeps, fval, device, &g_setup_err);
}

nsm_status nsm_halo_plan(const nsm_csr *A, const nsm_dist *dist, int64_t *recv_counts, int64_t *ghost_rows,
                         int64_t *n_ghost) {
    if (!A || !dist || dist->nranks < 1 || !dist->row_offsets || !recv_counts || !n_ghost) {
        g_setup_err = "nsm_halo_plan: NULL argument";
        return NSM_ERR_ARG;
    }
    const int64_t *ro = dist->row_offsets;
    const int64_t rb = ro[dist->rank], re = ro[dist->rank + 1];
    if (A->nrows != re - rb) { g_setup_err = "nsm_halo_plan: CSR rows do not match the partition"; return NSM_ERR_DIST; }
    std::vector<int64_t> g;
    for (int64_t i = 0; i < A->nrows; ++i)
        for (int64_t p = A->rowptr[i]; p < A->rowptr[i + 1]; ++p)
            if (A->colind[p] < rb || A->colind[p] >= re) g.push_back(A->colind[p]);
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    for (int q = 0; q < dist->nranks; ++q) recv_counts[q] = 0;
    for (int64_t c : g) {
        int q = (int)(std::upper_bound(ro, ro + dist->nranks + 1, c) - ro) - 1;
        if (q < 0 || q >= dist->nranks) { g_setup_err = "nsm_halo_plan: column outside the partition"; return NSM_ERR_DIST; }
        recv_counts[q]++;
    }
    if (ghost_rows) std::copy(g.begin(), g.end(), ghost_rows);
    *n_ghost = (int64_t)g.size();
    return NSM_OK;
}

nsm_status nsm_setup(nsm_handle **out, const nsm_csr *A, const nsm_csr *F, const nsm_dist *dist, int device) {
    if (!out || !A) { g_setup_err = "nsm_setup: NULL argument"; return NSM_ERR_ARG; }
    *out = nullptr;
    int rank = 0, nranks = 1;
    int64_t rb = 0, re = A->nrows, nglob = A->nrows;
    if (dist && dist->nranks > 1) {
        if (!dist->row_offsets || dist->rank < 0 || dist->rank >= dist->nranks ||
            (dist->mode != NSM_DIST_HYBRID && dist->mode != NSM_DIST_GLOBAL)) {
            g_setup_err = "nsm_setup: bad nsm_dist";
            return NSM_ERR_ARG;
        }
        rank = dist->rank;
        nranks = dist->nranks;
        for (int q = 0; q < nranks; ++q)
            if (dist->row_offsets[q + 1] < dist->row_offsets[q] || dist->row_offsets[0] != 0) {
                g_setup_err = "nsm_setup: row_offsets must start at 0 and ascend";
                return NSM_ERR_DIST;
            }
        rb = dist->row_offsets[rank];
        re = dist->row_offsets[rank + 1];
        nglob = dist->row_offsets[nranks];
        if (A->nrows != re - rb || A->ncols != nglob) {
            g_setup_err = "nsm_setup: CSR block does not match the partition (rows or global columns)";
            return NSM_ERR_DIST;
        }
    } else if (A->ncols != A->nrows) {
        g_setup_err = "nsm_setup: A must be square on one rank";
        return NSM_ERR_ARG;
    }
    Split sa, sf;
    nsm_status st = build_split(A, rb, re, &sa, &g_setup_err);
    if (st != NSM_OK) return st;
    if (F) {
        if (F->nrows != A->nrows || F->ncols != A->ncols) { g_setup_err = "nsm_setup: F shape differs from A"; return NSM_ERR_ARG; }
        st = build_split(F, rb, re, &sf, &g_setup_err);
        if (st != NSM_OK) { g_setup_err = "factor: " + g_setup_err; return st; }
        if (sf.ghost_gid != sa.ghost_gid) {
            g_setup_err = "nsm_setup: the factor couples to other ranks' columns that A does not";
            return NSM_ERR_PATTERN;
        }
    }
    if (cudaSetDevice(device) != cudaSuccess) { g_setup_err = "nsm_setup: cudaSetDevice failed"; return NSM_ERR_CUDA; }
    // load every kernel now: a lazy load during a spinning halo wait would stall
    preload_plain_kernels();
    preload_tma_kernels();
    preload_halo_kernels();
    preload_fused_kernels();
    preload_fused_w_kernels();
    preload_coupled_kernels();
    nsm_handle *h = new nsm_handle();
    h->uid = next_handle_uid();
    h->device = device;
    h->n = sa.n;
    h->row_begin = rb;
    h->n_ghost = sa.n_ghost;
    h->nnz_off = sa.nnz_off;
    h->nslices = (int)((sa.n + kSlice - 1) / kSlice);
    // PDL pays where kernels are short (C2: +5 %) and was measured to cost
    // 14 % on 16.7 M-row 7-point sweeps (profiles/r01_v5_pdl.md): default on
    // up to 8 M rows per rank
    h->pdl = sa.n <= (int64_t)8 * 1024 * 1024;
    h->rank = rank;
    h->nranks = nranks;
    h->mode = dist ? dist->mode : NSM_DIST_HYBRID;
    DevAlloc a{h};
    bool ok = a.get(&h->d, h->n) && upload(h->d, sa.d.data(), h->n) && a.get(&h->dl1, h->n) &&
              upload(h->dl1, sa.dl1.data(), h->n) && upload_sell(a, sa.L, &h->L) &&
              upload_sell(a, sa.U, &h->U) && upload_sell(a, sa.LG, &h->LG) && upload_sell(a, sa.UG, &h->UG);
    if (ok && F) {
        h->has_ilu = true;
        ok = a.get(&h->dU, h->n) && upload(h->dU, sf.d.data(), h->n) && upload_sell(a, sf.L, &h->Ls) &&
             upload_sell(a, sf.U, &h->Us) && upload_sell(a, sf.LG, &h->LsG) && upload_sell(a, sf.UG, &h->UsG);
    }
    if (ok) {  // gather windows (stream.cu): launches over tile-aligned slice ranges
        ok = make_window(a, h->n, {&sa.L, &sa.U}, &h->res_win) && make_window(a, h->n, {&sa.L}, &h->L.win) &&
             make_window(a, h->n, {&sa.U}, &h->U.win);
        if (ok && F) ok = make_window(a, h->n, {&sf.L}, &h->Ls.win) && make_window(a, h->n, {&sf.U}, &h->Us.win);
    }
    for (int i = 0; ok && i < 4; ++i) ok = a.get(&h->w[i], std::max<int64_t>(h->n, 1));
    ok = ok && a.get(&h->flag, 1) && a.get(&h->ghost_null, 1) && a.get(&h->d_dist_err, 1) &&
         cudaMemset(h->d_dist_err, 0, sizeof(unsigned int)) == cudaSuccess;
    if (ok) {
        unsigned long long init = ULLONG_MAX;
        ok = cudaMemcpy(h->flag, &init, sizeof(init), cudaMemcpyHostToDevice) == cudaSuccess;
    }
    if (ok && nranks == 1 && h->n > 0) {
        // dependency distances of the fused passes (fused.cu); their rings are
        // allocated when NSM_OPT_FUSED is switched on (fused_alloc)
        const int64_t tr = skew_tile_rows();
        auto tiles = [tr](int64_t bw) { return (int)((bw + tr - 1) / tr); };
        h->DLA = tiles(sa.bw_lower);
        h->DUA = tiles(sa.bw_upper);
        h->DLs = F ? tiles(sf.bw_lower) : 0;
        h->DUs = F ? tiles(sf.bw_upper) : 0;
        h->fused_possible = true;
        // PDL also pays for the windowed (27-point) kernels at any size: C3,
        // 3 reps, 1.3517 vs 1.3559 ms per application (tools/experiments/pdl_c3.sh;
        // 7-point and compact 16.7 M-row passes lose 1-3 %)
        if (h->res_win.wmax) h->pdl = true;
        ok = ok && coupled_alloc(a, h);
    }
    if (ok && nranks > 1) {
        h->row_offsets.assign(dist->row_offsets, dist->row_offsets + nranks + 1);
        h->ghost_gid = sa.ghost_gid;
        h->recv_off.assign(nranks + 1, 0);
        for (int q = 0; q <= nranks; ++q)
            h->recv_off[q] = (int64_t)(std::lower_bound(h->ghost_gid.begin(), h->ghost_gid.end(), h->row_offsets[q]) -
                                       h->ghost_gid.begin());
        // slices whose rows couple to ghosts are "boundary", the rest "interior"
        std::vector<int32_t> inner, bnd;
        for (int s = 0; s < h->nslices; ++s) {
            bool g = sa.LG.ptr[s + 1] > sa.LG.ptr[s] || sa.UG.ptr[s + 1] > sa.UG.ptr[s];
            (g ? bnd : inner).push_back(s);
        }
        h->n_interior = (int)inner.size();
        if (!inner.empty() && inner.back() - inner.front() + 1 == (int32_t)inner.size()) {
            h->interior_begin = inner.front();
            h->interior_end = inner.back() + 1;
        }
        h->n_boundary = (int)bnd.size();
        ok = a.get(&h->interior, h->n_interior) && upload(h->interior, inner.data(), h->n_interior) &&
             a.get(&h->boundary, h->n_boundary) && upload(h->boundary, bnd.data(), h->n_boundary);
        // neighbours we receive from (send side joins in nsm_halo_set_send)
        for (int q = 0; q < nranks; ++q)
            if (q != rank && h->recv_off[q + 1] > h->recv_off[q]) {
                Peer p;
                p.q = q;
                h->peers.push_back(p);
            }
        h->flags_bytes = flags_bytes_for(nranks);
        h->mailbox_bytes = h->flags_bytes + (size_t)2 * std::max<int64_t>(h->n_ghost, 1) * sizeof(double);
        ok = ok && cudaMalloc(&h->mailbox, h->mailbox_bytes) == cudaSuccess &&
             cudaMemset(h->mailbox, 0, h->mailbox_bytes) == cudaSuccess;
        if (ok) {
            h->device_bytes += (int64_t)h->mailbox_bytes;
            h->mb_flags = (unsigned long long *)h->mailbox;
            h->mb_data = (double *)((char *)h->mailbox + h->flags_bytes);
        }
    }
    if (!ok) {
        cudaGetLastError();
        g_setup_err = "nsm_setup: device allocation or upload failed";
        free_handle(h);
        return NSM_ERR_OOM;
    }
    *out = h;
    return NSM_OK;
}

// Single-rank set-up from a DEVICE CSR: the split / SELL-32 packing runs on
// the GPU (builder_gpu.cu) and yields the same arrays as nsm_setup's host
// builder; the rest of the handle is assembled as in nsm_setup.
nsm_status nsm_setup_device(nsm_handle **out, const nsm_csr *A, const nsm_csr *F, int device) {
    if (!out || !A) { g_setup_err = "nsm_setup_device: NULL argument"; return NSM_ERR_ARG; }
    *out = nullptr;
    if (A->ncols != A->nrows) { g_setup_err = "nsm_setup_device: A must be square"; return NSM_ERR_ARG; }
    if (F && (F->nrows != A->nrows || F->ncols != A->ncols)) {
        g_setup_err = "nsm_setup: F shape differs from A";
        return NSM_ERR_ARG;
    }
    if (cudaSetDevice(device) != cudaSuccess) { g_setup_err = "nsm_setup_device: cudaSetDevice failed"; return NSM_ERR_CUDA; }
    preload_plain_kernels();
    preload_tma_kernels();
    preload_halo_kernels();
    preload_fused_kernels();
    preload_fused_w_kernels();
    preload_coupled_kernels();
    nsm_handle *h = new nsm_handle();
    h->uid = next_handle_uid();
    h->device = device;
    DevSplit sa, sf;
    nsm_status st = build_split_device(A, &sa, &h->device_bytes, &g_setup_err);
    h->d = sa.d;
    h->dl1 = sa.dl1;
    h->L = sa.L;
    h->U = sa.U;
    if (st == NSM_OK && F) {
        st = build_split_device(F, &sf, &h->device_bytes, &g_setup_err);
        h->dU = sf.d;
        cudaFree(sf.dl1);
        h->Ls = sf.L;
        h->Us = sf.U;
        if (st != NSM_OK) g_setup_err = "factor: " + g_setup_err;
        h->has_ilu = st == NSM_OK;
    }
    if (st != NSM_OK) {
        free_handle(h);
        return st;
    }
    h->n = sa.n;
    h->nnz_off = sa.nnz_off;
    h->nslices = (int)((sa.n + kSlice - 1) / kSlice);
    h->pdl = sa.n <= (int64_t)8 * 1024 * 1024;  // as nsm_setup
    DevAlloc a{h};
    const int64_t ns = h->nslices;
    auto empty_part = [&](Sell *s) {  // no ghost couplings on one rank: zero slice pointers
        return a.get(&s->ptr, ns + 1) && cudaMemset(s->ptr, 0, (ns + 1) * sizeof(int64_t)) == cudaSuccess;
    };
    bool ok = empty_part(&h->LG) && empty_part(&h->UG) && (!F || (empty_part(&h->LsG) && empty_part(&h->UsG)));
    ok = ok && make_window(a, h->n, {&sa.Lh, &sa.Uh}, &h->res_win) && make_window(a, h->n, {&sa.Lh}, &h->L.win) &&
         make_window(a, h->n, {&sa.Uh}, &h->U.win);
    if (ok && F) ok = make_window(a, h->n, {&sf.Lh}, &h->Ls.win) && make_window(a, h->n, {&sf.Uh}, &h->Us.win);
    for (int i = 0; ok && i < 4; ++i) ok = a.get(&h->w[i], std::max<int64_t>(h->n, 1));
    ok = ok && a.get(&h->flag, 1) && a.get(&h->ghost_null, 1) && a.get(&h->d_dist_err, 1) &&
         cudaMemset(h->d_dist_err, 0, sizeof(unsigned int)) == cudaSuccess;
    if (ok) {
        unsigned long long init = ULLONG_MAX;
        ok = cudaMemcpy(h->flag, &init, sizeof(init), cudaMemcpyHostToDevice) == cudaSuccess;
    }
    if (ok && h->n > 0) {
        const int64_t tr = skew_tile_rows();
        auto tiles = [tr](int64_t bw) { return (int)((bw + tr - 1) / tr); };
        h->DLA = tiles(sa.bw_lower);
        h->DUA = tiles(sa.bw_upper);
        h->DLs = F ? tiles(sf.bw_lower) : 0;
        h->DUs = F ? tiles(sf.bw_upper) : 0;
        h->fused_possible = true;
        // PDL also pays for the windowed (27-point) kernels at any size: C3,
        // 3 reps, 1.3517 vs 1.3559 ms per application (tools/experiments/pdl_c3.sh;
        // 7-point and compact 16.7 M-row passes lose 1-3 %)
        if (h->res_win.wmax) h->pdl = true;
        ok = ok && coupled_alloc(a, h);
    }
    if (!ok) {
        cudaGetLastError();
        g_setup_err = "nsm_setup_device: device allocation failed";
        free_handle(h);
        return NSM_ERR_OOM;
    }
    *out = h;
    return NSM_OK;
}

// Copies of a handle's device arrays (diagnostics and the builder parity
// tests): part 0..7 = L, U, LG, UG, Ls, Us, LsG, UsG.
static const Sell *part_of(const nsm_handle *h, int part) {
    const Sell *p[8] = {&h->L, &h->U, &h->LG, &h->UG, &h->Ls, &h->Us, &h->LsG, &h->UsG};
    return part >= 0 && part < 8 ? p[part] : nullptr;
}

nsm_status nsm_part_info(const nsm_handle *h, int part, int64_t *padded, int64_t *nnz, int *maxw, int *aligned) {
    const Sell *s = h ? part_of(h, part) : nullptr;
    if (!s) return NSM_ERR_ARG;
    if (padded) *padded = s->padded;
    if (nnz) *nnz = s->nnz;
    if (maxw) *maxw = s->maxw;
    if (aligned) *aligned = s->off != nullptr;
    return NSM_OK;
}

nsm_status nsm_part_copy(const nsm_handle *h, int part, int64_t *ptr, int32_t *col, double *val, int32_t *off) {
    const Sell *s = h ? part_of(h, part) : nullptr;
    if (!s) return NSM_ERR_ARG;
    DeviceScope dev(h->device);
    const int64_t ns = h->nslices;
    bool ok = true;
    if (ptr && s->ptr) ok = cudaMemcpy(ptr, s->ptr, (ns + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost) == cudaSuccess;
    if (ok && col && s->padded) ok = cudaMemcpy(col, s->col, s->padded * sizeof(int32_t), cudaMemcpyDeviceToHost) == cudaSuccess;
    if (ok && val && s->padded) ok = cudaMemcpy(val, s->val, s->padded * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
    if (ok && off && s->off)
        ok = cudaMemcpy(off, s->off, s->padded / kSlice * sizeof(int32_t), cudaMemcpyDeviceToHost) == cudaSuccess;
    if (ok && ptr && !s->ptr) std::fill(ptr, ptr + ns + 1, (int64_t)0);
    return ok ? NSM_OK : NSM_ERR_CUDA;
}

nsm_status nsm_diag_copy(const nsm_handle *h, int which, double *out) {
    if (!h || !out || which < 0 || which > 2) return NSM_ERR_ARG;
    const double *src = which == 0 ? h->d : (which == 1 ? h->dl1 : h->dU);
    if (!src) return NSM_ERR_STATE;
    DeviceScope dev(h->device);
    return h->n == 0 || cudaMemcpy(out, src, h->n * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess ? NSM_OK
                                                                                                         : NSM_ERR_CUDA;
}

nsm_status nsm_halo_set_send(nsm_handle *h, int q, const int64_t *rows, int64_t count) {
    if (!h || q < 0 || q >= h->nranks || q == h->rank || count < 0 || (count > 0 && !rows)) return NSM_ERR_ARG;
    if (h->committed) { h->err = "nsm_halo_set_send after commit"; return NSM_ERR_STATE; }
    Peer *p = find_peer(h, q);
    if (!p) {
        if (count == 0) return NSM_OK;
        Peer np;
        np.q = q;
        h->peers.push_back(np);
        std::sort(h->peers.begin(), h->peers.end(), [](const Peer &a, const Peer &b) { return a.q < b.q; });
        p = find_peer(h, q);
    }
    p->send_rows.resize(count);
    for (int64_t i = 0; i < count; ++i) {
        int64_t l = rows[i] - h->row_begin;
        if (l < 0 || l >= h->n) {
            h->err = "nsm_halo_set_send: row " + std::to_string((long long)rows[i]) + " is not owned by this rank";
            return NSM_ERR_DIST;
        }
        p->send_rows[i] = (int32_t)l;
    }
    p->send_set = true;
    return NSM_OK;
}

nsm_status nsm_halo_mailbox(nsm_handle *h, void **base, void *ipc_handle, int64_t *recv_offsets) {
    if (!h || h->nranks < 2) return NSM_ERR_STATE;
    if (base) *base = h->mailbox;
    if (ipc_handle) {
        cudaIpcMemHandle_t ih;
        cudaSetDevice(h->device);
        cudaError_t e = cudaIpcGetMemHandle(&ih, h->mailbox);
        if (e != cudaSuccess) return cuda_fail(h, e, "cudaIpcGetMemHandle");
        std::memcpy(ipc_handle, &ih, sizeof(ih));
    }
    if (recv_offsets) std::copy(h->recv_off.begin(), h->recv_off.begin() + h->nranks, recv_offsets);
    return NSM_OK;
}

static nsm_status connect_common(nsm_handle *h, int q, void *peer_base, int64_t peer_n_ghost,
                                 int64_t peer_recv_off_for_us, void *ipc_base) {
    Peer *p = find_peer(h, q);
    if (!p) { h->err = "nsm_halo_connect: rank " + std::to_string(q) + " is not a neighbour"; return NSM_ERR_DIST; }
    const size_t fb = flags_bytes_for(h->nranks);
    p->remote_flags = (unsigned long long *)peer_base + h->rank;
    p->remote_data = (double *)((char *)peer_base + fb) + peer_recv_off_for_us;
    p->remote_stride = std::max<int64_t>(peer_n_ghost, 1);
    p->ipc_base = ipc_base;
    p->connected = true;
    return NSM_OK;
}

nsm_status nsm_halo_connect(nsm_handle *h, int q, void *peer_base, int64_t peer_n_ghost, int64_t peer_recv_off) {
    if (!h || !peer_base || q < 0 || q >= h->nranks) return NSM_ERR_ARG;
    return connect_common(h, q, peer_base, peer_n_ghost, peer_recv_off, nullptr);
}

nsm_status nsm_halo_connect_ipc(nsm_handle *h, int q, const void *ipc_handle, int64_t peer_n_ghost,
                                int64_t peer_recv_off) {
    if (!h || !ipc_handle || q < 0 || q >= h->nranks) return NSM_ERR_ARG;
    cudaSetDevice(h->device);
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, ipc_handle, sizeof(ih));
    void *ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaIpcOpenMemHandle");
    return connect_common(h, q, ptr, peer_n_ghost, peer_recv_off, ptr);
}

nsm_status nsm_halo_commit(nsm_handle *h) {
    if (!h || h->nranks < 2) return NSM_ERR_STATE;
    std::vector<PutDesc> desc;
    std::vector<int> ids;
    int blocks = 0;
    DevAlloc a{h};
    for (Peer &p : h->peers) {
        if (!p.connected) { h->err = "nsm_halo_commit: neighbour " + std::to_string(p.q) + " not connected"; return NSM_ERR_DIST; }
        int64_t cnt = (int64_t)p.send_rows.size();
        if (!a.get(&p.d_send_rows, cnt) || !upload(p.d_send_rows, p.send_rows.data(), cnt)) return NSM_ERR_OOM;
        PutDesc d{p.d_send_rows, cnt, p.remote_data, p.remote_stride, p.remote_flags, put_blocks(cnt), blocks};
        blocks += d.nblocks;
        desc.push_back(d);
        ids.push_back(p.q);
    }
    h->put_grid = blocks;
    int np = (int)desc.size();
    if (np > 0) {
        if (!a.get(&h->d_put, np) || !upload(h->d_put, desc.data(), np) || !a.get(&h->d_peer_ids, np) ||
            !upload(h->d_peer_ids, ids.data(), np) || !a.get(&h->d_counters, np) ||
            cudaMemset(h->d_counters, 0, np * sizeof(unsigned int)) != cudaSuccess)
            return NSM_ERR_OOM;
    }
    // side stream for the put (overlaps the interior kernel, see pass())
    DeviceScope dev(h->device);
    if (np > 0 && !h->side &&
        (cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking) != cudaSuccess ||
         cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
         cudaEventCreateWithFlags(&h->ev_put, cudaEventDisableTiming) != cudaSuccess)) {
        cudaGetLastError();
        h->err = "nsm_halo_commit: stream / event creation failed";
        return NSM_ERR_CUDA;
    }
    h->committed = true;
    return NSM_OK;
}

void nsm_destroy(nsm_handle *h) { free_handle(h); }

nsm_status nsm_set_option(nsm_handle *h, nsm_option opt, int64_t value) {
    if (!h) return NSM_ERR_ARG;
    DeviceScope dev(h->device);
    ++h->cfg_gen;
    switch (opt) {
        case NSM_OPT_PIPELINE: h->pipeline = value != 0; return NSM_OK;
        case NSM_OPT_FUSED:
            if (value < 0 || value > 3) return NSM_ERR_ARG;
            h->fused_mode = (int)value;
            return value ? fused_alloc(h) : NSM_OK;
        case NSM_OPT_FUSED_WINDOW:
            if (value < 0 || value > INT_MAX) return NSM_ERR_ARG;
            h->skew_dw = (int)value;
            return NSM_OK;
        case NSM_OPT_PDL: h->pdl = value != 0; return NSM_OK;
        case NSM_OPT_WINDOW: h->window = value != 0; return NSM_OK;
        case NSM_OPT_HOST_CHUNKS: h->chunked_host = value != 0; return NSM_OK;
        case NSM_OPT_PLANE_ROWS:
            if (value < 0 || value % 256) return NSM_ERR_ARG;
            h->plane_tiles = 0;
            if (value > 0 && fw_possible(h) && planes_ok(h, value / 256)) h->plane_tiles = value / 256;
            if (value > 0 && !h->plane_tiles) {
                h->err = "NSM_OPT_PLANE_ROWS: the matrix does not have the plane structure (or no gather windows)";
                return NSM_ERR_PATTERN;
            }
            if (h->fw_ready) {  // the rings were sized without the plane schedule
                const FusedWShape sp = fw_shape(h, kMaxPhW - 1, true);
                if (!sp.ok || sp.Mr > h->fw_Mr || sp.Mg > h->fw_Mg) h->plane_tiles = 0;
            }
            return NSM_OK;
        case NSM_OPT_PROFILE:
            h->profile = value != 0;
            if (h->profile && h->ev.empty()) {
                h->ev.resize(2 * 4096);
                for (cudaEvent_t &e : h->ev) cudaEventCreate(&e);
                h->ev_kind.assign(4096, 0);
            }
            h->ev_used = 0;
            return NSM_OK;
        case NSM_OPT_COUPLED:
            if (value < 0 || value > INT_MAX) return NSM_ERR_ARG;
            h->coupled = (int)value;
            return NSM_OK;
        case NSM_OPT_HALO_TIMEOUT_MS:
            if (value <= 0) return NSM_ERR_ARG;
            h->timeout_ns = (unsigned long long)value * 1000000ull;
            return NSM_OK;
    }
    return NSM_ERR_ARG;
}

nsm_status nsm_set_comm(nsm_handle *h, nsm_comm *c) {
    if (!h) return NSM_ERR_ARG;
    if (c && (comm_rank(c) != h->rank || comm_nranks(c) != h->nranks || comm_device(c) != h->device)) {
        h->err = "nsm_set_comm: the communicator's rank, rank count or device differs from the handle's";
        return NSM_ERR_ARG;
    }
    h->comm = c;
    ++h->cfg_gen;
    return NSM_OK;
}

nsm_status nsm_info(const nsm_handle *h, int64_t *n_local, int64_t *n_ghost, int64_t *nnz_offdiag,
                    int64_t *device_bytes) {
    if (!h) return NSM_ERR_ARG;
    if (n_local) *n_local = h->n;
    if (n_ghost) *n_ghost = h->n_ghost;
    if (nnz_offdiag) *nnz_offdiag = h->nnz_off;
    if (device_bytes) *device_bytes = h->device_bytes;
    return NSM_OK;
}

nsm_status nsm_profile(nsm_handle *h, double *ms, int64_t *count) {
    if (!h || !ms || !count) return NSM_ERR_ARG;
    for (int k = 0; k < 3; ++k) { ms[k] = 0.0; count[k] = 0; }
    for (int i = 0; i < h->ev_used; ++i) {
        float t = 0.f;
        if (cudaEventSynchronize(h->ev[2 * i + 1]) != cudaSuccess ||
            cudaEventElapsedTime(&t, h->ev[2 * i], h->ev[2 * i + 1]) != cudaSuccess)
            return cuda_fail(h, cudaGetLastError(), "nsm_profile");
        ms[h->ev_kind[i]] += t;
        count[h->ev_kind[i]] += 1;
    }
    h->ev_used = 0;
    return NSM_OK;
}

nsm_status nsm_ilut(const nsm_csr *A, double droptol, int lfil, int64_t *rowptr, int64_t *nnz, int64_t *colind,
                    double *val) {
    if (!A || !rowptr || !nnz) { g_setup_err = "nsm_ilut: NULL argument"; return NSM_ERR_ARG; }
    std::vector<int64_t> rp, ci;
    std::vector<double> va;
    nsm_status st = ilut_host(A, droptol, lfil, rp, ci, va, &g_setup_err);
    if (st != NSM_OK) return st;
    std::copy(rp.begin(), rp.end(), rowptr);
    *nnz = (int64_t)ci.size();
    if (colind) std::copy(ci.begin(), ci.end(), colind);
    if (val) std::copy(va.begin(), va.end(), val);
    return NSM_OK;
}

nsm_status nsm_ruiz(const nsm_csr *F, int max_iters, double *val, double *s_r, double *s_c) {
    if (!F || !val || !s_r || !s_c) { g_setup_err = "nsm_ruiz: NULL argument"; return NSM_ERR_ARG; }
    return ruiz_host(F, max_iters, val, s_r, s_c, &g_setup_err);
}

nsm_status nsm_ruiz_dep(const nsm_csr *F, int max_iters, double dep_tol, double *val, double *s_r, double *s_c,
                        int *iters, double *dep_hist) {
    if (!F || !val || !s_r || !s_c || dep_tol < 0.0) { g_setup_err = "nsm_ruiz_dep: bad argument"; return NSM_ERR_ARG; }
    return ruiz_host(F, max_iters, val, s_r, s_c, &g_setup_err, dep_tol, iters, dep_hist);
}

nsm_status nsm_dep(const nsm_csr *F, const double *val, int upper, nsm_dep_info *out) {
    return dep_host(F, val, upper, out, &g_setup_err);
}

nsm_status nsm_set_ruiz(nsm_handle *h, const double *s_r, const double *s_c) {
    if (!h || !h->has_ilu) return NSM_ERR_STATE;
    DeviceScope dev(h->device);
    ++h->cfg_gen;
    if (!s_r || !s_c) {
        h->ruiz = false;
        return NSM_OK;
    }
    DevAlloc a{h};
    if (!h->s_r && !(a.get(&h->s_r, std::max<int64_t>(h->n, 1)) && a.get(&h->s_c, std::max<int64_t>(h->n, 1))))
        return NSM_ERR_OOM;
    if (!upload(h->s_r, s_r, h->n) || !upload(h->s_c, s_c, h->n)) return cuda_fail(h, cudaGetLastError(), "nsm_set_ruiz");
    h->ruiz = true;
    return NSM_OK;
}

nsm_status nsm_layout(const nsm_handle *h, int *offset_aligned) {
    if (!h || !offset_aligned) return NSM_ERR_ARG;
    *offset_aligned = (h->L.off ? 1 : 0) | (h->U.off ? 2 : 0) | (h->Ls.off ? 4 : 0) | (h->Us.off ? 8 : 0) |
                      (h->res_win.wmax ? 16 : 0) | (h->L.win.wmax ? 32 : 0) | (h->U.win.wmax ? 64 : 0);
    return NSM_OK;
}

nsm_status nsm_fused_stats(nsm_handle *h, int64_t *waits, int64_t *wait_ns) {
    if (!h || !waits || !wait_ns) return NSM_ERR_ARG;
    *waits = 0;
    *wait_ns = 0;
    DeviceScope dev(h->device);
    if (h->skew_sync) {
        SkewSync v{};
        cudaError_t e = cudaMemcpy(&v, h->skew_sync, sizeof(v), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(h, e, "nsm_fused_stats");
        *waits += (int64_t)v.waits;
        *wait_ns += (int64_t)v.wait_ns;
    }
    if (h->fw_sync) {  // one-pass windowed kernel: the producer's frontier polls
        unsigned long long v[4] = {0, 0, 0, 0};
        cudaError_t e = cudaMemcpy(v, h->fw_sync, sizeof(v), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(h, e, "nsm_fused_stats");
        *waits += (int64_t)v[2];
        *wait_ns += (int64_t)v[3];
    }
    return NSM_OK;
}

nsm_status nsm_fused_counters(const nsm_handle *h, int64_t *out) {
    if (!h || !out) return NSM_ERR_ARG;
    for (int i = 0; i < 6; ++i) out[i] = 0;
    if (!h->fw_sync) return NSM_OK;
    DeviceScope dev(h->device);
    unsigned long long v[8] = {};
    if (cudaMemcpy(v, h->fw_sync, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
        return NSM_ERR_CUDA;
    for (int i = 0; i < 6; ++i) out[i] = (int64_t)v[2 + i];
    return NSM_OK;
}

nsm_status nsm_coupled_counters(const nsm_handle *h, int64_t *out) {
    if (!h || !out) return NSM_ERR_ARG;
    for (int i = 0; i < 16; ++i) out[i] = 0;
    if (!h->cp_stats) return NSM_OK;
    DeviceScope dev(h->device);
    unsigned long long v[16] = {};
    if (cudaMemcpy(v, h->cp_stats, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return NSM_ERR_CUDA;
    for (int i = 0; i < 16; ++i) out[i] = (int64_t)v[i];
    return NSM_OK;
}

nsm_status nsm_stats(const nsm_handle *h, int64_t *kernel_launches, int64_t *halo_exchanges) {
    if (!h) return NSM_ERR_ARG;
    if (kernel_launches) *kernel_launches = h->launches;
    if (halo_exchanges) *halo_exchanges = h->exchanges;
    return NSM_OK;
}

nsm_status nsm_residual(nsm_handle *h, const double *b, const double *x, double *r, void *stream) {
    if (!h) return NSM_ERR_ARG;
    if ((h->n > 0 && (!b || !x || !r)) || overlap(r, b, h->n) || overlap(r, x, h->n)) {
        h->err = "nsm_residual: NULL or aliased vector";
        return NSM_ERR_ARG;
    }
    DeviceScope dev(h->device);
    return residual_into(h, b, x, r, OUT_R, S(stream));
}

nsm_status nsm_spmv(nsm_handle *h, const double *x, double *y, void *stream) {
    if (!h) return NSM_ERR_ARG;
    if ((h->n > 0 && (!x || !y)) || overlap(x, y, h->n)) { h->err = "nsm_spmv: NULL or aliased vector"; return NSM_ERR_ARG; }
    DeviceScope dev(h->device);
    return residual_into(h, nullptr, x, y, OUT_AX, S(stream));
}

static nsm_status tri_solve(nsm_handle *h, bool lower, const double *r, double *x, int k, void *stream) {
    if (!h) return NSM_ERR_ARG;
    if (k < 0 || (h->n > 0 && (!r || !x)) || overlap(r, x, h->n)) {
        h->err = lower ? "nsm_lsolve: bad argument (k < 0, NULL or aliased vector)"
                       : "nsm_usolve: bad argument (k < 0, NULL or aliased vector)";
        return NSM_ERR_ARG;
    }
    DeviceScope dev(h->device);
    cudaStream_t s = S(stream);
    Stage stg;
    if (h->has_ilu) stg = lower ? Stage{&h->Ls, &h->LsG, nullptr, r, k} : Stage{&h->Us, &h->UsG, h->dU, r, k};
    else stg = lower ? Stage{&h->L, &h->LG, h->d, r, k} : Stage{&h->U, &h->UG, h->d, r, k};
    if (k == 0) return scale_into(h, false, r, stg.dT, x, s);
    return run_sweeps(h, stg, h->w[0], h->w[1], EPI_STORE, x, nullptr, nullptr, s);
}

nsm_status nsm_lsolve(nsm_handle *h, const double *r, double *x, int k, void *stream) {
    return tri_solve(h, true, r, x, k, stream);
}
nsm_status nsm_usolve(nsm_handle *h, const double *r, double *x, int k, void *stream) {
    return tri_solve(h, false, r, x, k, stream);
}

// One fused phase-skewed pass (fused.cu) if the handle allows it for this
// shape: fused_mode 1 always, 2 (auto) when the problem spans at least two
// skew distances.  *ran tells whether it was launched.
static nsm_status skew_run(nsm_handle *h, SkewLaunch &L, bool unit, int DT, int DA, cudaStream_t s, bool *ran) {
    *ran = false;
    if (!h->fused_ready || h->fused_mode == 0 || !h->pipeline || L.k < 1 || L.k > nsm_handle::kFusedKmax ||
        h->n == 0)
        return NSM_OK;
    const bool resid = L.ph0 == SKEW_RESID;
    L.shape = skew_shape(L.ph0, unit, resid ? h->L.maxw : 0, resid ? h->U.maxw : 0, L.T->maxw, L.k, h->n, DT, DA,
                         h->skew_dw);
    const SkewShape &sh = L.shape;
    if (!sh.ok || sh.Mr > h->ring_r_tiles || sh.Mg > h->ring_g_tiles || sh.grid > 4096) return NSM_OK;
    if (h->fused_mode == 2 && sh.nbig < 2 * (int64_t)sh.D) return NSM_OK;
    L.n = h->n;
    if (unit) L.dT = nullptr;
    L.ring_r = h->ring_r;
    L.ring_g = h->ring_g;
    L.flag = h->flag;
    L.sweep_id0 = h->sweep_counter + 1;
    h->sweep_counter += L.k;
    L.err = h->d_dist_err;
    L.timeout_ns = h->timeout_ns;
    L.sync = h->skew_sync;
    L.prog = h->skew_prog;
    ProfScope prof(h, 2, s);
#ifdef NSM_EXPERIMENTS
    // debug: per-unit timestamps of two CTAs, summarised on stderr
    static unsigned long long *trace = nullptr;
    static const bool want_trace = knob("NSM_DEBUG_SKEW_TRACE") != nullptr;
    if (want_trace && !trace) {
        cudaMalloc(&trace, 2 * 3 * 2048 * 4 * sizeof(unsigned long long));
    }
    if (want_trace) cudaMemsetAsync(trace, 0, 2 * 3 * 2048 * 4 * sizeof(unsigned long long), s);
    L.trace = want_trace ? trace : nullptr;
#else
    L.trace = nullptr;
#endif
    cudaError_t e = launch_skew(L, s);
#ifdef NSM_EXPERIMENTS
    if (want_trace && e == cudaSuccess) {
        std::vector<unsigned long long> tb(2 * 3 * 2048 * 4);
        cudaStreamSynchronize(s);
        cudaMemcpy(tb.data(), trace, tb.size() * 8, cudaMemcpyDeviceToHost);
        for (int cta = 0; cta < 2; ++cta) {
            // consumer warp 0: slot 0 full-wait start, 1 data ready, 2 unit done;
            // per item: slot 0 made ready, 1 published
            const unsigned long long *C = tb.data() + (cta * 3 + 0) * 2048 * 4;
            const unsigned long long *Y = tb.data() + (cta * 3 + 2) * 2048 * 4;
            const unsigned long long t0 = C[0];
            double full_wait = 0, compute = 0, gaps = 0;
            int nu = 0;
            for (int u = 0; u < 2048 && C[u * 4 + 2]; ++u, ++nu) {
                full_wait += (double)(C[u * 4 + 1] - C[u * 4 + 0]);
                compute += (double)(C[u * 4 + 2] - C[u * 4 + 1]);
                if (u > 0) gaps += (double)(C[u * 4 + 0] - C[u * 4 - 2]);
            }
            fprintf(stderr, "[skew trace] cta %d: %d units: full-wait %.1f us, unit work %.1f us, between units %.1f us\n",
                    cta, nu, full_wait / 1e3, compute / 1e3, gaps / 1e3);
            if (cta == 0) {
                for (int m = 0; m < 6; ++m)
                    fprintf(stderr, "   item %d ready at %.0f ns, published at %.0f ns\n", m,
                            Y[m * 4] ? (double)(Y[m * 4] - t0) : -1.0, Y[m * 4 + 1] ? (double)(Y[m * 4 + 1] - t0) : -1.0);
                for (int u = 0; u < 8 && u < nu; ++u)
                    fprintf(stderr, "   unit %d: wait %.0f..%.0f done %.0f ns\n", u, (double)(C[u * 4] - t0),
                            (double)(C[u * 4 + 1] - t0), (double)(C[u * 4 + 2] - t0));
            }
        }
    }
#endif
    ++h->launches;
    if (e != cudaSuccess) return cuda_fail(h, e, "fused pass launch");
    *ran = true;
    return NSM_OK;
}

// One smoother application of the given kind (rows a2-a5).  fresh: x is
// taken as 0 (its contents are ignored), so the residual is b (reading R3)
// and the last kernel STORES x instead of adding to it.
// One pGS application as ONE windowed pass (fused_w.cu), when the handle has
// the rings (NSM_OPT_FUSED) and the matrix is stencil-like.
static nsm_status fused_w_run(nsm_handle *h, const double *b, double *x, int k, bool fresh, cudaStream_t s, bool *ran) {
    *ran = false;
    if (!h->fw_ready || h->fused_mode != 3 || !h->pipeline || !h->window || k < 1 || k > kMaxPhW - 1 || h->n == 0)
        return NSM_OK;
    FusedWLaunch L{};
    L.shape = fw_shape(h, k, h->plane_tiles > 0);
    if (h->plane_tiles > 0 && !L.shape.ok) L.shape = fw_shape(h, k, false);  // (k = 1: the item schedule)
    const FusedWShape &sh = L.shape;
    if (!sh.ok || sh.Mr > h->fw_Mr || sh.Mg > h->fw_Mg || sh.grid > kFwProgStride) return NSM_OK;
    L.n = h->n;
    L.k = k;
    L.DT = h->DLA;
    L.DA = std::max(h->DLA, h->DUA);
    L.fresh = fresh ? 1 : 0;
    L.Lp = &h->L;
    L.Up = &h->U;
    L.wu = &h->U.win;
    L.tposL = h->fw_tpos[0];
    L.tposU = h->fw_tpos[1];
    L.nsegL = h->fw_nseg[0];
    L.nsegU = h->fw_nseg[1];
    L.tsegL = h->fw_tseg[0];
    L.tsegU = h->fw_tseg[1];
    L.pst = h->fw_pst;
    L.wl = &h->L.win;
    L.d = h->d;
    L.b = b;
    L.x = x;
    L.ring_r = h->fw_ring_r;
    L.ring_g = h->fw_ring_g;
    L.prog = h->fw_prog;
    L.pstride = kFwProgStride;
    L.flag = h->flag;
    L.sweep_id0 = h->sweep_counter + 1;
    h->sweep_counter += k;
    L.err = h->d_dist_err;
    L.timeout_ns = h->timeout_ns;
    L.sync = h->fw_sync;
    ProfScope prof(h, 2, s);
    const cudaError_t e = launch_fused_w(L, s);
    ++h->launches;
    if (e != cudaSuccess) return cuda_fail(h, e, "one-pass fused launch");
    *ran = true;
    return NSM_OK;
}

// Forward pGS application with k = 2, 3: the residual pass (r, g(0)), then
// the k sweeps as concurrent warp groups of one kernel (coupled.cu): one
// rank, offset-aligned L with a gather window; *ran = false otherwise.
static nsm_status coupled_run(nsm_handle *h, const double *b, double *x, int k, cudaStream_t s, bool *ran) {
    *ran = false;
    if (!h->coupled || !h->cp_prog || distributed(h) || !h->pipeline || !h->window || k < 2 || k > 3 || h->n == 0 ||
        !h->L.off || !h->L.win.wmax)
        return NSM_OK;
    CoupledLaunch L{};
    L.shape = coupled_shape(h->L.maxw, h->L.win.wmax, k, h->n);
    if (!L.shape.ok) return NSM_OK;
    double *R = h->w[0], *W0 = h->w[1], *W1 = h->w[2], *W2 = h->w[3];
    nsm_status st = residual_into(h, b, x, R, OUT_RG, s, W2);
    if (st != NSM_OK) return st;
    L.n = h->n;
    L.Lp = &h->L;
    L.wl = &h->L.win;
    L.d = h->d;
    L.r = R;
    L.x = x;
    L.g[0] = W2;
    L.g[1] = W0;
    L.g[2] = W1;
    L.prog = h->cp_prog;
    L.pstride = kCpProgStride;
    L.sync = h->cp_sync;
    L.flag = h->flag;
    L.sweep_id0 = h->sweep_counter + 1;
    L.err = h->d_dist_err;
    L.timeout_ns = h->timeout_ns;
    L.lag = h->coupled > 1 ? h->coupled : 0;
    L.stats = h->profile ? h->cp_stats : nullptr;
    ProfScope prof(h, 1, s);
    const cudaError_t e = launch_coupled(L, s);
    if (e != cudaSuccess) return cuda_fail(h, e, "coupled sweeps launch");
    h->sweep_counter += k;
    ++h->launches;
    *ran = true;
    return NSM_OK;
}

static nsm_status apply_once(nsm_handle *h, nsm_kind kind, const double *b, double *x, int k_l, int k_u, bool fresh,
                             cudaStream_t s) {
    double *R = h->w[0], *W0 = h->w[1], *W1 = h->w[2], *W2 = h->w[3];
    const double *rhs = fresh ? b : R;
    nsm_status st = NSM_OK;
    bool ran = false;
    if (kind == NSM_L1_JACOBI) {
        // l1-Jacobi: x += D_l1^{-1} (b - A x)
        if (!fresh) st = residual_into(h, b, x, R, OUT_R, s);
        return st != NSM_OK ? st : scale_into(h, !fresh, rhs, h->dl1, x, s);
    }
    if (kind == NSM_PGS || kind == NSM_PGS_BACKWARD) {
        const bool fwd = kind == NSM_PGS;
        if (fwd && k_l >= 1) {  // stencil-like matrices: the one-pass windowed kernel
            st = fused_w_run(h, b, x, k_l, fresh, s, &ran);
            if (st != NSM_OK || ran) return st;
        }
        if (k_l >= 1) {
            // rows a2-a4 in ONE pass over the matrix: residual, k sweeps, x update
            SkewLaunch L{};
            L.desc = !fwd;
            L.k = k_l;
            L.T = fwd ? &h->L : &h->U;
            L.dT = h->d;
            if (!fresh) {
                L.ph0 = SKEW_RESID;
                L.A0 = &h->L;
                L.A1 = &h->U;
                L.dA = h->d;
                L.b = b;
                L.xin = x;
                L.keep0 = fwd;   // the swept triangle is re-read by the later phases
                L.keep1 = !fwd;
                L.epi = SKEW_XADD;
                L.x = x;
            } else {
                L.ph0 = SKEW_NONE;  // r = b, g(0) = b / d gathered on the fly
                L.rhs = b;
                L.g0 = b;
                L.scaled_g0 = 1;
                L.epi = SKEW_STORE;
                L.out1 = x;
            }
            const int DT = fwd ? h->DLA : h->DUA;
            st = skew_run(h, L, false, DT, DT, s, &ran);
            if (st != NSM_OK || ran) return st;
        }
        if (fwd && !fresh) {  // rows a2-a4: residual, then the sweeps as concurrent warp groups (coupled.cu)
            st = coupled_run(h, b, x, k_l, s, &ran);
            if (st != NSM_OK || ran) return st;
        }
        // the residual pass also writes g^(0) = r / d (eq:jr-initial-guess)
        // when sweeps follow, so the first sweep gathers it instead of
        // dividing per gathered entry
        const bool rg = !fresh && k_l > 0;
        if (!fresh) st = residual_into(h, b, x, R, rg ? OUT_RG : OUT_R, s, rg ? W2 : nullptr);
        if (st != NSM_OK) return st;
        // rows a3/a4: k_l sweeps g <- D^{-1}(r - T g) (T = L forward, U
        // backward), the last fused with x += g
        if (k_l == 0) return scale_into(h, !fresh, rhs, h->d, x, s);
        Stage sg = fwd ? Stage{&h->L, &h->LG, h->d, rhs, k_l, rg ? W2 : nullptr}
                       : Stage{&h->U, &h->UG, h->d, rhs, k_l, rg ? W2 : nullptr};
        return fresh ? run_sweeps(h, sg, W0, W1, EPI_STORE, x, nullptr, nullptr, s)
                     : run_sweeps(h, sg, W0, W1, EPI_XADD, nullptr, x, nullptr, s);
    }
    // NSM_ILU0, row a5: y = sum_{j<=kL} (-Ls)^j r ; z = sum_{j<=kU} (-DU^{-1}Us)^j DU^{-1} y ; x += z.
    // With Ruiz (Alg. 2): y~ = y / s_r, v = U~^{-1} y~ (unit
    // diagonal), x += v / s_c.
    const bool ruiz = h->ruiz;
    const double *y = nullptr, *z0 = nullptr;  // after the L stage: rhs of the U sweeps, materialised z^(0)
    // ---- L stage (with the residual): one fused ascending pass
    if (k_l >= 1 && !(ruiz && k_u == 0)) {
        SkewLaunch L{};
        L.desc = 0;
        L.k = k_l;
        L.T = &h->Ls;
        if (!fresh) {
            L.ph0 = SKEW_RESID;
            L.A0 = &h->L;
            L.A1 = &h->U;
            L.dA = h->d;
            L.b = b;
            L.xin = x;
        } else {
            L.ph0 = SKEW_NONE;  // r = y(0) = b
            L.rhs = b;
            L.g0 = b;
        }
        if (ruiz) { L.epi = SKEW_STORE_SCALE; L.out1 = W2; L.dn = h->s_r; }
        else if (k_u >= 1) { L.epi = SKEW_STORE2; L.out1 = W0; L.out2 = W2; L.dn = h->dU; }
        else if (fresh) { L.epi = SKEW_STORE_SCALE; L.out1 = x; L.dn = h->dU; }
        else { L.epi = SKEW_XADD_SCALE; L.x = x; L.dn = h->dU; }
        st = skew_run(h, L, true, h->DLs, h->DLA, s, &ran);
        if (st != NSM_OK) return st;
        if (ran) {
            if (!ruiz && k_u == 0) return NSM_OK;
            y = ruiz ? W2 : W0;
            z0 = ruiz ? nullptr : W2;
        }
    }
    if (!y) {
        if (!fresh) st = residual_into(h, b, x, R, OUT_R, s);
        if (st != NSM_OK) return st;
        if (ruiz) {
            if (k_l > 0) {
                double *ybuf = (k_l & 1) ? W0 : W1;
                st = run_sweeps(h, Stage{&h->Ls, &h->LsG, nullptr, rhs, k_l}, W0, W1, EPI_STORE2, ybuf, nullptr,
                                h->s_r, s, W2);
            } else {
                st = scale_into(h, false, rhs, h->s_r, W2, s);
            }
            if (st != NSM_OK) return st;
            if (k_u == 0) return scale_into(h, !fresh, W2, h->s_c, x, s);
            y = W2;
        } else if (k_l > 0) {
            // L sweeps ping-pong in W0/W1; the last writes y and, when U sweeps
            // follow, z^(0) = y / dU into W2 (EPI_STORE2)
            double *ybuf = (k_l & 1) ? W0 : W1;
            Stage sl{&h->Ls, &h->LsG, nullptr, rhs, k_l};
            if (k_u == 0)
                return fresh ? run_sweeps(h, sl, W0, W1, EPI_STORE2, W2, nullptr, h->dU, s, x)   // x = y / dU
                             : run_sweeps(h, sl, W0, W1, EPI_XADD_SCALE, nullptr, x, h->dU, s);
            st = run_sweeps(h, sl, W0, W1, EPI_STORE2, ybuf, nullptr, h->dU, s, W2);
            if (st != NSM_OK) return st;
            z0 = W2;
            y = ybuf;
        } else if (k_u == 0) {
            return scale_into(h, !fresh, rhs, h->dU, x, s);
        } else {
            y = rhs;
        }
    }
    // ---- U stage: one fused descending pass
    {
        SkewLaunch L{};
        L.ph0 = SKEW_NONE;
        L.desc = 1;
        L.k = k_u;
        L.T = &h->Us;
        L.dT = h->dU;
        L.rhs = y;
        L.g0 = z0 ? z0 : y;
        L.scaled_g0 = z0 ? 0 : 1;
        if (ruiz) {
            L.dn = h->s_c;
            if (fresh) { L.epi = SKEW_STORE_SCALE; L.out1 = x; }
            else { L.epi = SKEW_XADD_SCALE; L.x = x; }
        } else if (fresh) {
            L.epi = SKEW_STORE;
            L.out1 = x;
        } else {
            L.epi = SKEW_XADD;
            L.x = x;
        }
        st = skew_run(h, L, false, h->DUs, 0, s, &ran);
        if (st != NSM_OK || ran) return st;
    }
    if (ruiz) {
        Stage su{&h->Us, &h->UsG, h->dU, W2, k_u, nullptr};
        return fresh ? run_sweeps(h, su, W0, W1, EPI_STORE2, R, nullptr, h->s_c, s, x)
                     : run_sweeps(h, su, W0, W1, EPI_XADD_SCALE, nullptr, x, h->s_c, s);
    }
    // z ping-pong in buffers holding neither y nor (for the first U sweep) z^(0)
    double *za, *zb;
    if (y == W0) { za = W1; zb = W2; }
    else if (y == W1) { za = W0; zb = W2; }
    else { za = W0; zb = W1; }
    Stage su{&h->Us, &h->UsG, h->dU, y, k_u, z0};
    return fresh ? run_sweeps(h, su, za, zb, EPI_STORE, x, nullptr, nullptr, s)
                 : run_sweeps(h, su, za, zb, EPI_XADD, nullptr, x, nullptr, s);
}

nsm_status nsm_smooth(nsm_handle *h, nsm_kind kind, const double *b, double *x, int nu, int k_l, int k_u,
                      int x_is_zero, void *stream) {
    if (!h) return NSM_ERR_ARG;
    if (nu < 0 || k_l < 0 || (kind == NSM_ILU0 && k_u < 0) || (h->n > 0 && (!b || !x)) || overlap(b, x, h->n)) {
        h->err = "nsm_smooth: bad argument (negative count, NULL or aliased vector)";
        return NSM_ERR_ARG;
    }
    if (kind < NSM_PGS || kind > NSM_L1_JACOBI) { h->err = "nsm_smooth: unknown kind"; return NSM_ERR_ARG; }
    if (kind == NSM_ILU0 && !h->has_ilu) { h->err = "nsm_smooth: ILU0 requested on a handle without factors"; return NSM_ERR_STATE; }
    DeviceScope dev(h->device);
    cudaStream_t s = S(stream);
    for (int it = 0; it < nu; ++it) {
        const bool fresh = it == 0 && x_is_zero;
        nsm_status st;
        if (kind == NSM_PGS_SYMMETRIC) {
            st = apply_once(h, NSM_PGS, b, x, k_l, k_u, fresh, s);
            if (st == NSM_OK) st = apply_once(h, NSM_PGS_BACKWARD, b, x, k_l, k_u, false, s);
        } else {
            st = apply_once(h, kind, b, x, k_l, k_u, fresh, s);
        }
        if (st != NSM_OK) return st;
    }
    return NSM_OK;
}

// nsm_smooth_host for one forward pGS application on one rank, in row
// chunks (tile-aligned, each longer than A's bandwidth) so that the
// host-to-device copies of b and x, the passes and the device-to-host copy
// of x overlap.  Chunk c's residual needs x of chunks c-1 .. c+1 (unmodified:
// the x update of chunk c-1 is launched after it); sweep j of chunk c-1 needs
// g(j-1) of chunks c-2 and c-1, each level in its own buffer (k <= 3).  Same
// kernels and per-row arithmetic as nsm_smooth: bit-identical results.
static nsm_status smooth_host_chunked(nsm_handle *h, const double *b_host, const double *x_in_host, double *x_out_host,
                                      int k, cudaStream_t s, bool *done) {
    *done = false;
    const int mwr = std::max(h->L.maxw, h->U.maxw);
    if (h->nranks != 1 || k < 1 || k > 3 || !h->pipeline || h->fused_mode != 0 || !tma_ok(2, mwr) ||
        wide_rows(mwr, h->nslices) || !tma_ok(1, h->L.maxw) || wide_rows(h->L.maxw, h->nslices))
        return NSM_OK;
    const int64_t nt = (h->n + 255) / 256;
    // chunk count, measured (tools/experiments/e2e_chunks.py, ms per step for
    // 8 / 12 / 16 / 24 / 32 / 48 chunks): C3 (27-point rows) 6.38 / 6.27 /
    // 6.30 / 5.93 / 5.95 / 6.27, C5 (7-point) 6.30 / 6.24 / 6.30 / 6.55 /
    // 6.90 / 6.78 — so 32 for wide rows, 12 for narrow ones (the copy pattern
    // alone takes 5.7 ms; one 256 MB + 128 MB copy pair 5.1)
    int64_t nchunks = h->nnz_off >= 16 * h->n ? 32 : 12;
    if (const char *v = knob("NSM_HOST_CHUNKS_N")) nchunks = std::max(3, atoi(v));   // experiments
    // tiles per chunk: longer than A's bandwidth (DLA / DUA, in 256-row
    // tiles), so chunk c's residual reads x only from chunks c - 1 .. c + 1
    // and never a row a finished sweep already updated
    const int64_t ct = std::max<int64_t>(std::max(h->DLA, h->DUA) + 1, (nt + nchunks - 1) / nchunks);
    const int64_t C = (nt + ct - 1) / ct;
    if (C < 3 || C > 64) return NSM_OK;
    if (!h->hs_in) {
        if (cudaStreamCreateWithFlags(&h->hs_in, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&h->hs_out, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            return NSM_OK;
        }
        h->hev.resize(2 * 64 + 2);
        for (cudaEvent_t &e : h->hev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                return NSM_OK;
            }
    }
    cudaEvent_t *hin = h->hev.data(), *fin = h->hev.data() + 64, ev0 = h->hev[128], ev1 = h->hev[129];
    auto rows = [&](int64_t c, int64_t &r0, int64_t &r1) {
        r0 = std::min(c * ct * 256, h->n);
        r1 = std::min((c + 1) * ct * 256, h->n);
    };
    auto slices = [&](int64_t c, int64_t &s0, int64_t &s1) {
        s0 = std::min<int64_t>(c * ct * kTileSlices, h->nslices);
        s1 = std::min<int64_t>((c + 1) * ct * kTileSlices, h->nslices);
    };
    double *R = h->w[0], *G0 = h->w[3], *G1 = h->w[1], *G2 = h->w[2];
    double *gbuf[3] = {G0, G1, G2};
    double *xd = h->hx_dev, *bd = h->hb_dev;
    cudaError_t e = cudaEventRecord(ev0, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->hs_in, ev0, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->hs_out, ev0, 0);
    for (int64_t c = 0; c < C && e == cudaSuccess; ++c) {  // all host-to-device copies, in chunk order
        int64_t r0, r1;
        rows(c, r0, r1);
        const size_t nb = (size_t)(r1 - r0) * sizeof(double);
        e = cudaMemcpyAsync(bd + r0, b_host + r0, nb, cudaMemcpyHostToDevice, h->hs_in);
        if (e == cudaSuccess) e = cudaMemcpyAsync(xd + r0, x_in_host + r0, nb, cudaMemcpyHostToDevice, h->hs_in);
        if (e == cudaSuccess) e = cudaEventRecord(hin[c], h->hs_in);
    }
    if (e != cudaSuccess) return cuda_fail(h, e, "nsm_smooth_host (chunked copies in)");
    const int64_t sid0 = h->sweep_counter + 1;
    h->sweep_counter += k;
    for (int64_t c = 0; c <= C; ++c) {
        if (c < C) {  // residual of chunk c (needs x of chunks c-1 .. c+1)
            e = cudaStreamWaitEvent(s, hin[std::min(c + 1, C - 1)], 0);
            int64_t s0, s1;
            slices(c, s0, s1);
            if (e == cudaSuccess)
                e = launch_residual_tma(h->window && h->res_win.wmax ? &h->res_win : nullptr, OUT_RG, h->n, s0, s1,
                                        h->L, h->U, h->d, bd, xd, R, G0, false, s);
            ++h->launches;
        }
        if (c >= 1 && e == cudaSuccess) {  // the k sweeps of chunk c-1, the last with x += g
            int64_t s0, s1;
            slices(c - 1, s0, s1);
            for (int j = 1; j <= k && e == cudaSuccess; ++j) {
                SweepArgs sa{};
                sa.n = h->n;
                sa.nslices = h->nslices;
                sa.T = &h->L;
                sa.TG = &h->LG;
                sa.unit = false;
                sa.epi = j == k ? EPI_XADD : EPI_STORE;
                sa.dT = h->d;
                sa.rhs = R;
                sa.gin = gbuf[j - 1];
                sa.gout = j < k ? gbuf[j] : nullptr;
                sa.x = xd;
                sa.flag = h->flag;
                sa.sweep_id = sid0 + j - 1;
                sa.pdl = false;
                sa.win = h->window && h->L.win.wmax ? &h->L.win : nullptr;
                e = launch_sweep_tma(sa, s0, s1, s);
                ++h->launches;
            }
            if (e == cudaSuccess) e = cudaEventRecord(fin[c - 1], s);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(h->hs_out, fin[c - 1], 0);
            int64_t r0, r1;
            rows(c - 1, r0, r1);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(x_out_host + r0, xd + r0, (size_t)(r1 - r0) * sizeof(double),
                                    cudaMemcpyDeviceToHost, h->hs_out);
        }
        if (e != cudaSuccess) return cuda_fail(h, e, "nsm_smooth_host (chunked passes)");
    }
    e = cudaEventRecord(ev1, h->hs_out);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev1, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(h, e, "nsm_smooth_host (device to host)");
    *done = true;
    return NSM_OK;
}

nsm_status nsm_smooth_host(nsm_handle *h, nsm_kind kind, const double *b_host, const double *x_in_host,
                           double *x_out_host, int nu, int k_l, int k_u, int x_is_zero, void *stream) {
    if (!h) return NSM_ERR_ARG;
    if (h->n > 0 && (!b_host || !x_out_host || (!x_is_zero && !x_in_host))) {
        h->err = "nsm_smooth_host: NULL host vector";
        return NSM_ERR_ARG;
    }
    if (overlap(b_host, x_out_host, h->n) || (!x_is_zero && overlap(b_host, x_in_host, h->n))) {
        h->err = "nsm_smooth_host: b aliases x";
        return NSM_ERR_ARG;
    }
    if (!x_is_zero && x_in_host != x_out_host && overlap(x_in_host, x_out_host, h->n)) {
        h->err = "nsm_smooth_host: x_in and x_out partially overlap";
        return NSM_ERR_ARG;
    }
    if (nu == 0) {  // no application: the result is the start vector
        if (h->n > 0) {
            if (x_is_zero) std::memset(x_out_host, 0, (size_t)h->n * sizeof(double));
            else if (x_out_host != x_in_host) std::memcpy(x_out_host, x_in_host, (size_t)h->n * sizeof(double));
        }
        return NSM_OK;
    }
    DeviceScope dev(h->device);
    const size_t bytes = (size_t)std::max<int64_t>(h->n, 1) * sizeof(double);
    if (!h->hb_dev) {
        cudaError_t e = cudaMalloc(&h->hb_dev, bytes);
        if (e == cudaSuccess) e = cudaMalloc(&h->hx_dev, bytes);
        if (e != cudaSuccess) {
            cudaFree(h->hb_dev);
            h->hb_dev = h->hx_dev = nullptr;
            cudaGetLastError();
            h->err = "nsm_smooth_host: staging allocation failed";
            return NSM_ERR_OOM;
        }
    }
    cudaStream_t s = S(stream);
    if (kind == NSM_PGS && nu == 1 && !x_is_zero && x_in_host != x_out_host && h->chunked_host) {
        bool done = false;
        const nsm_status cst = smooth_host_chunked(h, b_host, x_in_host, x_out_host, k_l, s, &done);
        if (cst != NSM_OK || done) return cst;
    }
    const size_t nb = (size_t)h->n * sizeof(double);
    cudaError_t e = cudaSuccess;
    if (nb) {
        e = cudaMemcpyAsync(h->hb_dev, b_host, nb, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess && !x_is_zero) e = cudaMemcpyAsync(h->hx_dev, x_in_host, nb, cudaMemcpyHostToDevice, s);
    }
    if (e != cudaSuccess) return cuda_fail(h, e, "nsm_smooth_host (host to device)");
    const nsm_status st = nsm_smooth(h, kind, h->hb_dev, h->hx_dev, nu, k_l, k_u, x_is_zero, stream);
    if (st != NSM_OK) return st;
    if (nb) e = cudaMemcpyAsync(x_out_host, h->hx_dev, nb, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(h, e, "nsm_smooth_host (device to host)");
    return NSM_OK;
}

nsm_status nsm_check(nsm_handle *h, int64_t *first_bad_sweep, void *stream) {
    if (!h) return NSM_ERR_ARG;
    DeviceScope dev(h->device);
    cudaError_t e = cudaStreamSynchronize(S(stream));
    if (e != cudaSuccess) return cuda_fail(h, e, "nsm_check");
    unsigned long long v = 0, init = ULLONG_MAX;
    unsigned int derr = 0;
    e = cudaMemcpy(&v, h->flag, sizeof(v), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(h->flag, &init, sizeof(init), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && h->d_dist_err) {
        e = cudaMemcpy(&derr, h->d_dist_err, sizeof(derr), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemset(h->d_dist_err, 0, sizeof(unsigned int));
    }
    if (e != cudaSuccess) return cuda_fail(h, e, "nsm_check");
    if (first_bad_sweep) *first_bad_sweep = v == ULLONG_MAX ? -1 : (int64_t)v;
    if (derr) {
        h->err = (derr & 1u) ? "halo exchange timed out waiting for a neighbour"
                             : "fused pass timed out waiting for an earlier work item";
        return NSM_ERR_DIST;
    }
    if (v != ULLONG_MAX) {
        h->err = "non-finite value produced by sweep " + std::to_string((long long)v);
        return NSM_ERR_NONFINITE;
    }
    return NSM_OK;
}

}  // extern "C"
