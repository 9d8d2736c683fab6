// nsm_internal.h — device data layout shared by the builder, the kernels and
// the C-ABI glue of libnsm.so (DESIGN.md §5 "Data layout in HBM").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/nsm.h"

// Experiment knobs (the A/B scripts under tools/experiments) exist only in a
// build with -DNSM_EXPERIMENTS; the product build reads no environment
// variable (knob() is a constant nullptr and the branches fold away).
#ifdef NSM_EXPERIMENTS
#include <cstdlib>
inline const char *knob(const char *name) { return std::getenv(name); }
#else
inline const char *knob(const char *) { return nullptr; }
#endif

namespace nsm {

constexpr int kSlice = 32;  // SELL-C slice height = warp width: one thread per row
constexpr int kTileSlices = 8;  // slices per tile of the pipelined kernels (stream.cu)

// Gather window of the pipelined kernels for offset-aligned parts (stream.cu
// "windowed" variants): for every tile of kTileSlices slices, the columns its
// rows gather (row + offset over the group's parts) merged into a few
// contiguous segments of the gathered vector, bulk-copied into shared memory
// with the tile, so the gathers become shared-memory loads.  Segment k of
// tile t: global first index glo[k] (even; may reach below 0 / past n at the
// ends of the matrix: the producer zero-fills those positions), length len[k]
// (even), start sbase[k] in the tile's window.  wpos[p][ptr[s]/32 + j] = the
// window index of lane 0's gather of entry j of slice s of part p (lane l
// adds l).  wmax = 0: no window (compact layout, or a window too large).
struct Window {
    int32_t *tseg = nullptr;   // ntiles + 1: first segment of tile t
    int64_t *glo = nullptr;
    int32_t *len = nullptr, *sbase = nullptr;
    int32_t *wpos[2] = {nullptr, nullptr};
    int32_t wmax = 0;          // largest window of a tile, in doubles
    int32_t maxseg = 0;        // most segments of a tile
};
struct WindowHost {
    std::vector<int32_t> tseg, len, sbase;
    std::vector<int64_t> glo;
    std::vector<int32_t> wpos[2];
    int32_t wmax = 0, maxseg = 0;
};
struct WinView {
    const int32_t *tseg;
    const int64_t *glo;
    const int32_t *len, *sbase;
    const int32_t *wpos[2];
    int32_t wcap;              // window capacity per stage (doubles, >= wmax)
};

// One strictly-triangular (or ghost) part in SELL-32 form (σ = 1: rows keep
// their order).  Slice s holds rows [32 s, 32 s + 32); its entries occupy
// [ptr[s], ptr[s+1]) laid out column-major: entry j of lane l at
// ptr[s] + 32 j + l.  Width w_s = (ptr[s+1]-ptr[s]) / 32 = longest row of
// the slice; shorter rows are padded with val = 0 and col = a valid index.
// Within a row the entries are in ascending column order.
struct Sell {
    int64_t *ptr = nullptr;   // device, nslices + 1
    int32_t *col = nullptr;   // device, padded entries
    double *val = nullptr;    // device, padded entries
    // Offset-aligned layout (stencil-like parts, builder.cpp pack_aligned):
    // entry j of every row of slice s has column row + off[ptr[s]/32 + j]
    // (a pad where the row lacks that offset: val 0, col = row + off if in
    // range, else the row).  nullptr: compact layout, columns only in `col`.
    int32_t *off = nullptr;
    int64_t padded = 0;       // stored entries incl. padding
    int64_t nnz = 0;          // real entries
    int32_t maxw = 0;         // widest slice
    Window win;               // gather window of sweeps over this part alone (offset-aligned only)
    bool empty() const { return padded == 0; }
};

// Host-side staging of a Sell before upload.
struct SellHost {
    std::vector<int64_t> ptr;
    std::vector<int32_t> col;
    std::vector<double> val;
    std::vector<int32_t> off;   // offset-aligned layout (empty: compact)
    int64_t nnz = 0;
    int32_t maxw = 0;
};

// What the kernels need of one part: raw pointers (kernel argument).
struct SellView {
    const int64_t *ptr;
    const int32_t *col;
    const double *val;
    const int32_t *off;
};

inline SellView view(const Sell &s) { return SellView{s.ptr, s.col, s.val, s.off}; }

// Gather-window plan of offset-aligned parts (builder.cpp): false if a
// tile's window would exceed wcap doubles or 32 segments.
bool build_window(int64_t n, const std::vector<const SellHost *> &parts, int32_t wcap, WindowHost *out);

// Result of splitting a CSR row block (builder.cpp).
struct Split {
    int64_t n = 0, row_begin = 0, n_ghost = 0;
    std::vector<double> d;            // diagonal of A (or of U for factors)
    std::vector<double> dl1;          // a_ii + sum_{j != i} |a_ij| (l1-Jacobi diagonal)
    SellHost L, U;                    // strict lower / upper, LOCAL columns
    SellHost LG, UG;                  // couplings to ghost columns below / above the block
    std::vector<int64_t> ghost_gid;   // global id of ghost k (ascending)
    int64_t nnz_off = 0;
    int64_t bw_lower = 0, bw_upper = 0;  // max (i - j) over L entries, max (j - i) over U entries
};

// The same split built on the device from a DEVICE CSR (builder_gpu.cu;
// single rank: no ghost parts).  d, dl1 and the parts are device memory owned
// by the caller afterwards; Lh / Uh hold host copies of the slice pointers and
// offsets (the gather-window plans are built from them).
struct DevSplit {
    int64_t n = 0, nnz_off = 0, bw_lower = 0, bw_upper = 0;
    double *d = nullptr, *dl1 = nullptr;
    Sell L, U;
    SellHost Lh, Uh;
};
nsm_status build_split_device(const nsm_csr *A, DevSplit *out, int64_t *device_bytes, std::string *err);

// Builds the SELL split of rows [row_begin, row_begin + n) of A.
//   unit_lower: the strictly-lower part belongs to a unit-lower factor (the
//               stored diagonal is the U factor's; used for ILU factors).
// Returns NSM_OK or an error with a message.
nsm_status build_split(const nsm_csr *A, int64_t row_begin, int64_t row_end, Split *out, std::string *err);

// ---- kernel launchers (kernels.cu) ------------------------------------------
// Sweep epilogues (see k_sweep in kernels.cu).
enum { EPI_STORE = 0, EPI_XADD = 1, EPI_STORE2 = 2, EPI_XADD_SCALE = 3 };

struct SweepArgs {
    int64_t n;
    int nslices;
    const int32_t *list;     // slice list or nullptr (= all slices 0..nslices-1)
    const Sell *T, *TG;      // local strict triangle, ghost part (or nullptr)
    int has_ghost;           // 0: none, 1: TG columns precede T's (lower), 2: follow (upper)
    bool unit;               // unit diagonal: no division
    int epi;
    bool gin_scaled;         // gather rhs[c]/dT[c] instead of gin[c] (first sweep)
    const double *dT, *rhs, *gin, *ghost;
    double *gout, *x;
    const double *dnext;
    double *gout2;
    unsigned long long *flag;
    int64_t sweep_id;
    bool pdl;                // programmatic dependent launch (pipelined kernels)
    const Window *win;       // gather window of T over the full slice range (or nullptr)
};

// Residual kernel output modes.
enum { OUT_R = 0, OUT_AX = 1, OUT_RG = 2 };
cudaError_t launch_residual(int out_mode, int64_t n, int nslices, const int32_t *list, const Sell &LG,
                            const Sell &L, const Sell &U, const Sell &UG, bool has_ghost, const double *d,
                            const double *b, const double *x, const double *ghost, double *out, double *out2,
                            bool pdl, cudaStream_t st);
cudaError_t launch_sweep(const SweepArgs &a, cudaStream_t st);
// Wide rows on a small level (coarse AMG levels): the plain launchers use one
// warp per row; the pipelined kernels are not used for them.
bool wide_rows(int maxw, int64_t nslices);
cudaError_t launch_scale(bool xadd, int64_t n, const double *rhs, const double *d, double *out,
                         unsigned long long *flag, int64_t sweep_id, bool pdl, cudaStream_t st);

// ---- halo exchange (halo.cu) --------------------------------------------------
// One outgoing message: entries rows[0..count) of the sent vector go to
// remote[parity * remote_stride + e] in the neighbour's mailbox; the last of
// the nblocks blocks writing it publishes the exchange's sequence number at
// remote_flag.  block0 = first block of this peer in the put grid.
struct PutDesc {
    const int32_t *rows;
    int64_t count;
    double *remote;
    int64_t remote_stride;
    unsigned long long *remote_flag;
    int nblocks;
    int block0;
};

int put_blocks(int64_t count);
cudaError_t launch_halo_put(const PutDesc *desc, int npeers, int total_blocks, const double *src,
                            const double *scale, int parity, unsigned long long seq, unsigned int *counters,
                            cudaStream_t st);
cudaError_t launch_halo_wait(const unsigned long long *flags, const int *peers, int npeers, unsigned long long seq,
                             unsigned long long timeout_ns, unsigned int *dist_err, cudaStream_t st);

// ---- bulk-copy pipelined kernels (stream.cu), contiguous slice ranges --------
bool tma_ok(int np, int maxw);
// win: gather window of (L, U) for the full slice range (or nullptr).
cudaError_t launch_residual_tma(const Window *win, int out_mode, int64_t n, int64_t s_begin, int64_t s_end, const Sell &L,
                                const Sell &U, const double *d, const double *b, const double *x, double *out,
                                double *out2, bool pdl, cudaStream_t st);
cudaError_t launch_sweep_tma(const SweepArgs &a, int64_t s_begin, int64_t s_end, cudaStream_t st);

// ---- phase-skewed fused passes (fused.cu) ---------------------------------------
enum { SKEW_RESID = 0, SKEW_NONE = 1 };  // phase 0 = residual r = b - A x; none (rhs, g(0) given)
enum { SKEW_STORE = 0, SKEW_XADD = 1, SKEW_STORE2 = 2, SKEW_XADD_SCALE = 3, SKEW_STORE_SCALE = 4 };

// Launch state in device memory (zeroed at setup except epoch = 1; reset by
// the last CTA of every launch).
struct SkewSync {
    unsigned long long ctr, wmark;  // (reserved)
    unsigned int epoch;         // tag of the progress counters in the current launch
    unsigned int exits;         // CTAs finished
    unsigned long long waits;   // statistics (cumulative, nsm_fused_stats): item waits that had to spin,
    unsigned long long wait_ns; //   and their total spin time
};

struct SkewShape {
    bool ok = false;
    const void *kernel = nullptr;
    int nst = 0, grid = 0, D = 0, Dw = 0;
    size_t smem = 0;
    int64_t cap0 = 0, cap1 = 0, stage_bytes = 0, ntiles = 0, nitems = 0;
    int64_t Mr = 0, Mg = 0;     // ring lengths in 256-row tiles (powers of two)
    int B = 1;                  // 256-row tiles per scheduling tile
    int64_t nbig = 0;           // scheduling tiles
};

// ph0 = SKEW_RESID: maxw0 / maxw1 = widths of A's strict lower / upper parts;
// DT = bandwidth of the swept triangle in tiles, DA = A's (for the in-place x);
// dw_override > 0 replaces the automatic wait distance (tests).
SkewShape skew_shape(int ph0, bool unit, int maxw0, int maxw1, int maxwT, int k, int64_t n, int DT, int DA,
                     int dw_override);
int skew_tile_rows();

struct SkewLaunch {
    SkewShape shape;
    int64_t n;
    int ph0, desc, k, epi, scaled_g0, keep0, keep1;
    const Sell *A0, *A1, *T;
    const double *dA, *b, *xin;     // phase 0
    const double *dT, *rhs, *g0;    // sweeps (rhs, g0: full vectors when ph0 = SKEW_NONE)
    double *x, *out1, *out2;
    const double *dn;
    double *ring_r, *ring_g;
    unsigned long long *flag;
    int64_t sweep_id0;
    unsigned int *err;
    unsigned long long timeout_ns;
    SkewSync *sync;
    unsigned long long *prog;       // >= grid per-CTA progress counters (zeroed at setup)
    unsigned long long *trace;      // debug timestamps or nullptr
};
cudaError_t launch_skew(const SkewLaunch &L, cudaStream_t st);
void preload_fused_kernels();

// ---- one-pass windowed pGS (fused_w.cu) ---------------------------------------
constexpr int kMaxPhW = 5;   // phases 0..k, k <= 4
struct FusedWShape {
    bool ok = false;
    const void *kernel = nullptr;
    int nst = 0, grid = 0, D = 0;
    size_t smem = 0;
    int64_t cap = 0, wcap = 0, stage_bytes = 0, ntiles = 0, nitems = 0;
    int64_t Mr = 0, Mg = 0;   // ring lengths in 256-row tiles (powers of two)
    int64_t tpp = 0, nplanes = 0;  // plane schedule (k_fused_pgs_planes): tiles per plane, planes
};
// maxw: widest slice of L and U; wmax: largest window (residual or L);
// DT, DA: bandwidths of L and A in 256-row tiles; d_extra: D - max(DT, DA)
// (0 = automatic).
// tpp > 0: the plane-wavefront schedule with tpp tiles per plane (k >= 2).
FusedWShape fused_w_shape(int maxw, int64_t wmax, int k, int64_t n, int DT, int DA, int d_extra, int64_t tpp = 0);
struct FusedWLaunch {
    FusedWShape shape;
    int64_t n;
    int k, DT, DA, fresh;
    const Sell *Lp, *Up;
    const Window *wu, *wl;          // gather windows of U and L (each alone)
    const int32_t *tposL, *tposU, *nsegL, *nsegU;   // per-tile tables (fused_w_tables)
    const int4 *tsegL, *tsegU;
    int pst;
    const double *d, *b;
    double *x;
    double *ring_r, *ring_g;
    unsigned long long *prog;
    int64_t pstride;
    unsigned long long *flag;
    int64_t sweep_id0;
    unsigned int *err;
    unsigned long long timeout_ns;
    unsigned int *sync;
};
cudaError_t launch_fused_w(const FusedWLaunch &L, cudaStream_t st);
// per-tile padded tables of window w of part T (pst >= 8 * T.maxw positions per tile)
cudaError_t fused_w_tables(int64_t n, const Sell &T, const Window &w, int pst, int32_t *tpos, int32_t *nseg,
                           int4 *tseg);
void preload_fused_w_kernels();
// plane structure of L and U for the plane wavefront (tpp tiles per plane)
bool fused_w_plane_check(int64_t n, int64_t tpp, const Sell &L, const Sell &U);

// ---- coupled sweeps (coupled.cu) ------------------------------------------------
// The k = 2, 3 sweeps of a forward pGS application as concurrent CTA groups of
// one cooperative kernel: offset-aligned L with a gather window, one rank.
struct CoupledShape {
    bool ok = false;
    const void *kernel = nullptr;
    int threads = 0, k = 0;
    int64_t cap = 0, wcap = 0, stage = 0;   // entries / window doubles / bytes per stage
};
// maxw_l: widest slice of L; wcap: largest L window (doubles)
CoupledShape coupled_shape(int maxw_l, int64_t wcap, int k, int64_t n);
struct CoupledLaunch {
    CoupledShape shape;
    int64_t n;
    const Sell *Lp;
    const Window *wl;                // L's gather window
    const double *d, *r;
    double *x;                       // updated in place
    double *g[3];                    // g(0) (from the residual), then scratch iterates
    unsigned long long *prog;        // [k][pstride], zero-initialised once
    int64_t pstride;
    unsigned int *sync;              // [0] epoch, [1] CTAs finished
    unsigned long long *flag;
    int64_t sweep_id0;
    unsigned int *err;
    unsigned long long timeout_ns;
    int64_t lag;                     // group 0's throttle distance in tiles (0: automatic)
    unsigned long long *stats;       // nullable: 16 cycle counters (nsm_coupled_counters)
};
cudaError_t launch_coupled(const CoupledLaunch &L, cudaStream_t st);
void preload_coupled_kernels();

// Force-load every kernel of the library (see kernels.cu "eager loading").
void preload_plain_kernels();
void preload_tma_kernels();
void preload_halo_kernels();
void preload_solver_kernels();

// True for handles of a multi-rank partition (their launches carry halo
// sequence numbers and must not be captured into a replayed CUDA graph).
bool nsm_is_distributed(const nsm_handle *h);
// Unique id of a handle (never reused, unlike its address).
uint64_t nsm_handle_uid(const nsm_handle *h);
// Device ordinal of a handle; the cross-rank reduction attached to it
// (nsm_set_comm), or nullptr.
int nsm_handle_device(const nsm_handle *h);
nsm_comm *nsm_handle_comm(const nsm_handle *h);
// comm.cu: device-side all-reduce (sum, ascending rank order) of m doubles;
// comm_failed reads the mapped error word (after a stream synchronisation).
nsm_status comm_allreduce(nsm_comm *c, const double *in, double *out, int64_t m, cudaStream_t s);
bool comm_failed(const nsm_comm *c);
int comm_rank(const nsm_comm *c);
int comm_nranks(const nsm_comm *c);
int64_t comm_capacity(const nsm_comm *c);
int comm_device(const nsm_comm *c);

// Configuration generation of a handle: bumped by every nsm_set_option /
// nsm_set_ruiz, so a replayed graph can tell that its launch sequence is stale.
uint64_t nsm_handle_cfg_gen(const nsm_handle *h);

// The C-ABI calls run on their object's device: make it current for the
// call and give the caller back its own current device afterwards
// (cudaGetDevice is a thread-local read).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceScope(const DeviceScope &) = delete;
    DeviceScope &operator=(const DeviceScope &) = delete;
};

// Host ILUT(droptol, lfil) and Ruiz scaling of the U factor (NEXT-3).
nsm_status ilut_host(const nsm_csr *A, double droptol, int lfil, std::vector<int64_t> &rp_out,
                     std::vector<int64_t> &ci_out, std::vector<double> &va_out, std::string *err);
nsm_status ruiz_host(const nsm_csr *F, int max_iters, double *v, double *s_r, double *s_c, std::string *err,
                     double dep_tol = 0.0, int *iters_done = nullptr, double *dep_hist = nullptr);
nsm_status dep_host(const nsm_csr *F, const double *val, int upper, nsm_dep_info *out, std::string *err);

// ILU(0) by Chow-Patel fixed-point sweeps on the GPU (nsm_ilu0_fixed_point).
nsm_status ilu0_fixed_point_device(const nsm_csr *A, int64_t row_begin, int sweeps, double *fval, int device,
                                   std::string *err);

// Host ILU(0) (nsm_ilu0).
nsm_status ilu0_host(const nsm_csr *A, int64_t row_begin, double *fval, std::string *err);

}  // namespace nsm
