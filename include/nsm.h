/*
 * nsm.h — Neumann-series smoothers for B200 (sm_100a): the C-ABI boundary.
 *
 * The library implements the data-parallel hot path of arXiv 2112.14681
 * ("Neumann series in GMRES and algebraic multigrid smoothers", PAPER.md):
 * the sparse triangular solves inside the C-AMG smoothers are replaced by
 * SpMV-only Jacobi inner sweeps, i.e. truncated Neumann series.
 *
 *   polynomial Gauss-Seidel (§5.2):
 *       r = b - A x ;  g0 = D^{-1} r ;  g_{j+1} = D^{-1}(r - L g_j) (k times) ;
 *       x = x + g_k  =  x + sum_{j=0..k} (-D^{-1}L)^j D^{-1} r
 *   ILU(0) with Jacobi-iterated factor solves (§5.3, Alg. 2 P:L1020-1045 with
 *   the LDU row scaling of P:L858-874 / P:L1012-1013 in place of Ruiz):
 *       r = b - A x ;  y = sum_{j<=kL} (-L_s)^j r ;
 *       z = sum_{j<=kU} (-D_U^{-1} U_s)^j D_U^{-1} y ;  x = x + z
 *
 * Sweep-count convention (reading R1): k counts products with the
 * strict triangle AFTER the diagonally scaled start, so k sweeps give k+1
 * Neumann terms and k = 0 is pure diagonal scaling (Jacobi).
 *
 * Conventions for every call:
 *   - Matrices enter as HOST CSR (nsm_csr), 0-based, int64 row pointers and
 *     GLOBAL int64 column ids, columns strictly ascending within a row.  The
 *     library copies what it needs at setup and never retains the pointers.
 *   - Vectors (b, x, r) are DEVICE pointers to fp64 arrays of length n_local
 *     (the handle's row count), caller-owned, on the handle's device.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Hot calls are asynchronous on that stream, never allocate and
 *     never synchronise; their return value only reports argument and launch
 *     errors.  Divergence (a non-finite value produced by a sweep) is recorded
 *     in a sticky device flag and reported by nsm_check().
 *   - A handle owns device workspace: it must not be used concurrently from
 *     two streams.  Distinct handles are independent.
 *   - All arithmetic is fp64.  Each row sum is accumulated sequentially in
 *     ascending column order without FMA contraction and D^{-1} is an IEEE
 *     division, the same rounding sequence the oracle uses (R10).
 */
#ifndef NSM_H
#define NSM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nsm_handle nsm_handle;

typedef enum {
    NSM_OK = 0,
    NSM_ERR_ARG = 1,        /* bad argument: NULL pointer, negative count, aliasing */
    NSM_ERR_PATTERN = 2,    /* CSR invariant violated: rowptr not monotone, columns
                               unsorted/duplicated/out of range, factor not triangular */
    NSM_ERR_ZERO_DIAG = 3,  /* missing or zero diagonal / pivot (row in nsm_last_error) */
    NSM_ERR_NONFINITE = 4,  /* a sweep produced Inf/NaN (divergence) */
    NSM_ERR_CUDA = 5,       /* CUDA runtime error (message in nsm_last_error) */
    NSM_ERR_OOM = 6,        /* device or host allocation failed */
    NSM_ERR_STATE = 7,      /* call not valid for this handle (e.g. ILU call on a pGS handle) */
    NSM_ERR_DIST = 8        /* halo plan / peer connection error */
} nsm_status;

typedef enum {
    NSM_PGS = 0,          /* polynomial Gauss-Seidel, forward (M = D + L), §5.2 */
    NSM_ILU0 = 1,         /* ILU(0) with Jacobi-iterated L and U solves, §5.3 / Alg. 2 */
    NSM_PGS_BACKWARD = 2, /* polynomial GS with M = D + U (eq:one-stage backward) */
    NSM_PGS_SYMMETRIC = 3,/* one forward then one backward pGS application per outer iteration */
    NSM_L1_JACOBI = 4     /* l1-Jacobi, x += D_l1^{-1}(b - A x), D_l1 = a_ii + sum_{j!=i} |a_ij|
                             (the paper's comparison smoother; definition) */
} nsm_kind;

typedef enum {
    NSM_DIST_HYBRID = 0, /* hypre's hybrid smoother: the x halo is exchanged
                            once per outer iteration for the residual; the inner sweeps
                            drop couplings to other ranks (block-Jacobi across ranks) */
    NSM_DIST_GLOBAL = 1  /* exact global Neumann sweeps: the lower (L sweeps) or upper
                            (U sweeps) ghost values of the inner iterate are exchanged
                            before every sweep; the result does not depend on the
                            partition */
} nsm_dist_mode;

/* HOST CSR block: rows [row_begin, row_begin + nrows) of an ncols-column
 * matrix (row_begin comes from nsm_dist; 0 on a single GPU).  rowptr has
 * nrows + 1 entries starting at 0; colind holds GLOBAL column ids. */
typedef struct {
    int64_t nrows;
    int64_t ncols;
    const int64_t *rowptr;
    const int64_t *colind;
    const double *val;
} nsm_csr;

/* Row-block partition.  HOST array
 * row_offsets[nranks + 1], ascending, row_offsets[0] = 0: rank q owns global
 * rows [row_offsets[q], row_offsets[q+1]).  The CSR passed to nsm_setup must
 * hold exactly this rank's rows. */
typedef struct {
    int rank;
    int nranks;
    const int64_t *row_offsets;
    nsm_dist_mode mode;
} nsm_dist;

/*
 * nsm_setup — build the split-triangular device storage (§8(a) row a1).
 *   A:    the system matrix (P:L717-721 splitting A = L + D + U).  Required.
 *   F:    NULL for pGS.  For ILU(0): the incomplete factors stored on ONE
 *         pattern (nsm_ilu0 output layout): strictly-lower entries = L_s of
 *         the unit-lower L = I + L_s, upper entries incl. the
 *         diagonal = U = D_U (I + D_U^{-1} U_s).  Rows/columns as A.
 *   dist: NULL on one GPU; else this rank's place in the row partition.
 *   device: CUDA device ordinal the handle lives on.
 * Validates both matrices synchronously (NSM_ERR_PATTERN / NSM_ERR_ZERO_DIAG
 * with the offending global row in nsm_last_error(NULL)), copies them to the
 * device as SELL-32 slices and allocates all workspace.  On
 * failure *out is NULL.  Synchronous w.r.t. the host.
 */
nsm_status nsm_setup(nsm_handle **out, const nsm_csr *A, const nsm_csr *F, const nsm_dist *dist,
                     int device);

/*
 * nsm_ilu0 — ILU(0) factorisation on the host (setup input for nsm_setup;
 * not on the timed path).  IKJ variant restricted to the
 * pattern of A, no pivoting.  `fval` (length nnz(A), caller-allocated HOST
 * memory) receives the factor values on A's pattern in the layout nsm_setup
 * expects for F.  With a dist partition of nranks > 1 pass the rank's own
 * rows and row_begin: the factorisation is of the diagonal block A_pp
 * (block-Jacobi ILU, HYBRID reading R5) and off-block entries get 0.
 * Zero pivot -> NSM_ERR_ZERO_DIAG.
 */
nsm_status nsm_ilu0(const nsm_csr *A, int64_t row_begin, double *fval);

/*
 * nsm_ilu0_fixed_point — ILU(0) factor values computed ON THE GPU by
 * Chow-Patel fixed-point sweeps (the set-up algorithm the paper plans for
 * reducing C-AMG set-up cost; reading
 * R19).  The factors solve (LU)_ij = a_ij on pattern(A) (L unit lower); each
 * synchronous sweep updates every entry from the previous sweep,
 *   l_ij = (a_ij - sum_{k<j} l_ik u_kj) / u_jj,   u_ij = a_ij - sum_{k<i} l_ik u_kj,
 * starting from l_ij = a_ij / a_jj, u_ij = a_ij.  `sweeps` = 0 returns that
 * initial guess; once `sweeps` reaches the dependency depth of the pattern
 * the result equals nsm_ilu0 bit for bit (same operations, same order); a
 * few sweeps give the approximate factors Chow and Patel use.  A is HOST CSR,
 * fval (length nnz(A), caller-allocated HOST memory) receives the values in
 * nsm_ilu0's layout (row_begin / off-block entries as there).  Runs on
 * `device`, synchronous.  Missing or zero diagonal, or a zero u_jj during the
 * sweeps -> NSM_ERR_ZERO_DIAG; unsorted columns -> NSM_ERR_PATTERN.
 */
nsm_status nsm_ilu0_fixed_point(const nsm_csr *A, int64_t row_begin, int sweeps, double *fval, int device);

/*
 * nsm_ilut — ILUT(droptol, lfil) factorisation on the host (Saad's
 * dual-threshold ILU, "Compute A ~ LU with droptol and lfill imposed", Alg. 2
 * P:L1024-1025; single rank).  Row i: pivots eliminated in ascending column
 * order, L entries w_k / u_kk below droptol * ||a_i||_2 dropped, then every
 * off-diagonal entry below that threshold dropped and the lfil largest of the
 * L part and of the U part kept (ties: smaller column); the diagonal is kept.
 * Output: factor CSR on its own pattern (strict lower = L_s, upper incl.
 * diagonal = U), the layout nsm_setup takes as F.  rowptr (n+1) and *nnz are
 * always written; colind / val (nnz entries, caller-allocated) may be NULL to
 * query the size first.  Zero pivot -> NSM_ERR_ZERO_DIAG.
 */
nsm_status nsm_ilut(const nsm_csr *A, double droptol, int lfil, int64_t *rowptr, int64_t *nnz, int64_t *colind,
                    double *val);

/*
 * nsm_ruiz — Ruiz scaling of the U part of a factor CSR (Alg. 2 P:L1032;
 * P:L996-1008): max_iters rounds of sup-norm row/column equilibration, then an
 * exact unit diagonal.  val (same pattern as F) receives L_s unchanged and
 * U~ = diag(1/s_r) U diag(1/s_c); s_r, s_c (length n) receive the DIVISORS.
 */
nsm_status nsm_ruiz(const nsm_csr *F, int max_iters, double *val, double *s_r, double *s_c);

/*
 * nsm_ruiz_dep — nsm_ruiz with the early termination the paper proposes
 * (P:L1216-1228): after each round the departure from normality of the
 * current scaled U is computed, dep_hist[k] (NULL or max_iters + 1 entries;
 * k = 0 is the input) receives it, and the rounds stop once it is below
 * dep_tol (> 0; 0 = never, i.e. nsm_ruiz).  *iters (NULL ok) = rounds done.
 * For a triangular matrix dep = ||U_s||_F (its eigenvalues are its diagonal).
 */
nsm_status nsm_ruiz_dep(const nsm_csr *F, int max_iters, double dep_tol, double *val, double *s_r, double *s_c,
                        int *iters, double *dep_hist);

/*
 * nsm_dep — departure-from-normality diagnostics of a factor CSR's
 * triangle (host only): upper = 1 the U part (upper incl. diagonal), 0 the
 * unit-lower L (strict lower part + implicit unit diagonal).  val: values on
 * F's pattern (NULL = F->val; e.g. the nsm_ruiz output).
 *   dep          Henrici: sqrt(||T||_F^2 - ||eig(T)||^2) = ||T_s||_F
 *   fro, fro_strict   ||T||_F, ||T_s||_F
 *   delta        Definition 2: max_i max(0, sum_{j!=i}|t_ij| - |t_ii|)
 *   bound_thm3   Theorem 3: sqrt((2 sqrt(n) + nu) nu), nu = ||T_s||_F
 *   bound_table5 the same with nu = ||T||_F — how Table 5
 *                evaluates it (reading R20)
 *   bound_thm4   Theorem 4: sqrt(n) (1 + delta)
 * Theorems 3 and 4 assume a unit diagonal (a Ruiz-scaled U, or L).
 */
typedef struct {
    int64_t n;
    double dep, fro, fro_strict, delta, bound_thm3, bound_table5, bound_thm4;
} nsm_dep_info;
nsm_status nsm_dep(const nsm_csr *F, const double *val, int upper, nsm_dep_info *out);

/*
 * nsm_set_ruiz — make NSM_ILU0 smoothing use the Ruiz form of Alg. 2: the
 * handle's factor F must then hold U~ (nsm_ruiz output); after the L solve
 * y~ = y / s_r, the U~ solve runs on the unit-diagonal U~, and x += v / s_c
 * (P:L1032-1040).  s_r = s_c = NULL switches back.  Host arrays, length n.
 */
nsm_status nsm_set_ruiz(nsm_handle *h, const double *s_r, const double *s_c);

/* ---- multi-GPU halo plan (setup time) ---------
 * A handle set up with nranks > 1 owns a "mailbox" (device memory: one flag
 * per source rank + two parity copies of its ghost array) that its
 * neighbours write into directly over NVLink / NVSwitch.  Connecting a set of
 * ranks takes four host steps, all synchronous, done once after nsm_setup
 * (the Python binding does them with torch.distributed as plumbing):
 *   1. nsm_halo_plan: the global rows this rank needs from each rank (its
 *      ghost columns, ascending, grouped by owner).  Host-only: no device.
 *   2. nsm_halo_set_send(h, q, rows, count): the global rows (owned here) rank
 *      q needs — i.e. rank q's step-1 list for us.  Call for every q whose
 *      list is non-empty.
 *   3. nsm_halo_mailbox exports the mailbox (base pointer, a 64-byte
 *      cudaIpcMemHandle_t, and recv_offsets[q] = first ghost index owned by
 *      q); every neighbour q then calls nsm_halo_connect_ipc (other process)
 *      or nsm_halo_connect (same process and device) with it.
 *   4. nsm_halo_commit uploads the tables.  Hot calls that need an exchange
 *      before commit return NSM_ERR_STATE.
 * Exchanges are symmetric (every neighbour is signalled every time), so all
 * ranks must issue the same sequence of hot calls.  A neighbour that does
 * not answer within 20 s makes the waiting kernel give up; nsm_check then
 * reports NSM_ERR_DIST (no GPU hang).
 */

/* recv_counts[nranks] receives, per owner rank, how many ghost columns this
 * rank's rows reference; ghost_rows (NULL, or n_ghost entries) their global
 * ids ascending; *n_ghost their total.  The CSR is this rank's row block. */
nsm_status nsm_halo_plan(const nsm_csr *A, const nsm_dist *dist, int64_t *recv_counts, int64_t *ghost_rows,
                         int64_t *n_ghost);

/* The global rows owned by this rank that rank q needs (q's nsm_halo_plan
 * list for this rank).  NSM_ERR_DIST if a row is not owned here. */
nsm_status nsm_halo_set_send(nsm_handle *h, int q, const int64_t *rows, int64_t count);

/* Exports this rank's mailbox: *base (device pointer, may be NULL), the IPC
 * handle (64 bytes, may be NULL) and recv_offsets[nranks] (may be NULL). */
nsm_status nsm_halo_mailbox(nsm_handle *h, void **base, void *ipc_handle, int64_t *recv_offsets);

/* Connect to neighbour q's mailbox: peer_n_ghost = q's ghost count,
 * peer_recv_off = q's recv_offsets[this rank].  _ipc opens the handle of
 * another process (closed again by nsm_destroy); the plain form takes a
 * pointer valid in this process (ranks sharing one device and process). */
nsm_status nsm_halo_connect_ipc(nsm_handle *h, int q, const void *ipc_handle, int64_t peer_n_ghost,
                                int64_t peer_recv_off);
nsm_status nsm_halo_connect(nsm_handle *h, int q, void *peer_base, int64_t peer_n_ghost, int64_t peer_recv_off);

/* Finalise the halo tables (after every nsm_halo_set_send / connect). */
nsm_status nsm_halo_commit(nsm_handle *h);

/* r = b - A x.  With nranks > 1 the x halo is exchanged first.
 * b, x, r: device, length n_local; r must not alias b or x. */
nsm_status nsm_residual(nsm_handle *h, const double *b, const double *x, double *r, void *stream);

/*
 * nsm_lsolve — approximate the lower-triangular solve by k Jacobi sweeps
 * (eq:jr-initial-guess / eq:jacobi P:L753-764; eq:LUiterMat P:L826-828):
 *   pGS handle: x = sum_{j=0..k} (-D^{-1} L)^j D^{-1} r    ((D + L) of A)
 *   ILU handle: x = sum_{j=0..k} (-L_s)^j r                (unit-lower factor)
 * k = 0 is legal (diagonal scaling).  r and x must not alias.  In HYBRID
 * mode couplings to other ranks are dropped; in GLOBAL mode lower ghosts of
 * every iterate are exchanged.
 */
nsm_status nsm_lsolve(nsm_handle *h, const double *r, double *x, int k_sweeps, void *stream);

/*
 * nsm_usolve — same for the upper triangle (eq:Neu P:L1064-1066):
 *   pGS handle: x = sum_{j=0..k} (-D^{-1} U)^j D^{-1} r    ((D + U) of A)
 *   ILU handle: x = sum_{j=0..k} (-D_U^{-1} U_s)^j D_U^{-1} r   (U factor)
 */
nsm_status nsm_usolve(nsm_handle *h, const double *r, double *x, int k_sweeps, void *stream);

/*
 * nsm_smooth — nu outer smoothing iterations in place on x (eq:one-stage
 * P:L723-725; §8(a) rows a2-a6):
 *   NSM_PGS : x <- x + sum_{j<=k_l} (-D^{-1}L)^j D^{-1} (b - A x)     (k_u ignored)
 *   NSM_ILU0: x <- x + U~^{-1}_{k_u} L~^{-1}_{k_l} (b - A x)  (Jacobi-iterated factors)
 *   NSM_PGS_BACKWARD: x <- x + sum_{j<=k_l} (-D^{-1}U)^j D^{-1} (b - A x)
 *   NSM_PGS_SYMMETRIC: NSM_PGS then NSM_PGS_BACKWARD (each with its residual)
 *   NSM_L1_JACOBI: x <- x + D_l1^{-1} (b - A x)                      (k_l, k_u ignored)
 * x_is_zero != 0: the first iteration takes x = 0 whatever x holds on entry
 * (its contents are ignored and overwritten), so the first residual is b and
 * is not computed (V-cycle pre-smoothing; exact).  b and x must not alias.
 * Requesting NSM_ILU0 on a handle set up without factors -> NSM_ERR_STATE.
 */
nsm_status nsm_smooth(nsm_handle *h, nsm_kind kind, const double *b, double *x, int nu, int k_l,
                      int k_u, int x_is_zero, void *stream);

/*
 * nsm_smooth_host — nsm_smooth on HOST vectors (the end-to-end call): copies
 * b_host and x_in_host (not read when x_is_zero; may then be NULL) to two
 * handle-owned device vectors on `stream`, runs nsm_smooth there, copies the
 * result to x_out_host and synchronises the stream before returning.
 * All three are n doubles in host memory; x_out_host may equal x_in_host
 * (in place) but must not partially overlap it, and b_host aliases neither.
 * Pinned (cudaHostAlloc / cudaHostRegister) memory gets full PCIe/C2C
 * bandwidth; pageable memory works through the driver's staging.  The first
 * call allocates the two staging vectors (2 n doubles, freed by nsm_destroy;
 * NSM_ERR_OOM if that fails); later calls do not allocate.  Errors as
 * nsm_smooth; a failed copy -> NSM_ERR_CUDA.  On error x_out_host is
 * unspecified.
 */
nsm_status nsm_smooth_host(nsm_handle *h, nsm_kind kind, const double *b_host, const double *x_in_host,
                           double *x_out_host, int nu, int k_l, int k_u, int x_is_zero, void *stream);

/* y = A x  (plain SpMV with the stored split; used by the GMRES/V-cycle
 * driver).  With nranks > 1 the x halo is exchanged first. */
nsm_status nsm_spmv(nsm_handle *h, const double *x, double *y, void *stream);

/* Synchronises the stream, then reports NSM_ERR_NONFINITE if any sweep since
 * setup (or the last nsm_check) produced Inf/NaN; *first_bad_sweep receives
 * the smallest global sweep counter that did (-1 if none).  Clears the flag. */
nsm_status nsm_check(nsm_handle *h, int64_t *first_bad_sweep, void *stream);

/* Handle facts: local rows, ghost columns, stored (unpadded) entries and the
 * device bytes of the split storage. */
nsm_status nsm_info(const nsm_handle *h, int64_t *n_local, int64_t *n_ghost, int64_t *nnz_offdiag,
                    int64_t *device_bytes);

/* Counters since setup: kernels this handle launched (every launch of every
 * call) and halo exchanges it performed.  Host-side, no synchronisation. */
nsm_status nsm_stats(const nsm_handle *h, int64_t *kernel_launches, int64_t *halo_exchanges);

/* Storage layout of the strict triangles: bit 1 / 2 / 4 / 8
 * set when A's L / A's U / the factor's L_s / U_s uses the offset-aligned
 * SELL layout (stencil-like rows: one int32 column offset per slice entry
 * position; the pipelined kernels then read 8 instead of 12 bytes per entry).
 * Chosen automatically at setup when it widens the slices by <= 15 %.
 * Bits 16 / 32 / 64: the residual (L and U) / L / U have a shared-memory
 * gather window (built where it is at most half the staged
 * entries), i.e. the windowed kernels run. */
nsm_status nsm_layout(const nsm_handle *h, int *offset_aligned);

/* Fused-pass synchronisation statistics since setup: work items whose
 * consumer warps found the item not yet ready (its condition "all items <=
 * w - Dw done", unmet) and had to wait, and the total time
 * they waited in ns (one warp per CTA measures).  Synchronises the device. */
nsm_status nsm_fused_stats(nsm_handle *h, int64_t *waits, int64_t *wait_ns);

/* In-stream pass timing (after nsm_set_option(h, NSM_OPT_PROFILE, 1)):
 * waits for the recorded events, returns the summed milliseconds and counts
 * of residual passes (ms[0], count[0]), sweep passes (ms[1], count[1]) and
 * fused passes (ms[2], count[2]) since the last call, and clears the
 * records.  `ms` and `count` have 3 entries. */
nsm_status nsm_profile(nsm_handle *h, double *ms, int64_t *count);

/* Last error message: of `h`, or of the last failed setup when h == NULL.
 * The pointer stays valid until the next call on the same handle. */
const char *nsm_last_error(const nsm_handle *h);

/* Handle options (not on the hot path; take effect for subsequent calls):
 *   NSM_OPT_PIPELINE        1 (default) = bulk-copy pipelined kernels for
 *                           contiguous slice ranges (cp.async.bulk + mbarrier,
 *                           DESIGN.md §6); 0 = the plain register-blocked
 *                           kernels.  Both give bit-identical results.
 *   NSM_OPT_HALO_TIMEOUT_MS how long a halo or wavefront wait spins before
 *                           giving up and flagging NSM_ERR_DIST (default 20000).
 *   NSM_OPT_FUSED           single-rank applications as phase-skewed fused
 *                           passes: pGS (forward / backward)
 *                           = ONE pass (residual + k sweeps + x update, the
 *                           matrix read from HBM once), ILU(0) = two passes
 *                           (residual + k_l L sweeps ascending; k_u U sweeps
 *                           + x update descending); needs 1 <= k <= 8.
 *                           0 (default) = one kernel per pass; 1 = fused
 *                           whenever possible; 2 = fused when the problem
 *                           spans at least two skew distances (large
 *                           problems).  Bit-identical results either way.
 *                           The fused passes read ~2.4x fewer HBM bytes but
 *                           are currently latency-bound and slower than the
 *                           per-pass kernels.  Switching it
 *                           on allocates the passes' L2 ring buffers (up to
 *                           ~9 n-vectors; NSM_ERR_OOM if that fails).
 *                           3 = as 1, and a forward pGS application on a
 *                           stencil-like matrix (offset-aligned L and U with
 *                           gather windows) runs as ONE windowed pass with
 *                           per-phase readiness (fused_w.cu; experimental:
 *                           reads the matrix from HBM once but is slower,
 *                           DESIGN.md §6).
 *   NSM_OPT_FUSED_WINDOW    wait distance Dw of the fused passes in work
 *                           items (0 = automatic, about the items in flight);
 *                           a small value forces frequent waits and ring
 *                           reuse (a test knob; slower).
 *   NSM_OPT_PDL             1 = launch the pipelined kernels with
 *                           programmatic dependent launch (a kernel's matrix
 *                           prefetch overlaps the previous kernel's drain);
 *                           0 = plain stream order.  Default: 1 up to 8 M
 *                           rows per rank and for single-rank matrices with
 *                           gather windows, 0 otherwise (measured per
 *                           configuration). */
typedef enum {
    NSM_OPT_PIPELINE = 0, NSM_OPT_HALO_TIMEOUT_MS = 1, NSM_OPT_FUSED = 2, NSM_OPT_PDL = 3,
    NSM_OPT_PROFILE = 4 /* 1: record a CUDA event pair around every residual / sweep / fused pass
                           (up to 4096 passes) for nsm_profile(); 0: off (default) */,
    NSM_OPT_FUSED_WINDOW = 5,
    NSM_OPT_WINDOW = 6 /* 1 (default): pipelined kernels over an offset-aligned part stage the gathered
                        * vector's window (the tile's columns, merged into a few segments) into shared
                        * memory with the tile and gather from there (single rank); 0: gathers from
                        * global memory through L1/L2.  Results are identical. */,
    NSM_OPT_PLANE_ROWS = 7 /* > 0 (a multiple of 256): the rows form planes of this many rows whose 256-row
                            * tiles couple only to tiles within two lines (tile index mod plane) in the same
                            * or a neighbouring plane (lexicographic 7- / 27-point grids with 256-point grid
                            * lines; checked: NSM_ERR_PATTERN otherwise).  With NSM_OPT_FUSED = 3 a forward
                            * pGS application with k >= 2 then runs as a plane wavefront: one CTA per line,
                            * readiness from the neighbouring lines' step counters only (fused_w.cu). */,
    NSM_OPT_HOST_CHUNKS = 8 /* 1 (default): nsm_smooth_host runs a single-rank forward pGS application
                             * (nu = 1, k <= 3, x_in != x_out) in row chunks longer than A's bandwidth, so
                             * the host-to-device copies, the passes and the device-to-host copy overlap
                             * (separate copy streams); 0: copy in, smooth, copy out.  Same results. */,
    NSM_OPT_COUPLED = 9 /* 1: a single-rank forward pGS application with k = 2 or 3 on an offset-aligned L
                         * with a gather window (27-point stencils) runs the residual pass, then its k sweeps
                         * as concurrent CTA groups of ONE cooperative kernel (coupled.cu): the
                         * later sweeps re-read L from L2, so L is streamed from HBM once instead of k times.
                         * Bit-identical to the per-pass kernels.  Experimental: reads the predicted bytes
                         * (C3: 2.3 GB for both sweeps instead of 4.6) but is latency-bound and slower than the
                         * per-pass sweeps.  0 (default): one kernel per pass; > 1: on, with this throttle
                         * distance in 256-row tiles (a test knob: 2 makes group 0 wait at almost every tile). */
} nsm_option;
nsm_status nsm_set_option(nsm_handle *h, nsm_option opt, int64_t value);

/* ---- GPU-resident solver around the smoothers ---
 * nsm_spmat: a general (rectangular) CSR matrix on the device for the AMG
 * transfer operators; y = alpha * M x + beta * y.  HOST CSR in, device
 * vectors at apply time. */
typedef struct nsm_spmat nsm_spmat;
nsm_status nsm_spmat_setup(nsm_spmat **out, const nsm_csr *M, int device);
nsm_status nsm_spmat_apply(nsm_spmat *M, const double *x, double *y, double alpha, double beta, void *stream);
void nsm_spmat_destroy(nsm_spmat *M);

/* nsm_amg: one C-AMG V(nu_pre, nu_post) cycle
 * over a hierarchy built by the caller: smoothers[l] (l < nlevels) are
 * nsm handles of A_l (BORROWED: must outlive the nsm_amg), P[l] the HOST
 * prolongation A_l -> A_{l+1} (n_l x n_{l+1}; R = P^T), coarse the
 * HOST coarsest matrix A_{nlevels} (<= 8192 rows; inverted densely at setup
 * with partial pivoting: the coarse direct solve).  nsm_amg_vcycle computes
 * x = V(b) from x = 0: per level pre-smooth (x_is_zero), residual, restrict,
 * recurse, prolong-add, post-smooth; b and x device, length n_0, distinct.
 * Default smoother on every level: NSM_PGS, nu = 1/1, k = 2. */
typedef struct nsm_amg nsm_amg;
nsm_status nsm_amg_setup(nsm_amg **out, int nlevels, nsm_handle *const *smoothers, const nsm_csr *const *P,
                         const nsm_csr *coarse, int device);
nsm_status nsm_amg_set_smoother(nsm_amg *M, int level, nsm_kind kind, int nu_pre, int nu_post, int k_l, int k_u);
nsm_status nsm_amg_vcycle(nsm_amg *M, const double *b, double *x, void *stream);
void nsm_amg_destroy(nsm_amg *M);
const char *nsm_solver_last_error(const nsm_amg *M);

/* nsm_gmres: right-preconditioned one-reduce MGS-GMRES with lagged
 * normalisation (Algorithm 1), x0 = 0, no restart.  Per
 * iteration: w = A M u, ONE reduction [V, u]^T [u, w] (one device -> host
 * read), projection with T = I - L (t_mode 0: the paper's truncated Neumann
 * series) or T = (I + L)^{-1} (t_mode 1).  Stops when
 * the implicit relative residual < tol or after maxit iterations.
 * M = NULL: no preconditioner.  *iters = Krylov dimension m; hist (NULL or
 * maxit + 1 entries) receives the implicit relative residuals.  b, x device,
 * length n; synchronises `stream`.  Workspace (the Krylov basis, grown in
 * blocks of columns as the iteration needs them, pinned host buffers, the
 * captured V-cycle graph) is kept in M across calls and freed by
 * nsm_amg_destroy; with M = NULL it is allocated and freed per call.  One M
 * must not be used by concurrent nsm_gmres calls.  The graph is re-captured
 * when a handle's options or Ruiz scaling changed (nsm_set_option,
 * nsm_set_ruiz, nsm_set_comm).
 * Distributed A (a row block per rank): every rank calls nsm_gmres with its
 * rows of b and x; the reduction runs through the comm attached with
 * nsm_set_comm (NSM_ERR_STATE without one; NSM_ERR_DIST if a rank timed
 * out), so every rank takes the same iteration count. */
nsm_status nsm_gmres(nsm_handle *A, nsm_amg *M, const double *b, double *x, int maxit, double tol, int t_mode,
                     int *iters, double *hist, void *stream);

/* ---- cross-rank reduction of the distributed solver (NEXT-1) ------------
 * Algorithm 1 step 6 is "Global synchronization": ONE all-reduce of the
 * 2(k+1) partial dot products per iteration ("one MPI_AllReduce per
 * iteration").  nsm_comm is that all-reduce on the device, over
 * NVLink / NVSwitch peer memory: every rank stores its m values into slot
 * `rank` of every rank's mailbox (CUDA IPC mappings across processes, plain
 * device pointers for ranks sharing a process) and each rank adds the slots
 * in ascending rank order, so all ranks hold bit-identical sums.
 *
 * nsm_comm_create: rank / nranks of the partition, capacity = largest m
 * (GMRES needs 2 (maxit + 2); the distributed V-cycle the first coarse
 * level's size), device ordinal.  nsm_comm_mailbox: the device base of this
 * rank's mailbox and (ipc_handle != NULL) its 64-byte CUDA IPC handle.
 * nsm_comm_connect[_ipc]: peer q's mailbox (base pointer in this process, or
 * its IPC handle); once every rank is connected the comm is usable.
 * nsm_comm_allreduce: out[j] = sum over ranks of in[j] (j < m), in and out
 * device arrays of this rank (may alias), stream-ordered, no host sync; every
 * rank must call it the same number of times in the same order.  A rank that
 * waits longer than the timeout (default 20 s, nsm_comm_set_timeout) flags
 * the comm; nsm_comm_check (synchronises `stream`) then returns
 * NSM_ERR_DIST.  NSM_ERR_STATE before every rank is connected, NSM_ERR_ARG
 * for m > capacity.
 *
 * nsm_set_comm attaches a comm (BORROWED, same rank / nranks / device) to a
 * distributed handle: nsm_gmres on a distributed operator reduces its dot
 * products through it (NSM_ERR_STATE without one), and an nsm_amg whose
 * finest smoother is distributed restricts onto the replicated coarse levels
 * through it: level 0 holds the rank's rows (P[0] = the rank's rows of the
 * prolongation, n_local x n_1, global coarse columns), levels >= 1 are
 * identical single-rank handles on every rank. */
typedef struct nsm_comm nsm_comm;
nsm_status nsm_comm_create(nsm_comm **out, int rank, int nranks, int64_t capacity, int device);
nsm_status nsm_comm_mailbox(nsm_comm *c, void **base, void *ipc_handle);
nsm_status nsm_comm_connect(nsm_comm *c, int q, void *peer_base);
nsm_status nsm_comm_connect_ipc(nsm_comm *c, int q, const void *ipc_handle);
nsm_status nsm_comm_allreduce(nsm_comm *c, const double *in, double *out, int64_t m, void *stream);
nsm_status nsm_comm_check(nsm_comm *c, void *stream);
nsm_status nsm_comm_set_timeout(nsm_comm *c, int64_t ms);
nsm_status nsm_comm_stats(const nsm_comm *c, int64_t *allreduces);
const char *nsm_comm_last_error(const nsm_comm *c);
void nsm_comm_destroy(nsm_comm *c);
nsm_status nsm_set_comm(nsm_handle *h, nsm_comm *c);

/* ---- device-side set-up -----------
 * nsm_setup_device: single-rank nsm_setup from a DEVICE CSR — A's (and F's)
 * rowptr / colind / val are device pointers of `device` (int64 / int64 /
 * fp64, the nsm_csr layout), borrowed for the call.  The split, the SELL-32
 * packing (compact or offset-aligned, the same decision) and the diagonals
 * are built by GPU kernels and are identical to nsm_setup's host build;
 * errors as nsm_setup (pattern, zero diagonal with the first offending row).
 *
 * nsm_part_info / nsm_part_copy / nsm_diag_copy: host copies of a handle's
 * device arrays (diagnostics, builder parity).  part 0..7 = L, U, LG, UG,
 * Ls, Us, LsG, UsG (slice pointers nslices + 1, columns / values `padded`
 * entries, offsets padded / 32 when aligned; NULL buffers are skipped);
 * which 0 = d, 1 = l1 diagonal, 2 = d_U (NSM_ERR_STATE without factors). */
nsm_status nsm_setup_device(nsm_handle **out, const nsm_csr *A, const nsm_csr *F, int device);
nsm_status nsm_part_info(const nsm_handle *h, int part, int64_t *padded, int64_t *nnz, int *maxw, int *aligned);
nsm_status nsm_part_copy(const nsm_handle *h, int part, int64_t *ptr, int32_t *col, double *val, int32_t *off);
nsm_status nsm_diag_copy(const nsm_handle *h, int which, double *out);

/* nsm_fused_counters: cumulative counters of the one-pass windowed pGS
 * (NSM_OPT_FUSED on stencil-like matrices), summed over its CTAs' producer
 * warps: out[0] synchronous frontier polls, [1] their ns, [2] ns waiting for a
 * free stage, [3] ns in readiness checks, [4] ns per unit in total, [5]
 * acquire fences.  Diagnostics; out has 6 entries. */
nsm_status nsm_fused_counters(const nsm_handle *h, int64_t *out);

/* nsm_coupled_counters: cumulative SM-cycle counters of the coupled sweeps
 * kernel (coupled.cu), collected while NSM_OPT_PROFILE is on: for sweep group
 * g = 0..2, out[4g + 0] producer cycles in dependency waits, out[4g + 1]
 * producer cycles waiting for a free stage, out[4g + 2] producer cycles in
 * total (summed over CTAs), out[4g + 3] consumer cycles waiting for staged
 * data (warp 0 of the group, summed over CTAs).  `out` has 16 entries;
 * synchronises the device. */
nsm_status nsm_coupled_counters(const nsm_handle *h, int64_t *out);

/* Frees all device memory of the handle (synchronises its device).  NULL ok. */
void nsm_destroy(nsm_handle *h);

#ifdef __cplusplus
}
#endif
#endif /* NSM_H */
