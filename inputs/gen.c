/*
 * inputs/gen.c — seeded synthetic inputs shared by the oracle tests and the
 * CUDA path (SURVEY.md §8(d) "Synthetic inputs"; DESIGN.md §3 "Input recipe").
 *
 * This module holds NO arithmetic of the method (no residual, no sweep, no
 * factorisation).  It only assembles stencil matrices of the shapes the paper's
 * workloads have (§6.1 Nalu-Wind pressure; §6.2 PeleLM
 * nodal projection), draws counter-based random vectors, and
 * computes a reverse Cuthill-McKee ordering (the "symrcm" preprocessing of
 * Table 1) that both sides then read as plain input.
 *
 * Conventions (all generators):
 *   - grid point (ix, iy, iz) has lexicographic id  ix + nx*(iy + ny*iz)
 *     (x fastest);
 *   - a generator produces the CSR rows [row_begin, row_end) of the global
 *     matrix with GLOBAL column ids, columns strictly ascending per row;
 *   - Dirichlet boundaries are eliminated (missing neighbours dropped from the
 *     row; their coupling weight is still added to the diagonal);
 *   - random numbers come from splitmix64 keyed by (seed, global index), so any
 *     row partition regenerates identical data.
 *
 * Two-call protocol: *_nnz() returns the number of stored entries of the row
 * range, *_fill() writes rowptr[nrows+1] (int64, starting at 0), col[nnz]
 * (int64) and val[nnz] (double).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG --- */
static inline uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
/* uniform double in [0,1) from the counter (seed, idx) */
static inline double u01(uint64_t seed, uint64_t idx) {
    uint64_t h = splitmix64(splitmix64(seed * 0xD1B54A32D192ED03ull + 0x1234567ull) ^ idx);
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

/* out[i] = lo + (hi-lo) * U[0,1) for global indices idx0 .. idx0+n-1 */
void gen_uniform(uint64_t seed, int64_t idx0, int64_t n, double lo, double hi, double *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * u01(seed, (uint64_t)(idx0 + i));
}

/* integers uniform in [-2^bits, 2^bits) stored as doubles (exactly representable) */
void gen_uniform_int(uint64_t seed, int64_t idx0, int64_t n, int bits, double *out) {
    const double span = ldexp(1.0, bits + 1);
    for (int64_t i = 0; i < n; ++i) {
        double v = floor(u01(seed, (uint64_t)(idx0 + i)) * span) - ldexp(1.0, bits);
        out[i] = v;
    }
}

/* standard normal via Box-Muller from two counter draws */
static inline double gauss(uint64_t seed, uint64_t idx) {
    double a = u01(seed, 2 * idx), b = u01(seed, 2 * idx + 1);
    if (a < 1e-300) a = 1e-300;
    return sqrt(-2.0 * log(a)) * cos(6.283185307179586 * b);
}

/* ------------------------------------------------------- coefficient field */
/*
 * Smoothed Gaussian field on an nx*ny*nz grid, normalised to [0,1], mapped to
 * kappa = contrast^u  (so kappa in [1, contrast]).  Three passes of a 3-point
 * box filter per axis; at the boundary the window is truncated (average of
 * the available points).  SURVEY.md §8(d) "C3 matrix detail".
 */
static void box3_axis(double *f, double *tmp, int64_t nx, int64_t ny, int64_t nz, int axis) {
    int64_t n = nx * ny * nz;
    int64_t stride = axis == 0 ? 1 : (axis == 1 ? nx : nx * ny);
    int64_t len = axis == 0 ? nx : (axis == 1 ? ny : nz);
    for (int64_t id = 0; id < n; ++id) {
        int64_t c = axis == 0 ? id % nx : (axis == 1 ? (id / nx) % ny : id / (nx * ny));
        double s = f[id];
        int cnt = 1;
        if (c > 0) { s += f[id - stride]; ++cnt; }
        if (c + 1 < len) { s += f[id + stride]; ++cnt; }
        tmp[id] = s / cnt;
    }
    memcpy(f, tmp, (size_t)n * sizeof(double));
}

int gen_kappa_field(int64_t nx, int64_t ny, int64_t nz, uint64_t seed, double contrast, double *kappa) {
    int64_t n = nx * ny * nz;
    double *tmp = (double *)malloc((size_t)n * sizeof(double));
    if (!tmp) return -1;
    for (int64_t i = 0; i < n; ++i) kappa[i] = gauss(seed, (uint64_t)i);
    for (int pass = 0; pass < 3; ++pass)
        for (int ax = 0; ax < 3; ++ax) box3_axis(kappa, tmp, nx, ny, nz, ax);
    double lo = kappa[0], hi = kappa[0];
    for (int64_t i = 1; i < n; ++i) { if (kappa[i] < lo) lo = kappa[i]; if (kappa[i] > hi) hi = kappa[i]; }
    double span = hi > lo ? hi - lo : 1.0;
    double lc = log(contrast);
    for (int64_t i = 0; i < n; ++i) kappa[i] = exp(lc * ((kappa[i] - lo) / span));
    free(tmp);
    return 0;
}

/* ------------------------------------------------------- stencil helpers -- */
typedef struct { int64_t nx, ny, nz; } grid3;

static inline void decode(const grid3 *g, int64_t id, int64_t *x, int64_t *y, int64_t *z) {
    *x = id % g->nx; *y = (id / g->nx) % g->ny; *z = id / (g->nx * g->ny);
}
static inline int inside(const grid3 *g, int64_t x, int64_t y, int64_t z) {
    return x >= 0 && y >= 0 && z >= 0 && x < g->nx && y < g->ny && z < g->nz;
}

/* Offsets of the 7-point and 27-point stencils in ascending linear order
 * (dz outer, dy, dx inner) so that emitted columns are strictly ascending. */
static const int OFF7[7][3] = {{0,0,-1},{0,-1,0},{-1,0,0},{0,0,0},{1,0,0},{0,1,0},{0,0,1}};

/* ---- 2-D 5-point / 3-D 7-point constant-coefficient Laplacian ------------
 * 2-D: nz = 1 gives the 5-point stencil (4, -1 x 4)   [config C1]
 * 3-D: 7-point (6, -1 x 6)                           [configs C2, C5]
 * The diagonal is the full stencil weight (Dirichlet neighbours eliminated).  */
static int64_t lap_row(const grid3 *g, int dim, int64_t id, int64_t *col, double *val) {
    int64_t x, y, z; decode(g, id, &x, &y, &z);
    int64_t k = 0;
    for (int o = 0; o < 7; ++o) {
        int dx = OFF7[o][0], dy = OFF7[o][1], dz = OFF7[o][2];
        if (dim == 2 && dz != 0) continue;
        int64_t xx = x + dx, yy = y + dy, zz = z + dz;
        if (!inside(g, xx, yy, zz)) continue;
        if (col) {
            col[k] = xx + g->nx * (yy + g->ny * zz);
            val[k] = (dx == 0 && dy == 0 && dz == 0) ? (dim == 2 ? 4.0 : 6.0) : -1.0;
        }
        ++k;
    }
    return k;
}

int64_t gen_lap_nnz(int64_t nx, int64_t ny, int64_t nz, int dim, int64_t r0, int64_t r1) {
    grid3 g = {nx, ny, nz};
    int64_t s = 0;
    for (int64_t i = r0; i < r1; ++i) s += lap_row(&g, dim, i, NULL, NULL);
    return s;
}
void gen_lap_fill(int64_t nx, int64_t ny, int64_t nz, int dim, int64_t r0, int64_t r1,
                  int64_t *rowptr, int64_t *col, double *val) {
    grid3 g = {nx, ny, nz};
    rowptr[0] = 0;
    for (int64_t i = r0; i < r1; ++i) {
        int64_t p = rowptr[i - r0];
        rowptr[i - r0 + 1] = p + lap_row(&g, dim, i, col + p, val + p);
    }
}

/* ---- 27-point variable-coefficient pressure matrix (Nalu-Wind shaped) ----
 * w_io = harm(kappa_i, kappa_{i+o}) * c_{|o|_1} * a(o),  c1 = 1, c2 = 1/2,
 * c3 = 1/4, a(o) = 100 for pure-z face offsets (anisotropy proxy for the
 * O(40000) cell aspect ratios of P:L1307-1309), 1 otherwise.  Off-diagonal
 * -w_io, diagonal = sum of w over all 26 offsets (missing Dirichlet neighbours
 * use kappa_i).  Symmetric, irreducibly diagonally dominant M-matrix.  [C3] */
static inline double harm(double a, double b) { return 2.0 * a * b / (a + b); }

static int64_t var27_row(const grid3 *g, const double *kappa, int64_t id, int64_t *col, double *val) {
    int64_t x, y, z; decode(g, id, &x, &y, &z);
    double ki = kappa[id];
    double diag = 0.0;
    int64_t k = 0, kdiag = -1;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int l1 = abs(dx) + abs(dy) + abs(dz);
                int64_t xx = x + dx, yy = y + dy, zz = z + dz;
                int in = inside(g, xx, yy, zz);
                if (l1 == 0) {
                    if (col) { col[k] = id; kdiag = k; }
                    ++k;
                    continue;
                }
                double c = l1 == 1 ? 1.0 : (l1 == 2 ? 0.5 : 0.25);
                double a = (dx == 0 && dy == 0) ? 100.0 : 1.0;
                int64_t j = in ? xx + g->nx * (yy + g->ny * zz) : -1;
                double w = harm(ki, in ? kappa[j] : ki) * c * a;
                diag += w;
                if (!in) continue;
                if (col) { col[k] = j; val[k] = -w; }
                ++k;
            }
    if (col) val[kdiag] = diag;
    return k;
}

int64_t gen_var27_nnz(int64_t nx, int64_t ny, int64_t nz, int64_t r0, int64_t r1) {
    grid3 g = {nx, ny, nz};
    int64_t s = 0;
    for (int64_t i = r0; i < r1; ++i) {
        int64_t x, y, z; decode(&g, i, &x, &y, &z);
        int64_t cx = 1 + (x > 0) + (x + 1 < nx), cy = 1 + (y > 0) + (y + 1 < ny), cz = 1 + (z > 0) + (z + 1 < nz);
        s += cx * cy * cz;
    }
    return s;
}
void gen_var27_fill(int64_t nx, int64_t ny, int64_t nz, const double *kappa, int64_t r0, int64_t r1,
                    int64_t *rowptr, int64_t *col, double *val) {
    grid3 g = {nx, ny, nz};
    rowptr[0] = 0;
    for (int64_t i = r0; i < r1; ++i) {
        int64_t p = rowptr[i - r0];
        rowptr[i - r0 + 1] = p + var27_row(&g, kappa, i, col + p, val + p);
    }
}

/* ---- nonsymmetric convection-diffusion, 7-point upwind (PeleLM shaped) ----
 * -div(kappa grad u) + v . grad u, first-order upwind, unit spacing.
 * Face coefficient kappa_f = harm(kappa_i, kappa_j) (kappa_i for a missing
 * Dirichlet neighbour).  For axis a with velocity v_a: the upstream neighbour
 * (i - sign(v_a) e_a) gets -kappa_f - |v_a|, the downstream one -kappa_f; the
 * diagonal is sum_faces kappa_f + sum_a |v_a|.  M-matrix with a symmetric
 * pattern and nonsymmetric values.  [C4, before RCM]                        */
static int64_t cd_row(const grid3 *g, const double *kappa, const double v[3], int64_t id,
                      int64_t *col, double *val) {
    int64_t x, y, z; decode(g, id, &x, &y, &z);
    double ki = kappa[id];
    double diag = fabs(v[0]) + fabs(v[1]) + fabs(v[2]);
    int64_t k = 0, kdiag = -1;
    for (int o = 0; o < 7; ++o) {
        int dx = OFF7[o][0], dy = OFF7[o][1], dz = OFF7[o][2];
        if (!dx && !dy && !dz) {
            if (col) { col[k] = id; kdiag = k; }
            ++k;
            continue;
        }
        int axis = dx ? 0 : (dy ? 1 : 2);
        int dir = dx + dy + dz; /* -1 or +1 */
        int64_t xx = x + dx, yy = y + dy, zz = z + dz;
        int in = inside(g, xx, yy, zz);
        int64_t j = in ? xx + g->nx * (yy + g->ny * zz) : -1;
        double kf = harm(ki, in ? kappa[j] : ki);
        diag += kf;
        if (!in) continue;
        /* upstream neighbour: the one the flow comes from, i.e. dir == -sign(v) */
        int upstream = (v[axis] > 0 && dir < 0) || (v[axis] < 0 && dir > 0);
        if (col) { col[k] = j; val[k] = -kf - (upstream ? fabs(v[axis]) : 0.0); }
        ++k;
    }
    if (col) val[kdiag] = diag;
    return k;
}

/* velocity: |v_a| = Pe_a * sqrt(contrast) with Pe_a ~ U[1,20), random sign   */
void gen_cd_velocity(uint64_t seed, double contrast, double v[3]) {
    for (int a = 0; a < 3; ++a) {
        double pe = 1.0 + 19.0 * u01(seed ^ 0xC0FFEEull, (uint64_t)a);
        double sg = u01(seed ^ 0xBEEFull, (uint64_t)a) < 0.5 ? -1.0 : 1.0;
        v[a] = sg * pe * sqrt(contrast);
    }
}

int64_t gen_cd_nnz(int64_t nx, int64_t ny, int64_t nz, int64_t r0, int64_t r1) {
    return gen_lap_nnz(nx, ny, nz, 3, r0, r1);
}
void gen_cd_fill(int64_t nx, int64_t ny, int64_t nz, const double *kappa, const double *v,
                 int64_t r0, int64_t r1, int64_t *rowptr, int64_t *col, double *val) {
    grid3 g = {nx, ny, nz};
    rowptr[0] = 0;
    for (int64_t i = r0; i < r1; ++i) {
        int64_t p = rowptr[i - r0];
        rowptr[i - r0 + 1] = p + cd_row(&g, kappa, v, i, col + p, val + p);
    }
}

/* ------------------------------------------------------ RCM (symrcm) ------
 * Reverse Cuthill-McKee on the pattern of a structurally symmetric matrix
 * ("symmetric reverse Cuthill-McKee").  Start node: George-Liu
 * pseudo-peripheral node search from node 0; neighbours visited in
 * (degree, index) order; the Cuthill-McKee order is reversed.  Disconnected
 * components are handled one after another (lowest unvisited index first).
 * Output order[k] = old index placed at new position k.                     */
static int64_t bfs_levels(int64_t n, const int64_t *rp, const int64_t *ci, int64_t s,
                          int64_t *level, int64_t *queue, int64_t *last_begin) {
    for (int64_t i = 0; i < n; ++i) level[i] = -1;
    int64_t head = 0, tail = 0;
    queue[tail++] = s; level[s] = 0;
    int64_t maxlev = 0, lb = 0;
    while (head < tail) {
        int64_t u = queue[head++];
        if (level[u] > maxlev) { maxlev = level[u]; lb = head - 1; }
        for (int64_t p = rp[u]; p < rp[u + 1]; ++p) {
            int64_t w = ci[p];
            if (level[w] < 0) { level[w] = level[u] + 1; queue[tail++] = w; }
        }
    }
    *last_begin = lb;
    (void)tail;
    return maxlev;
}

typedef struct { int64_t idx, deg; } nd_t;
static int cmp_nd(const void *a, const void *b) {
    const nd_t *x = (const nd_t *)a, *y = (const nd_t *)b;
    if (x->deg != y->deg) return x->deg < y->deg ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

int gen_rcm(int64_t n, const int64_t *rp, const int64_t *ci, int64_t *order) {
    int64_t *level = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *queue = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    char *vis = (char *)calloc((size_t)n, 1);
    if (!level || !queue || !vis) { free(level); free(queue); free(vis); return -1; }
    int64_t pos = 0, maxdeg = 1;
    for (int64_t i = 0; i < n; ++i) if (rp[i + 1] - rp[i] > maxdeg) maxdeg = rp[i + 1] - rp[i];
    nd_t *nb = (nd_t *)malloc((size_t)maxdeg * sizeof(nd_t));
    if (!nb) { free(level); free(queue); free(vis); return -1; }
    for (int64_t root = 0; root < n; ++root) {
        if (vis[root]) continue;
        /* pseudo-peripheral node within root's component (components are
           visited whole, so level[] of other visited nodes is irrelevant) */
        int64_t s = root, lb, ecc = bfs_levels(n, rp, ci, s, level, queue, &lb);
        for (int it = 0; it < 8; ++it) {
            /* candidate: min-degree node of the last level */
            int64_t best = -1, bdeg = 0;
            for (int64_t q = lb; q < n && level[queue[q]] == ecc; ++q) {
                int64_t u = queue[q], d = rp[u + 1] - rp[u];
                if (best < 0 || d < bdeg || (d == bdeg && u < best)) { best = u; bdeg = d; }
            }
            int64_t lb2, ecc2 = bfs_levels(n, rp, ci, best, level, queue, &lb2);
            if (ecc2 > ecc) { s = best; ecc = ecc2; lb = lb2; } else break;
        }
        /* Cuthill-McKee BFS from s */
        int64_t head = pos, tail = pos;
        order[tail++] = s; vis[s] = 1;
        while (head < tail) {
            int64_t u = order[head++];
            int64_t m = 0;
            for (int64_t p = rp[u]; p < rp[u + 1]; ++p) {
                int64_t w = ci[p];
                if (!vis[w]) { nb[m].idx = w; nb[m].deg = rp[w + 1] - rp[w]; ++m; vis[w] = 1; }
            }
            qsort(nb, (size_t)m, sizeof(nd_t), cmp_nd);
            for (int64_t q = 0; q < m; ++q) order[tail++] = nb[q].idx;
        }
        pos = tail;
    }
    /* reverse */
    for (int64_t i = 0, j = n - 1; i < j; ++i, --j) { int64_t t = order[i]; order[i] = order[j]; order[j] = t; }
    free(level); free(queue); free(vis); free(nb);
    return pos == n ? 0 : -2;
}

/* Symmetric permutation B = A(order, order): new row k is old row order[k],
 * column old j becomes inv[j]; columns re-sorted ascending (rows are short). */
int gen_permute(int64_t n, const int64_t *rp, const int64_t *ci, const double *va, const int64_t *order,
                int64_t *rp2, int64_t *ci2, double *va2) {
    int64_t *inv = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    if (!inv) return -1;
    for (int64_t k = 0; k < n; ++k) inv[order[k]] = k;
    rp2[0] = 0;
    for (int64_t k = 0; k < n; ++k) {
        int64_t o = order[k], len = rp[o + 1] - rp[o], p2 = rp2[k];
        for (int64_t q = 0; q < len; ++q) {
            int64_t c = inv[ci[rp[o] + q]];
            double v = va[rp[o] + q];
            int64_t t = p2 + q;
            while (t > p2 && ci2[t - 1] > c) { ci2[t] = ci2[t - 1]; va2[t] = va2[t - 1]; --t; }
            ci2[t] = c; va2[t] = v;
        }
        rp2[k + 1] = p2 + len;
    }
    free(inv);
    return 0;
}

/* Bandwidth max |i - j| over stored entries (diagnostic for the RCM tests). */
int64_t gen_bandwidth(int64_t n, const int64_t *rp, const int64_t *ci) {
    int64_t bw = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            int64_t d = ci[p] > i ? ci[p] - i : i - ci[p];
            if (d > bw) bw = d;
        }
    return bw;
}
