// builder.cpp — split-triangular storage builder.
//
// Splits a host CSR row block into the paper's A = L + D + U (P:L181-186,
// P:L717-721) and packs each strict part as SELL-32 slices (nsm_internal.h).
// Couplings to columns owned by other ranks go to separate ghost parts LG
// (columns below the block) and UG (above), so that visiting LG, L, D, U, UG
// in this order is still the ascending column order of the full row.
// Also: nsm_ilu0's host ILU(0) factorisation (setup input).
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "nsm_internal.h"

namespace nsm {

namespace {

enum Part { P_LG = 0, P_L = 1, P_D = 2, P_U = 3, P_UG = 4 };

inline int classify(int64_t i_glob, int64_t c, int64_t rb, int64_t re) {
    if (c < rb) return P_LG;
    if (c >= re) return P_UG;
    if (c < i_glob) return P_L;
    if (c == i_glob) return P_D;
    return P_U;
}

// Pack per-row entry lists into SELL-32.  cnt[i] = entries of row i in this
// part; first[i] = index into the CSR arrays of the row's first such entry
// (entries of one part are contiguous in a sorted row); colmap maps a CSR
// column to the stored int32 index.
template <class ColMap>
void pack(int64_t n, const std::vector<int32_t> &cnt, const std::vector<int64_t> &first,
          const int64_t *ci, const double *va, ColMap colmap, SellHost *out) {
    int64_t ns = (n + kSlice - 1) / kSlice;
    out->ptr.assign(ns + 1, 0);
    std::vector<int32_t> w(ns, 0);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < ns; ++s) {
        int32_t m = 0;
        for (int64_t i = s * kSlice; i < std::min(n, (s + 1) * kSlice); ++i) m = std::max(m, cnt[i]);
        w[s] = m;
    }
    int32_t maxw = 0;
    int64_t nnz = 0;
    for (int64_t s = 0; s < ns; ++s) {
        out->ptr[s + 1] = out->ptr[s] + (int64_t)w[s] * kSlice;
        maxw = std::max(maxw, w[s]);
    }
    for (int64_t i = 0; i < n; ++i) nnz += cnt[i];
    out->maxw = maxw;
    out->nnz = nnz;
    int64_t tot = out->ptr[ns];
    out->col.assign(tot, 0);
    out->val.assign(tot, 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < ns; ++s) {
        int64_t base = out->ptr[s];
        for (int l = 0; l < kSlice; ++l) {
            int64_t i = s * kSlice + l;
            int32_t c = i < n ? cnt[i] : 0;
            // padding column: the row itself (local) or 0 (ghost parts): any
            // valid address, multiplied by 0.0
            int32_t pad = colmap.pad(i < n ? i : 0);
            for (int32_t j = 0; j < w[s]; ++j) {
                int64_t e = base + (int64_t)j * kSlice + l;
                if (j < c) {
                    int64_t src = first[i] + j;
                    out->col[e] = colmap(ci[src]);
                    out->val[e] = va[src];
                } else {
                    out->col[e] = pad;
                    out->val[e] = 0.0;
                }
            }
        }
    }
}

// Offset-aligned packing of a LOCAL part (stencil-like matrices): slice s
// stores, for every offset o in the sorted union U_s of (column - row) over its
// rows, one entry per row — the row's a_{i,i+o} or a pad (val 0) — so a slice
// needs one int32 offset per entry position instead of one column per entry.
// Within each row the entries stay in ascending column order (pads add 0).
// Used only if the union widens the slices by at most 15 %, pads are at
// most 3 % of the stored entries and no slice's union exceeds 2 w + 8 (the
// device builder, builder_gpu.cu, takes the same decision).
bool pack_aligned(int64_t n, int64_t rb, const std::vector<int32_t> &cnt, const std::vector<int64_t> &first,
                  const int64_t *ci, const double *va, SellHost *out) {
    const int64_t ns = (n + kSlice - 1) / kSlice;
    std::vector<std::vector<int32_t>> uni(ns);
    std::vector<int64_t> wc(ns, 0);
    int64_t sum_u = 0, sum_c = 0;
    int over = 0;
#pragma omp parallel for schedule(static) reduction(+ : sum_u, sum_c) reduction(max : over)
    for (int64_t s = 0; s < ns; ++s) {
        std::vector<int32_t> &u = uni[s];
        int32_t m = 0;
        for (int64_t i = s * kSlice; i < std::min(n, (s + 1) * kSlice); ++i) {
            m = std::max(m, cnt[i]);
            for (int32_t j = 0; j < cnt[i]; ++j) u.push_back((int32_t)(ci[first[i] + j] - rb - i));
        }
        std::sort(u.begin(), u.end());
        u.erase(std::unique(u.begin(), u.end()), u.end());
        if ((int64_t)u.size() > 2 * (int64_t)m + 8) over = 1;  // a scattered slice: keep it compact
        wc[s] = m;
        sum_u += (int64_t)u.size();
        sum_c += m;
    }
    // profitable only with (almost) no pads: a pad gathers a column the row
    // does not couple to (lexicographic stencils: grid-line ends only)
    int64_t nnz_part = 0;
    for (int64_t i = 0; i < n; ++i) nnz_part += cnt[i];
    if (over || sum_c == 0 || sum_u * 100 > sum_c * 115 || (sum_u * kSlice - nnz_part) * 100 > sum_u * kSlice * 3)
        return false;
    out->ptr.assign(ns + 1, 0);
    int32_t maxw = 0;
    int64_t nnz = 0;
    for (int64_t s = 0; s < ns; ++s) {
        out->ptr[s + 1] = out->ptr[s] + (int64_t)uni[s].size() * kSlice;
        maxw = std::max(maxw, (int32_t)uni[s].size());
    }
    for (int64_t i = 0; i < n; ++i) nnz += cnt[i];
    out->maxw = maxw;
    out->nnz = nnz;
    const int64_t tot = out->ptr[ns];
    out->col.assign(tot, 0);
    out->val.assign(tot, 0.0);
    out->off.assign(tot / kSlice, 0);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < ns; ++s) {
        const std::vector<int32_t> &u = uni[s];
        const int64_t base = out->ptr[s];
        for (size_t j = 0; j < u.size(); ++j) out->off[base / kSlice + j] = u[j];
        for (int l = 0; l < kSlice; ++l) {
            const int64_t i = s * kSlice + l;
            int32_t q = 0;  // next entry of the row
            for (size_t j = 0; j < u.size(); ++j) {
                const int64_t e = base + (int64_t)j * kSlice + l;
                const int64_t c = i + u[j];
                if (i < n && q < cnt[i] && ci[first[i] + q] - rb == c) {
                    out->col[e] = (int32_t)c;
                    out->val[e] = va[first[i] + q];
                    ++q;
                } else {  // pad: val 0 at row + offset (or the row itself when out of range)
                    out->col[e] = (int32_t)((i < n && c >= 0 && c < n) ? c : (i < n ? i : 0));
                    out->val[e] = 0.0;
                }
            }
        }
    }
    return true;
}

struct LocalMap {
    int64_t rb;
    int32_t operator()(int64_t c) const { return (int32_t)(c - rb); }
    int32_t pad(int64_t i) const { return (int32_t)i; }
};
struct GhostMap {
    const std::vector<int64_t> *gid;
    int32_t operator()(int64_t c) const {
        return (int32_t)(std::lower_bound(gid->begin(), gid->end(), c) - gid->begin());
    }
    int32_t pad(int64_t) const { return 0; }
};

}  // namespace

// Gather-window plan (nsm_internal.h "Window"): per tile the ranges
// [row0_s + o, row0_s + 32 + o) of every entry position of every slice of the
// group's parts, aligned to even indices (16-byte bulk copies), sorted and
// merged when they overlap or lie within 32 values of each other.
bool build_window(int64_t n, const std::vector<const SellHost *> &parts, int32_t wcap, WindowHost *out) {
    const int np = (int)parts.size();
    if (np < 1 || np > 2) return false;
    for (const SellHost *p : parts)
        if (p->off.empty()) return false;
    const int64_t ns = (n + kSlice - 1) / kSlice;
    const int64_t nt = (ns + kTileSlices - 1) / kTileSlices;
    struct Seg { int64_t lo, hi; };
    std::vector<std::vector<Seg>> segs(nt);
    bool ok = true;
    for (int p = 0; p < np; ++p) out->wpos[p].assign(parts[p]->off.size(), 0);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t t = 0; t < nt; ++t) {
        const int64_t s0 = t * kTileSlices, s1 = std::min(ns, s0 + kTileSlices);
        std::vector<Seg> r;
        for (int p = 0; p < np; ++p)
            for (int64_t s = s0; s < s1; ++s) {
                const int64_t e0 = parts[p]->ptr[s] / kSlice, e1 = parts[p]->ptr[s + 1] / kSlice;
                for (int64_t e = e0; e < e1; ++e) {
                    const int64_t lo = s * kSlice + parts[p]->off[e];
                    r.push_back(Seg{lo & ~(int64_t)1, (lo + kSlice + 1) & ~(int64_t)1});
                }
            }
        std::sort(r.begin(), r.end(), [](const Seg &a, const Seg &b) { return a.lo < b.lo; });
        std::vector<Seg> m;
        for (const Seg &g : r) {
            if (!m.empty() && g.lo <= m.back().hi + kSlice) m.back().hi = std::max(m.back().hi, g.hi);
            else m.push_back(g);
        }
        int64_t tot = 0;
        for (const Seg &g : m) tot += g.hi - g.lo;
        if (tot > wcap || m.size() > 32) {
#pragma omp atomic write
            ok = false;
        }
        // window positions of every (slice, entry) of the tile
        std::vector<int64_t> base(m.size());
        int64_t acc = 0;
        for (size_t k = 0; k < m.size(); ++k) { base[k] = acc; acc += m[k].hi - m[k].lo; }
        for (int p = 0; p < np; ++p)
            for (int64_t s = s0; s < s1; ++s) {
                const int64_t e0 = parts[p]->ptr[s] / kSlice, e1 = parts[p]->ptr[s + 1] / kSlice;
                for (int64_t e = e0; e < e1; ++e) {
                    const int64_t lo = s * kSlice + parts[p]->off[e];
                    size_t k = std::upper_bound(m.begin(), m.end(), lo, [](int64_t v, const Seg &g) { return v < g.lo; }) -
                               m.begin() - 1;
                    out->wpos[p][e] = (int32_t)(base[k] + (lo - m[k].lo));
                }
            }
        segs[t] = std::move(m);
    }
    if (!ok) return false;
    // Worth it only where each staged window value replaces several gathers:
    // measured a win for 27-point rows (window / gathers 0.35-0.4: C3
    // residual 0.83 -> 0.94 of peak, sweeps 0.77 -> 0.97) and a loss for
    // 7-point rows (0.85-1.0: the per-tile window bookkeeping of the
    // producer is not hidden behind a tile that small; C5 0.59 -> 0.97 ms).
    int64_t entries = 0, wtot = 0;
    for (const SellHost *p : parts) entries += p->ptr[ns];
    for (int64_t t = 0; t < nt; ++t)
        for (const Seg &g : segs[t]) wtot += g.hi - g.lo;
    if (wtot * 2 > entries && !knob("NSM_WINDOW_ALWAYS")) return false;   // (experiments: windows for any ratio)
    out->tseg.assign(nt + 1, 0);
    for (int64_t t = 0; t < nt; ++t) out->tseg[t + 1] = out->tseg[t] + (int32_t)segs[t].size();
    const int64_t nseg = out->tseg[nt];
    out->glo.resize(nseg);
    out->len.resize(nseg);
    out->sbase.resize(nseg);
    out->wmax = 0;
    out->maxseg = 0;
    for (int64_t t = 0; t < nt; ++t) {
        int32_t acc = 0;
        for (size_t k = 0; k < segs[t].size(); ++k) {
            const int64_t q = out->tseg[t] + (int64_t)k;
            out->glo[q] = segs[t][k].lo;
            out->len[q] = (int32_t)(segs[t][k].hi - segs[t][k].lo);
            out->sbase[q] = acc;
            acc += out->len[q];
        }
        out->wmax = std::max(out->wmax, acc);
        out->maxseg = std::max(out->maxseg, (int32_t)segs[t].size());
    }
    return true;
}


nsm_status build_split(const nsm_csr *A, int64_t rb, int64_t re, Split *out, std::string *err) {
    const int64_t n = A->nrows;
    const int64_t *rp = A->rowptr;
    const int64_t *ci = A->colind;
    const double *va = A->val;
    if (n != re - rb || n < 0 || !rp || (rp[n] > 0 && (!ci || !va))) {
        *err = "nsm_setup: inconsistent CSR arguments";
        return NSM_ERR_ARG;
    }
    if (n >= (int64_t)1 << 31 || A->ncols >= (int64_t)1 << 31) {
        *err = "nsm_setup: more than 2^31-1 rows/columns per rank is not supported (int32 device indices)";
        return NSM_ERR_ARG;
    }
    if (rp[0] != 0) { *err = "nsm_setup: rowptr[0] != 0"; return NSM_ERR_PATTERN; }
    // ---- validate (P:L717-721 needs a nonzero diagonal; S:L24-27 invariants)
    int bad_kind = 0;  // 1 pattern, 2 diagonal
#pragma omp parallel for schedule(static) reduction(max : bad_kind)
    for (int64_t i = 0; i < n; ++i) {
        int kind = 0;
        if (rp[i + 1] < rp[i]) kind = 1;
        else {
            bool has_d = false;
            for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
                int64_t c = ci[p];
                if (c < 0 || c >= A->ncols || (p > rp[i] && ci[p - 1] >= c)) { kind = 1; break; }
                if (c == rb + i) has_d = va[p] != 0.0 && std::isfinite(va[p]);
            }
            if (!kind && !has_d) kind = 2;
        }
        bad_kind = std::max(bad_kind, kind);
    }
    if (bad_kind) {
        // report the first offending row deterministically
        for (int64_t i = 0; i < n; ++i) {
            bool pat = rp[i + 1] < rp[i], has_d = false;
            for (int64_t p = rp[i]; !pat && p < rp[i + 1]; ++p) {
                int64_t c = ci[p];
                if (c < 0 || c >= A->ncols || (p > rp[i] && ci[p - 1] >= c)) pat = true;
                else if (c == rb + i) has_d = va[p] != 0.0 && std::isfinite(va[p]);
            }
            if (pat) {
                *err = "nsm_setup: CSR pattern invariant violated at global row " + std::to_string(rb + i);
                return NSM_ERR_PATTERN;
            }
            if (!has_d) {
                *err = "nsm_setup: missing or zero diagonal at global row " + std::to_string(rb + i);
                return NSM_ERR_ZERO_DIAG;
            }
        }
    }
    // ---- per-row part counts
    std::vector<int32_t> cnt[5];
    std::vector<int64_t> first[5];
    for (int k = 0; k < 5; ++k) { cnt[k].assign(n, 0); first[k].assign(n, 0); }
    out->d.assign(n, 0.0);
    out->dl1.assign(n, 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        for (int k = 0; k < 5; ++k) first[k][i] = rp[i];
        int prev = -1;
        double l1 = 0.0;  // sum of |a_ij|, j != i, ascending columns
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            int k = classify(rb + i, ci[p], rb, re);
            if (k != prev) { first[k][i] = p; prev = k; }
            cnt[k][i]++;
            if (k == P_D) out->d[i] = va[p];
            else l1 = l1 + std::fabs(va[p]);
        }
        out->dl1[i] = out->d[i] + l1;
    }
    // ---- ghost columns (ascending global ids)
    std::vector<int64_t> &g = out->ghost_gid;
    g.clear();
    for (int64_t i = 0; i < n; ++i) {
        for (int k : {P_LG, P_UG})
            for (int32_t j = 0; j < cnt[k][i]; ++j) g.push_back(ci[first[k][i] + j]);
    }
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    out->n = n;
    out->row_begin = rb;
    out->n_ghost = (int64_t)g.size();
    LocalMap lm{rb};
    GhostMap gm{&g};
    static const bool no_align = knob("NSM_NO_ALIGNED_LAYOUT") != nullptr;  // A/B experiments
    if (no_align || !pack_aligned(n, rb, cnt[P_L], first[P_L], ci, va, &out->L))
        pack(n, cnt[P_L], first[P_L], ci, va, lm, &out->L);
    if (no_align || !pack_aligned(n, rb, cnt[P_U], first[P_U], ci, va, &out->U))
        pack(n, cnt[P_U], first[P_U], ci, va, lm, &out->U);
    pack(n, cnt[P_LG], first[P_LG], ci, va, gm, &out->LG);
    pack(n, cnt[P_UG], first[P_UG], ci, va, gm, &out->UG);
    out->nnz_off = out->L.nnz + out->U.nnz + out->LG.nnz + out->UG.nnz;
    // local lower / upper bandwidths (dependency distances of the fused kernel)
    int64_t bwl = 0, bwu = 0;
#pragma omp parallel for schedule(static) reduction(max : bwl, bwu)
    for (int64_t i = 0; i < n; ++i) {
        if (cnt[P_L][i] > 0) bwl = std::max(bwl, rb + i - ci[first[P_L][i]]);
        if (cnt[P_U][i] > 0) bwu = std::max(bwu, ci[first[P_U][i] + cnt[P_U][i] - 1] - rb - i);
    }
    out->bw_lower = bwl;
    out->bw_upper = bwu;
    return NSM_OK;
}

// ILU(0) on the pattern of A (IKJ, no pivoting, the building
// block of P:L945 / P:L1409-1421).  Row i is eliminated with the already
// factored rows k < i in ascending k; the update of entry (i, j) by row k is
// found by merging the sorted column lists of rows i and k (entries outside
// the pattern are dropped: zero fill).  With row_begin the block is the
// diagonal block of a row partition: columns outside [row_begin, row_begin+n)
// are not eliminated and get the value 0.
nsm_status ilu0_host(const nsm_csr *A, int64_t rb, double *fval, std::string *err) {
    const int64_t n = A->nrows;
    const int64_t *rp = A->rowptr;
    const int64_t *ci = A->colind;
    const double *va = A->val;
    if (!rp || !fval || n < 0 || (rp[n] > 0 && (!ci || !va))) { *err = "nsm_ilu0: bad argument"; return NSM_ERR_ARG; }
    const int64_t re = rb + n;
    std::vector<int64_t> dpos(n, -1);
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            if (ci[p] == rb + i) dpos[i] = p;
            bool inblock = ci[p] >= rb && ci[p] < re;
            fval[p] = inblock ? va[p] : 0.0;
        }
        if (dpos[i] < 0) {
            *err = "nsm_ilu0: missing diagonal at global row " + std::to_string(rb + i);
            return NSM_ERR_ZERO_DIAG;
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        const int64_t gi = rb + i;
        for (int64_t p = rp[i]; p < rp[i + 1] && ci[p] < gi; ++p) {
            if (ci[p] < rb) continue;  // other rank's column: not part of A_pp
            const int64_t k = ci[p] - rb;
            const double ukk = fval[dpos[k]];
            if (ukk == 0.0) {
                *err = "nsm_ilu0: zero pivot at global row " + std::to_string(rb + k);
                return NSM_ERR_ZERO_DIAG;
            }
            const double lik = fval[p] / ukk;
            fval[p] = lik;
            // merge row k (columns > k) with row i (columns > ci[p])
            int64_t q = dpos[k] + 1, t = p + 1;
            const int64_t qe = rp[k + 1], te = rp[i + 1];
            while (q < qe && t < te) {
                const int64_t cq = ci[q], ct = ci[t];
                if (cq >= re) break;
                if (cq < ct) ++q;
                else if (ct < cq) ++t;
                else { fval[t] = fval[t] - lik * fval[q]; ++q; ++t; }
            }
        }
        if (fval[dpos[i]] == 0.0) {
            *err = "nsm_ilu0: zero pivot at global row " + std::to_string(gi);
            return NSM_ERR_ZERO_DIAG;
        }
    }
    return NSM_OK;
}

}  // namespace nsm

// ---- ILUT(droptol, lfil) and Ruiz scaling (Alg. 2; NEXT-3) ----
// Saad's dual-threshold ILUT, row by row: the pivots k < i of the working
// row are eliminated in ascending column order (a min-heap, fill included);
// w_k / u_kk below tau_i = droptol * ||a_i||_2 is dropped, otherwise row k of
// U is subtracted; then off-diagonal entries below tau_i are dropped and the
// lfil largest of the L part and of the U part kept (ties: smaller column).
#include <queue>

namespace nsm {

nsm_status ilut_host(const nsm_csr *A, double droptol, int lfil, std::vector<int64_t> &rp_out,
                     std::vector<int64_t> &ci_out, std::vector<double> &va_out, std::string *err) {
    const int64_t n = A->nrows;
    if (!A->rowptr || n < 0 || A->ncols != n || droptol < 0 || lfil < 0) { *err = "nsm_ilut: bad argument"; return NSM_ERR_ARG; }
    std::vector<double> w(n, 0.0);
    std::vector<char> present(n, 0);
    std::vector<int64_t> nz;
    // U rows kept for elimination: start offsets into (ucol, uval)
    std::vector<int64_t> ustart(n + 1, 0), ucol;
    std::vector<double> uval;
    rp_out.assign(n + 1, 0);
    ci_out.clear();
    va_out.clear();
    for (int64_t i = 0; i < n; ++i) {
        double nrm2 = 0.0;
        nz.clear();
        std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> heap;
        for (int64_t p = A->rowptr[i]; p < A->rowptr[i + 1]; ++p) {
            const int64_t j = A->colind[p];
            nrm2 = nrm2 + A->val[p] * A->val[p];
            w[j] = A->val[p];
            present[j] = 1;
            nz.push_back(j);
            if (j < i) heap.push(j);
        }
        const double tau = droptol * std::sqrt(nrm2);
        std::vector<int64_t> dropped;
        while (!heap.empty()) {
            const int64_t k = heap.top();
            heap.pop();
            const double ukk = uval[ustart[k]];  // diagonal is the first entry of U row k
            const double wk = w[k] / ukk;
            if (std::fabs(wk) < tau) {
                w[k] = 0.0;
                dropped.push_back(k);
                continue;
            }
            w[k] = wk;
            for (int64_t q = ustart[k] + 1; q < ustart[k + 1]; ++q) {
                const int64_t j = ucol[q];
                if (!present[j]) {
                    present[j] = 1;
                    w[j] = 0.0;
                    nz.push_back(j);
                    if (j < i) heap.push(j);
                }
                w[j] = w[j] - wk * uval[q];
            }
        }
        for (int64_t k : dropped) present[k] = 2;  // removed from the row
        if (!present[i] || w[i] == 0.0) {
            *err = "nsm_ilut: zero pivot at row " + std::to_string(i);
            for (int64_t j : nz) { present[j] = 0; w[j] = 0.0; }
            return NSM_ERR_ZERO_DIAG;
        }
        std::vector<std::pair<int64_t, double>> lpart, upart;
        for (int64_t j : nz) {
            if (present[j] != 1 || j == i) continue;
            if (std::fabs(w[j]) < tau) continue;
            (j < i ? lpart : upart).push_back({j, w[j]});
        }
        auto bigger = [](const std::pair<int64_t, double> &a, const std::pair<int64_t, double> &b) {
            const double fa = std::fabs(a.second), fb = std::fabs(b.second);
            return fa != fb ? fa > fb : a.first < b.first;
        };
        std::sort(lpart.begin(), lpart.end(), bigger);
        std::sort(upart.begin(), upart.end(), bigger);
        if ((int64_t)lpart.size() > lfil) lpart.resize(lfil);
        if ((int64_t)upart.size() > lfil) upart.resize(lfil);
        std::vector<std::pair<int64_t, double>> row(lpart);
        row.push_back({i, w[i]});
        row.insert(row.end(), upart.begin(), upart.end());
        std::sort(row.begin(), row.end());
        for (auto &e : row) { ci_out.push_back(e.first); va_out.push_back(e.second); }
        rp_out[i + 1] = (int64_t)ci_out.size();
        // U row i (diagonal first, then ascending columns)
        ustart[i] = (int64_t)ucol.size();
        ucol.push_back(i);
        uval.push_back(w[i]);
        for (auto &e : upart) (void)e;
        std::vector<std::pair<int64_t, double>> us(upart);
        std::sort(us.begin(), us.end());
        for (auto &e : us) { ucol.push_back(e.first); uval.push_back(e.second); }
        ustart[i + 1] = (int64_t)ucol.size();
        for (int64_t j : nz) { present[j] = 0; w[j] = 0.0; }
    }
    return NSM_OK;
}

// Ruiz equilibration of the upper part (incl. diagonal) of a factor CSR, then
// an exact unit diagonal; the scaling is returned as divisors s_r, s_c.
// Departure from normality of the U part (upper incl. diagonal) of a factor
// CSR with values v: Henrici's dep(A) = sqrt(||A||_F^2 - ||Lambda||_F^2)
// (P:L847-855); a triangular matrix's eigenvalues are its diagonal entries,
// so dep(U) = ||U_s||_F.  Row-wise sums in stored order, then over rows.
static double dep_upper(const nsm_csr *F, const double *v) {
    double s = 0.0;
    for (int64_t i = 0; i < F->nrows; ++i) {
        double r = 0.0;
        for (int64_t p = F->rowptr[i]; p < F->rowptr[i + 1]; ++p)
            if (F->colind[p] > i) r = r + v[p] * v[p];
        s = s + r;
    }
    return std::sqrt(s);
}

nsm_status ruiz_host(const nsm_csr *F, int max_iters, double *v, double *s_r, double *s_c, std::string *err,
                     double dep_tol, int *iters_done, double *dep_hist) {
    const int64_t n = F->nrows;
    if (!F->rowptr || n < 0 || max_iters < 0) { *err = "nsm_ruiz: bad argument"; return NSM_ERR_ARG; }
    const int64_t nnz = F->rowptr[n];
    std::copy(F->val, F->val + nnz, v);
    for (int64_t i = 0; i < n; ++i) { s_r[i] = 1.0; s_c[i] = 1.0; }
    std::vector<double> rmax(n), cmax(n);
    int it = 0;
    if (dep_hist) dep_hist[0] = dep_upper(F, v);
    while (it < max_iters) {
        std::fill(rmax.begin(), rmax.end(), 0.0);
        std::fill(cmax.begin(), cmax.end(), 0.0);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t p = F->rowptr[i]; p < F->rowptr[i + 1]; ++p) {
                const int64_t j = F->colind[p];
                if (j < i) continue;
                rmax[i] = std::max(rmax[i], std::fabs(v[p]));
                cmax[j] = std::max(cmax[j], std::fabs(v[p]));
            }
        for (int64_t i = 0; i < n; ++i) {
            rmax[i] = rmax[i] == 0.0 ? 1.0 : std::sqrt(rmax[i]);
            cmax[i] = cmax[i] == 0.0 ? 1.0 : std::sqrt(cmax[i]);
        }
        for (int64_t i = 0; i < n; ++i)
            for (int64_t p = F->rowptr[i]; p < F->rowptr[i + 1]; ++p) {
                const int64_t j = F->colind[p];
                if (j >= i) v[p] = v[p] / rmax[i] / cmax[j];
            }
        for (int64_t i = 0; i < n; ++i) { s_r[i] = s_r[i] * rmax[i]; s_c[i] = s_c[i] * cmax[i]; }
        ++it;
        // early termination on the departure from normality:
        // dep(U) after this round below the caller's tolerance
        if (dep_hist || dep_tol > 0.0) {
            const double dk = dep_upper(F, v);
            if (dep_hist) dep_hist[it] = dk;
            if (dep_tol > 0.0 && dk < dep_tol) break;
        }
    }
    if (iters_done) *iters_done = it;
    for (int64_t i = 0; i < n; ++i) {
        double dg = 1.0;
        bool has = false;
        for (int64_t p = F->rowptr[i]; p < F->rowptr[i + 1]; ++p)
            if (F->colind[p] == i) { dg = v[p]; has = true; }
        if (!has || dg == 0.0) { *err = "nsm_ruiz: missing or zero diagonal at row " + std::to_string(i); return NSM_ERR_ZERO_DIAG; }
        for (int64_t p = F->rowptr[i]; p < F->rowptr[i + 1]; ++p)
            if (F->colind[p] >= i) v[p] = v[p] / dg;
        s_r[i] = s_r[i] * dg;
    }
    return NSM_OK;
}

// Departure-from-normality diagnostics of a triangular factor (P:L847-855,
// Theorem 3, Definition 2 / Theorem 4).
nsm_status dep_host(const nsm_csr *F, const double *val, int upper, nsm_dep_info *out, std::string *err) {
    if (!F || !F->rowptr || !out || F->nrows < 0 || (F->rowptr[F->nrows] > 0 && (!F->colind || !(val ? val : F->val)))) {
        *err = "nsm_dep: bad argument";
        return NSM_ERR_ARG;
    }
    const double *v = val ? val : F->val;
    const int64_t n = F->nrows;
    double strict = 0.0, diag = 0.0, delta = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double r2 = 0.0, rabs = 0.0, dii = upper ? 0.0 : 1.0;  // unit-lower L: implicit diagonal 1
        for (int64_t p = F->rowptr[i]; p < F->rowptr[i + 1]; ++p) {
            const int64_t j = F->colind[p];
            if (upper ? j > i : j < i) {
                r2 = r2 + v[p] * v[p];
                rabs = rabs + std::fabs(v[p]);
            } else if (upper && j == i) {
                dii = v[p];
            }
        }
        strict = strict + r2;
        diag = diag + dii * dii;
        delta = std::max(delta, rabs - std::fabs(dii));   // delta_i of Definition 2 (>= 0)
    }
    out->n = n;
    out->dep = std::sqrt(strict);                 // eigenvalues = diagonal: dep = ||T_s||_F
    out->fro_strict = std::sqrt(strict);
    out->fro = std::sqrt(strict + diag);
    out->delta = delta;
    const double sq = std::sqrt((double)n);
    out->bound_thm3 = std::sqrt((2.0 * sq + out->fro_strict) * out->fro_strict);
    out->bound_table5 = std::sqrt((2.0 * sq + out->fro) * out->fro);
    out->bound_thm4 = sq * (1.0 + delta);
    return NSM_OK;
}

}  // namespace nsm
