// Exact native restatement of the reference's sequential index build
// (GraphIndex.insert, /root/reference/pkg/src/nann/index.py:283-319) — host C++,
// part of libgmpgr.so.  The reference spends ~1 ms per insert in the Python driver
// around its Cython beam search; this runs the same algorithm with no
// interpreter in the loop and produces the SAME graph node for node:
//
//   * search_layer: best-first beam search with an epoch-stamp visited array, binary
//     min/max heaps on the lexicographic (dist2, slot) order, identical push/pop
//     sequences (kernels/_chot.pyx:15-179);  dist2 is the plain sequential fp64 sum
//     (_chot.pyx:19-26; this file is compiled with -ffp-contract=off, so no FMA);
//   * _select: keep-M, or the diversity heuristic (index.py:226-239);
//   * _connect: symmetric insertion with capacity re-selection (index.py:250-281),
//     re-selection distances in numpy's fp64 einsum('ij,ij->i') order (2 SSE2 lanes,
//     4x-unrolled 8-blocks, zero-padded pair tail, lane0 + lane1), ties by item id;
//   * _row_remove: swap-with-last (index.py:241-248), so row ORDER matches too.
//
// Level draws stay on the host (numpy Generator stream, index.py:196-209); the caller
// fills levels[] before calling.
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/gmpgr.h"

namespace {

inline bool before(double d1, int64_t i1, double d2, int64_t i2) {
    return d1 < d2 || (d1 == d2 && i1 < i2);
}

struct Heap {  // array heap identical to _chot.pyx's _min_*/_max_* (MAXH: max-heap)
    std::vector<double> d;
    std::vector<int64_t> i;
    int64_t n = 0;
    void reserve(size_t c) {
        if (d.size() < c) { d.resize(c); i.resize(c); }
    }
    template <bool MAXH>
    bool lt(int64_t a, int64_t b) const {  // "a should be above b"
        return MAXH ? before(d[b], i[b], d[a], i[a]) : before(d[a], i[a], d[b], i[b]);
    }
    template <bool MAXH>
    void push(double dd, int64_t ii) {
        int64_t c = n;
        d[c] = dd;
        i[c] = ii;
        n = c + 1;
        while (c > 0) {
            const int64_t p = (c - 1) >> 1;
            if (lt<MAXH>(c, p)) {
                std::swap(d[c], d[p]);
                std::swap(i[c], i[p]);
                c = p;
            } else {
                break;
            }
        }
    }
    template <bool MAXH>
    void pop() {
        const int64_t last = n - 1;
        int64_t c = 0;
        d[0] = d[last];
        i[0] = i[last];
        n = last;
        for (;;) {
            const int64_t l = 2 * c + 1, r = l + 1;
            int64_t m = c;
            if (l < last && lt<MAXH>(l, m)) m = l;
            if (r < last && lt<MAXH>(r, m)) m = r;
            if (m == c) break;
            std::swap(d[c], d[m]);
            std::swap(i[c], i[m]);
            c = m;
        }
    }
};

struct Builder {
    const double *vec;
    int32_t dim;
    const int64_t *ids;
    const int32_t *levels;
    int32_t m, efc, max_layers;
    bool heuristic;
    int32_t *const *nbrs;
    int32_t *const *cnts;
    int64_t *stamps;
    int64_t stamp;
    Heap cand, res;
    std::vector<double> diffs;

    int cap_of(int layer) const { return layer == 0 ? 2 * m : m; }
    const double *row(int64_t s) const { return vec + s * (int64_t)dim; }

    double dist2(int64_t r, const double *q) const {  // _chot.pyx:19-26
        const double *v = row(r);
        double s = 0.0;
        for (int j = 0; j < dim; ++j) {
            const double t = v[j] - q[j];
            s += t * t;
        }
        return s;
    }
    // the same sequential sums for up to 8 rows at once: independent dependency chains
    // (each row's additions stay in order, so every result is bit-identical to dist2)
    void dist2_x8(const int64_t *r, int n, const double *q, double *out) const {
        const double *v[8];
        for (int u = 0; u < 8; ++u) v[u] = row(r[u < n ? u : 0]);
        double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int j = 0; j < dim; ++j) {
            const double qj = q[j];
#pragma GCC unroll 8
            for (int u = 0; u < 8; ++u) {
                const double t = v[u][j] - qj;
                acc[u] += t * t;
            }
        }
        for (int u = 0; u < n; ++u) out[u] = acc[u];
    }
    std::vector<int64_t> fresh;
    std::vector<double> fresh_d;

    // numpy einsum('ij,ij->i') of one fp64 row d[0..K) with itself (oracle sqnorm_rows_f64)
    static double einsum_sq(const double *x, int K) {
        double a0 = 0.0, a1 = 0.0;
        const int nb = K / 8;
        for (int b = 0; b < nb; ++b) {
            const double *p = x + 8 * b;
            double s0 = p[6] * p[6] + a0, s1 = p[7] * p[7] + a1;
            s0 = p[4] * p[4] + s0; s1 = p[5] * p[5] + s1;
            s0 = p[2] * p[2] + s0; s1 = p[3] * p[3] + s1;
            a0 = p[0] * p[0] + s0; a1 = p[1] * p[1] + s1;
        }
        for (int p = 8 * nb; p < K; p += 2) {
            const double x0 = x[p], x1 = p + 1 < K ? x[p + 1] : 0.0;
            a0 = x0 * x0 + a0;
            a1 = x1 * x1 + a1;
        }
        return a0 + a1;
    }
    double einsum_dist(int64_t a, int64_t b) {  // (V[a] - V[b]) . itself
        const double *va = row(a), *vb = row(b);
        for (int j = 0; j < dim; ++j) diffs[j] = va[j] - vb[j];
        return einsum_sq(diffs.data(), dim);
    }
    // einsum_dist(a[u], b) for u < n <= 4, interleaved (each result identical to einsum_dist)
    void einsum_dist_x4(const int64_t *a, int n, int64_t b, double *out) const {
        const double *vb = row(b);
        const double *va[4];
        for (int u = 0; u < 4; ++u) va[u] = row(a[u < n ? u : 0]);
        double l0[4] = {0.0, 0.0, 0.0, 0.0}, l1[4] = {0.0, 0.0, 0.0, 0.0};
        const int nb = dim / 8;
        for (int blk = 0; blk < nb; ++blk) {
            const int p = 8 * blk;
#pragma GCC unroll 4
            for (int u = 0; u < 4; ++u) {
                double x[8];
                for (int t = 0; t < 8; ++t) x[t] = va[u][p + t] - vb[p + t];
                double s0 = x[6] * x[6] + l0[u], s1 = x[7] * x[7] + l1[u];
                s0 = x[4] * x[4] + s0; s1 = x[5] * x[5] + s1;
                s0 = x[2] * x[2] + s0; s1 = x[3] * x[3] + s1;
                l0[u] = x[0] * x[0] + s0; l1[u] = x[1] * x[1] + s1;
            }
        }
        for (int p = 8 * nb; p < dim; p += 2)
            for (int u = 0; u < 4; ++u) {
                const double x0 = va[u][p] - vb[p], x1 = p + 1 < dim ? va[u][p + 1] - vb[p + 1] : 0.0;
                l0[u] = x0 * x0 + l0[u];
                l1[u] = x1 * x1 + l1[u];
            }
        for (int u = 0; u < n; ++u) out[u] = l0[u] + l1[u];
    }

    // kernels/_chot.pyx:116-179; returns (slots, dist2) ascending
    void search(int layer, const double *q, const std::vector<int64_t> &entries, int ef,
                std::vector<int64_t> &out_i, std::vector<double> &out_d) {
        ++stamp;
        const int32_t *nb = nbrs[layer];
        const int32_t *ct = cnts[layer];
        const int capl = cap_of(layer);
        res.reserve((size_t)ef + 1);
        res.n = 0;
        cand.n = 0;
        for (int64_t node : entries) {
            if (stamps[node] == stamp) continue;
            stamps[node] = stamp;
            const double d = dist2(node, q);
            cand.push<false>(d, node);
            res.push<true>(d, node);
            if (res.n > ef) res.pop<true>();
        }
        while (cand.n > 0) {
            const double d = cand.d[0];
            const int64_t node = cand.i[0];
            cand.pop<false>();
            if (res.n >= ef && before(res.d[0], res.i[0], d, node)) break;
            const int c = ct[node];
            const int32_t *r = nb + node * (int64_t)capl;
            // stamp in row order and compute the distances of the unvisited neighbours first
            // (pure), then run the reference's admission logic over them in the same order
            fresh.clear();
            for (int j = 0; j < c; ++j) {
                const int64_t v = r[j];
                if (stamps[v] == stamp) continue;
                stamps[v] = stamp;
                fresh.push_back(v);
            }
            const int nf = (int)fresh.size();
            fresh_d.resize(nf);
            // rows are random accesses into a table far larger than the caches: start every
            // line of every row now so the distance chains below stream from L1/L2
            for (int j = 0; j < nf; ++j) {
                const char *p = reinterpret_cast<const char *>(row(fresh[j]));
                for (int b = 0; b < dim * 8; b += 64) __builtin_prefetch(p + b);
            }
            for (int j = 0; j < nf; j += 8) dist2_x8(fresh.data() + j, std::min(8, nf - j), q, fresh_d.data() + j);
            for (int j = 0; j < nf; ++j) {
                const int64_t v = fresh[j];
                const double dn = fresh_d[j];
                if (res.n >= ef && before(res.d[0], res.i[0], dn, v)) continue;
                cand.push<false>(dn, v);
                res.push<true>(dn, v);
                if (res.n > ef) res.pop<true>();
            }
        }
        const int64_t n = res.n;
        out_i.resize(n);
        out_d.resize(n);
        for (int64_t k = n - 1; k >= 0; --k) {
            out_i[k] = res.i[0];
            out_d[k] = res.d[0];
            res.pop<true>();
        }
    }

    // index.py:226-239
    void select(const int64_t *ci, const double *cd, int64_t nc, int k, std::vector<int64_t> &kept) {
        kept.clear();
        if (!heuristic || nc <= k) {
            for (int64_t j = 0; j < std::min<int64_t>(nc, k); ++j) kept.push_back(ci[j]);
            return;
        }
        for (int64_t j = 0; j < nc; ++j) {
            if ((int64_t)kept.size() >= k) break;
            bool dominated = false;
            for (int64_t s : kept)
                if (einsum_dist(s, ci[j]) < cd[j]) { dominated = true; break; }
            if (!dominated) kept.push_back(ci[j]);
        }
    }

    void row_remove(int layer, int64_t slot, int64_t target) {  // index.py:241-248
        int32_t *r = nbrs[layer] + slot * (int64_t)cap_of(layer);
        const int c = cnts[layer][slot];
        for (int j = 0; j < c; ++j)
            if (r[j] == target) {
                r[j] = r[c - 1];
                cnts[layer][slot] = c - 1;
                return;
            }
    }

    void append(int layer, int64_t slot, int64_t v) {
        const int c = cnts[layer][slot];
        nbrs[layer][slot * (int64_t)cap_of(layer) + c] = (int32_t)v;
        cnts[layer][slot] = c + 1;
    }

    // index.py:250-281
    void connect(int layer, int64_t nw, int64_t nbr) {
        const int cap = cap_of(layer);
        const int c = cnts[layer][nbr];
        if (c < cap) {
            append(layer, nbr, nw);
            append(layer, nw, nbr);
            return;
        }
        const int32_t *r = nbrs[layer] + nbr * (int64_t)cap;
        std::vector<int64_t> old(r, r + c), cands(old);
        cands.push_back(nw);
        const int nc = (int)cands.size();
        std::vector<double> d2(nc);
        for (int j = 0; j < nc; j += 4) einsum_dist_x4(cands.data() + j, std::min(4, nc - j), nbr, d2.data() + j);
        std::vector<int> order(nc);
        for (int j = 0; j < nc; ++j) order[j] = j;
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
            if (d2[a] != d2[b]) return d2[a] < d2[b];
            return ids[cands[a]] < ids[cands[b]];
        });
        std::vector<int64_t> oi(nc), kept;
        std::vector<double> od(nc);
        for (int j = 0; j < nc; ++j) { oi[j] = cands[order[j]]; od[j] = d2[order[j]]; }
        select(oi.data(), od.data(), nc, cap, kept);
        auto in_kept = [&](int64_t s) { return std::find(kept.begin(), kept.end(), s) != kept.end(); };
        for (int64_t o : old)
            if (!in_kept(o)) row_remove(layer, o, nbr);
        int32_t *w = nbrs[layer] + nbr * (int64_t)cap;
        for (size_t j = 0; j < kept.size(); ++j) w[j] = (int32_t)kept[j];
        cnts[layer][nbr] = (int32_t)kept.size();
        if (in_kept(nw)) append(layer, nw, nbr);
    }

    // index.py:283-319 (slot already holds its vector, id and level)
    void insert(int64_t slot, int32_t &entry, int32_t &top) {
        const int level = levels[slot];
        for (int l = 0; l < max_layers; ++l) cnts[l][slot] = 0;
        if (entry < 0) {
            entry = (int32_t)slot;
            top = level;
            return;
        }
        const double *q = row(slot);
        std::vector<int64_t> entries{entry}, ci, kept;
        std::vector<double> cd;
        for (int l = top; l > level; --l) {
            search(l, q, entries, 1, ci, cd);
            entries = ci;
        }
        for (int l = std::min(level, top); l >= 0; --l) {
            search(l, q, entries, efc, ci, cd);
            select(ci.data(), cd.data(), (int64_t)ci.size(), m, kept);
            for (int64_t nb : kept) connect(l, slot, nb);
            entries = ci;
        }
        if (level > top) {
            top = level;
            entry = (int32_t)slot;
        }
    }
};

}  // namespace

extern "C" int gr_hnsw_insert(int64_t n0, int64_t n1, int32_t dim, const double *vectors,
                              const int64_t *ids, const int32_t *levels, int32_t m,
                              int32_t ef_construction, int32_t max_layers, int select_heuristic,
                              int32_t *const *nbrs, int32_t *const *cnts, int64_t *stamps,
                              int64_t *stamp, int32_t *entry_slot, int32_t *top_level) {
    if (!vectors || !ids || !levels || !nbrs || !cnts || !stamps || !stamp || !entry_slot || !top_level)
        return GR_EINVAL;
    if (n0 < 0 || n1 < n0 || dim < 1 || m < 1 || ef_construction < 1 || max_layers < 1 ||
        max_layers > GR_MAX_GRAPH_LAYERS)
        return GR_EINVAL;
    for (int64_t s = n0; s < n1; ++s)
        if (levels[s] < 0 || levels[s] >= max_layers) return GR_EINVAL;
    Builder B;
    B.vec = vectors;
    B.dim = dim;
    B.ids = ids;
    B.levels = levels;
    B.m = m;
    B.efc = ef_construction;
    B.max_layers = max_layers;
    B.heuristic = select_heuristic != 0;
    B.nbrs = nbrs;
    B.cnts = cnts;
    B.stamps = stamps;
    B.stamp = *stamp;
    B.cand.reserve((size_t)n1 + 1);
    B.diffs.resize(dim);
    int32_t entry = *entry_slot, top = *top_level;
    for (int64_t s = n0; s < n1; ++s) B.insert(s, entry, top);
    *stamp = B.stamp;
    *entry_slot = entry;
    *top_level = top;
    return GR_OK;
}
