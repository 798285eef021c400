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
// fills levels[] before calling.  Inserts run as a speculative parallel build (Workers,
// below) whose result is, by construction, the sequential graph.
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include <sys/mman.h>

#include "../../include/gmpgr.h"

namespace {

inline bool before(double d1, int64_t i1, double d2, int64_t i2) {
    return d1 < d2 || (d1 == d2 && i1 < i2);
}

// Anonymous mapping with transparent huge pages requested (madvise mode is common): the
// build's arrays are GBs of random-access data, 4 KB pages would make every row a TLB miss.
// Zero-filled.
template <class T>
struct Huge {
    T *p = nullptr;
    size_t bytes = 0;
    Huge() = default;
    Huge(const Huge &) = delete;
    Huge &operator=(const Huge &) = delete;
    ~Huge() { release(); }
    bool alloc(size_t count) {
        release();
        const size_t hp = 2u << 20;
        bytes = std::max<size_t>(hp, (count * sizeof(T) + hp - 1) / hp * hp);
        void *m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (m == MAP_FAILED) { p = nullptr; bytes = 0; return false; }
        madvise(m, bytes, MADV_HUGEPAGE);
        p = static_cast<T *>(m);
        return true;
    }
    void release() {
        if (p) munmap(p, bytes);
        p = nullptr;
        bytes = 0;
    }
    T &operator[](size_t i) { return p[i]; }
    const T &operator[](size_t i) const { return p[i]; }
};

// Rows and counts are read by planning threads while the committing thread rewrites them:
// relaxed atomic accesses (plain moves on x86).  A plan that read a row modified after it
// started is discarded (Plan::base / Builder::mod), so such reads never reach the graph.
inline int32_t ld(const int32_t *p) { return __atomic_load_n(p, __ATOMIC_RELAXED); }
inline void st(int32_t *p, int32_t v) { __atomic_store_n(p, v, __ATOMIC_RELAXED); }

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

// Per-thread search context: heaps, buffers, a private visited-stamp array (equivalent to
// the reference's shared one: each _search call sees a fresh visited set) and the record of
// adjacency rows the searches READ (for the speculative parallel build below).
struct Ctx {
    Heap cand, res;
    Huge<uint32_t> stamps;
    uint32_t stamp = 0;
    std::vector<int64_t> fresh;
    std::vector<double> fresh_d, diffs;
    std::vector<uint64_t> reads;  // layer << 32 | node of every expanded row
};

// The searches and selections of one insert, computed without writing the graph.
struct Plan {
    int64_t slot = -1;
    int level = 0;
    int32_t entry = -1, top = -1;       // graph entry / top level the plan was made against
    int64_t base = -1;                   // first uncommitted slot when planned (-1: no plan)
    std::vector<int64_t> kept[GR_MAX_GRAPH_LAYERS];  // neighbours to connect per layer
    std::vector<double> kept_d[GR_MAX_GRAPH_LAYERS];  // their einsum distances to the new node
    std::vector<uint64_t> reads;
    std::vector<uint64_t> rset;  // open-addressing set of `reads` (~0 = empty)

    void index_reads() {
        size_t cap = 16;
        while (cap < 2 * reads.size()) cap <<= 1;
        rset.assign(cap, ~0ull);
        for (uint64_t r : reads) {
            size_t h = (size_t)((r * 0x9E3779B97F4A7C15ull) >> 40) & (cap - 1);
            while (rset[h] != ~0ull && rset[h] != r) h = (h + 1) & (cap - 1);
            rset[h] = r;
        }
    }
    bool has_read(uint64_t r) const {
        const size_t cap = rset.size();
        size_t h = (size_t)((r * 0x9E3779B97F4A7C15ull) >> 40) & (cap - 1);
        while (rset[h] != ~0ull) {
            if (rset[h] == r) return true;
            h = (h + 1) & (cap - 1);
        }
        return false;
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
    // rows modified by each of the last MR commits (layer << 32 | node): a plan made when
    // `base` slots were committed is still exact at slot s iff no commit in [base, s)
    // modified a row it read
    std::vector<std::vector<uint64_t>> modlog;
    int64_t MR = 1;
    int64_t cur = -1;  // slot being committed
    std::vector<double> diffs;
    // rowd[l][s * cap_l + j]: einsum distance of row s's j-th neighbour to s (the values the
    // capacity re-selection sorts, index.py:265-268), kept in step with the rows so a
    // re-selection computes one new distance instead of cap + 1
    Huge<double> rowd[GR_MAX_GRAPH_LAYERS];

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
    double einsum_dist(int64_t a, int64_t b, std::vector<double> &buf) const {  // (V[a] - V[b]) . itself
        const double *va = row(a), *vb = row(b);
        for (int j = 0; j < dim; ++j) buf[j] = va[j] - vb[j];
        return einsum_sq(buf.data(), dim);
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

    // kernels/_chot.pyx:116-179; returns (slots, dist2) ascending.  Reads only.
    void search(Ctx &c, int layer, const double *q, const std::vector<int64_t> &entries, int ef,
                std::vector<int64_t> &out_i, std::vector<double> &out_d) const {
        if (++c.stamp == 0) {  // u32 wrap: restart the private visited stamps
            std::memset(c.stamps.p, 0, c.stamps.bytes);
            c.stamp = 1;
        }
        const uint32_t stamp = c.stamp;
        uint32_t *stamps = c.stamps.p;
        const int32_t *nb = nbrs[layer];
        const int32_t *ct = cnts[layer];
        const int capl = cap_of(layer);
        Heap &res = c.res, &cand = c.cand;
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
            c.reads.push_back(((uint64_t)layer << 32) | (uint64_t)node);
            const int cn = ld(ct + node);
            const int32_t *r = nb + node * (int64_t)capl;
            // stamp in row order and compute the distances of the unvisited neighbours first
            // (pure), then run the reference's admission logic over them in the same order
            c.fresh.clear();
            for (int j = 0; j < cn; ++j) {
                const int64_t v = ld(r + j);
                if (stamps[v] == stamp) continue;
                stamps[v] = stamp;
                c.fresh.push_back(v);
            }
            const int nf = (int)c.fresh.size();
            c.fresh_d.resize(nf);
            // rows are random accesses into a table far larger than the caches: start every
            // line of every row now so the distance chains below stream from L1/L2
            for (int j = 0; j < nf; ++j) {
                const char *p = reinterpret_cast<const char *>(row(c.fresh[j]));
                for (int b = 0; b < dim * 8; b += 64) __builtin_prefetch(p + b);
            }
            for (int j = 0; j < nf; j += 8)
                dist2_x8(c.fresh.data() + j, std::min(8, nf - j), q, c.fresh_d.data() + j);
            for (int j = 0; j < nf; ++j) {
                const int64_t v = c.fresh[j];
                const double dn = c.fresh_d[j];
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
    void select(const int64_t *ci, const double *cd, int64_t nc, int k, std::vector<int64_t> &kept,
                std::vector<double> &buf) const {
        kept.clear();
        if (!heuristic || nc <= k) {
            for (int64_t j = 0; j < std::min<int64_t>(nc, k); ++j) kept.push_back(ci[j]);
            return;
        }
        for (int64_t j = 0; j < nc; ++j) {
            if ((int64_t)kept.size() >= k) break;
            bool dominated = false;
            for (int64_t s : kept)
                if (einsum_dist(s, ci[j], buf) < cd[j]) { dominated = true; break; }
            if (!dominated) kept.push_back(ci[j]);
        }
    }

    // the search / selection half of insert (index.py:283-319): the connects at layer l
    // touch only layer-l rows, so running every layer's search first is equivalent
    void plan(Ctx &c, int64_t slot, int32_t entry, int32_t top, Plan &P) const {
        P.slot = slot;
        P.level = levels[slot];
        P.entry = entry;
        P.top = top;
        c.reads.clear();
        for (int l = 0; l < GR_MAX_GRAPH_LAYERS; ++l) {
            P.kept[l].clear();
            P.kept_d[l].clear();
        }
        if (entry >= 0) {
            const double *q = row(slot);
            std::vector<int64_t> entries{entry}, ci;
            std::vector<double> cd;
            for (int l = top; l > P.level; --l) {
                search(c, l, q, entries, 1, ci, cd);
                entries = ci;
            }
            for (int l = std::min(P.level, (int)top); l >= 0; --l) {
                search(c, l, q, entries, efc, ci, cd);
                select(ci.data(), cd.data(), (int64_t)ci.size(), m, P.kept[l], c.diffs);
                // the connects' new-edge distances are pure: compute them here, off the
                // sequential commit path
                for (int64_t nb : P.kept[l]) P.kept_d[l].push_back(einsum_dist(slot, nb, c.diffs));
                entries = ci;
            }
        }
        P.reads.swap(c.reads);
        P.index_reads();
    }

    bool still_exact(const Plan &P, int64_t s, int32_t entry, int32_t top) const {
        if (P.entry != entry || P.top != top) return false;
        for (int64_t c = P.base; c < s; ++c)
            for (uint64_t r : modlog[c % MR])
                if (P.has_read(r)) return false;
        return true;
    }

    void touch(int layer, int64_t s) { modlog[cur % MR].push_back(((uint64_t)layer << 32) | (uint64_t)s); }

    void row_remove(int layer, int64_t slot, int64_t target) {  // index.py:241-248
        const int64_t base = slot * (int64_t)cap_of(layer);
        int32_t *r = nbrs[layer] + base;
        const int c = cnts[layer][slot];
        for (int j = 0; j < c; ++j)
            if (r[j] == target) {
                st(r + j, r[c - 1]);
                rowd[layer][base + j] = rowd[layer][base + c - 1];
                st(cnts[layer] + slot, c - 1);
                touch(layer, slot);
                return;
            }
    }

    void append(int layer, int64_t slot, int64_t v, double d) {
        const int c = cnts[layer][slot];
        const int64_t base = slot * (int64_t)cap_of(layer);
        st(nbrs[layer] + base + c, (int32_t)v);
        rowd[layer][base + c] = d;
        st(cnts[layer] + slot, c + 1);
        touch(layer, slot);
    }

    // fill the distance cache of rows that existed before this call
    bool init_rowd(int64_t n_old, int64_t n_cap, int T) {
        for (int l = 0; l < max_layers; ++l)
            if (!rowd[l].alloc((size_t)n_cap * cap_of(l))) return false;
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                std::vector<double> buf(dim);
                for (int l = 0; l < max_layers; ++l)
                    for (int64_t s = t; s < n_old; s += T) {
                        const int64_t base = s * (int64_t)cap_of(l);
                        for (int j = 0; j < cnts[l][s]; ++j) rowd[l][base + j] = einsum_dist(nbrs[l][base + j], s, buf);
                    }
            });
        for (auto &x : th) x.join();
        return true;
    }

    // index.py:250-281
    std::vector<int64_t> c_i, c_kept, c_drop;
    std::vector<double> c_d, c_wd;
    // dn = einsum distance of nw and nbr (symmetric: (a - b)^2 == (b - a)^2)
    void connect(int layer, int64_t nw, int64_t nbr, double dn) {
        const int cap = cap_of(layer);
        const int c = cnts[layer][nbr];
        if (c < cap) {
            append(layer, nbr, nw, dn);
            append(layer, nw, nbr, dn);
            return;
        }
        // nb is full: candidates old + [new] sorted by (dist2, id) (stable: unique ids), then
        // re-selected; the row is rewritten in that sorted order
        const int64_t rb = nbr * (int64_t)cap;
        const int32_t *r = nbrs[layer] + rb;
        const int nc = c + 1;
        c_i.resize(nc);
        c_d.resize(nc);
        for (int j = 0; j < nc; ++j) {  // insertion sort (nc <= 2m + 1)
            const int64_t ci = j < c ? (int64_t)r[j] : nw;
            const double cd = j < c ? rowd[layer][rb + j] : dn;
            int k = j;
            while (k > 0 && (c_d[k - 1] > cd || (c_d[k - 1] == cd && ids[c_i[k - 1]] > ids[ci]))) {
                c_i[k] = c_i[k - 1];
                c_d[k] = c_d[k - 1];
                --k;
            }
            c_i[k] = ci;
            c_d[k] = cd;
        }
        select(c_i.data(), c_d.data(), nc, cap, c_kept, diffs);
        const int nk = (int)c_kept.size();
        // kept is an ordered subsequence of the sorted candidates: walk both once; every
        // dropped old neighbour loses its edge back to nbr (each a different row, so the
        // reference's old-row order of these removals does not matter)
        int32_t *w = nbrs[layer] + rb;
        bool nw_kept = false;
        c_drop.clear();
        for (int j = 0, o = 0; o < nc; ++o) {
            if (j < nk && c_i[o] == c_kept[j]) {
                c_wd.push_back(c_d[o]);
                nw_kept |= c_i[o] == nw;
                ++j;
            } else if (c_i[o] != nw) {
                c_drop.push_back(c_i[o]);
            }
        }
        for (int64_t o : c_drop) row_remove(layer, o, nbr);
        for (int j = 0; j < nk; ++j) {
            st(w + j, (int32_t)c_kept[j]);
            rowd[layer][rb + j] = c_wd[j];
        }
        c_wd.clear();
        st(cnts[layer] + nbr, nk);
        touch(layer, nbr);
        if (nw_kept) append(layer, nw, nbr, dn);
    }

    // the write half of insert: connects in the reference's order, entry update
    // start every row a commit of P will touch (the committer calls it one plan ahead too)
    void prefetch_rows(const Plan &P, int32_t top) const {
        for (int l = std::min(P.level, (int)top); l >= 0; --l)
            for (int64_t nb : P.kept[l]) {
                const int64_t rb = nb * (int64_t)cap_of(l);
                __builtin_prefetch(cnts[l] + nb, 1);
                __builtin_prefetch(nbrs[l] + rb, 1);
                for (int b = 0; b < cap_of(l) * 8; b += 64)
                    __builtin_prefetch(reinterpret_cast<const char *>(rowd[l].p + rb) + b, 1);
            }
    }

    void commit(const Plan &P, int32_t &entry, int32_t &top) {
        cur = P.slot;
        modlog[cur % MR].clear();
        for (int l = 0; l < max_layers; ++l) {
            st(cnts[l] + P.slot, 0);
            touch(l, P.slot);
        }
        if (entry < 0) {
            entry = (int32_t)P.slot;
            top = P.level;
            return;
        }
        const int l0 = std::min(P.level, (int)top);
        prefetch_rows(P, top);
        for (int l = l0; l >= 0; --l)
            for (size_t j = 0; j < P.kept[l].size(); ++j) connect(l, P.slot, P.kept[l][j], P.kept_d[l][j]);
        if (P.level > top) {
            top = P.level;
            entry = (int32_t)P.slot;
        }
    }
};

// Speculative parallel build, exact: inserts are taken in windows of W consecutive slots.
// Every slot of a window is planned concurrently against the graph as it stood at the
// window start; the window is then committed in slot order, and a plan is used only if
// none of the rows its searches read has been modified since the window start (and the
// entry point / top level are unchanged) -- then its searches see exactly what they would
// have seen sequentially (new nodes are reachable only through modified rows).  Otherwise
// the slot is re-planned against the current graph.  The result is the sequential graph.
class Workers {
  public:
    explicit Workers(int n) : n_(n) {
        for (int t = 1; t < n; ++t) th_.emplace_back([this, t] { loop(t); });
    }
    ~Workers() {
        stop_ = true;
        gen_.fetch_add(1, std::memory_order_acq_rel);
        for (auto &t : th_) t.join();
    }
    // run fn(worker index) on every worker (the caller is worker 0) and wait for all
    void run(const std::function<void(int)> &fn) {
        fn_ = &fn;
        done_.store(0, std::memory_order_relaxed);
        gen_.fetch_add(1, std::memory_order_acq_rel);
        fn(0);
        while (done_.load(std::memory_order_acquire) != n_ - 1) std::this_thread::yield();
    }

  private:
    void loop(int t) {
        uint64_t seen = 0;
        for (;;) {
            uint64_t g;
            while ((g = gen_.load(std::memory_order_acquire)) == seen) std::this_thread::yield();
            seen = g;
            if (stop_) return;
            (*fn_)(t);
            done_.fetch_add(1, std::memory_order_acq_rel);
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<int> done_{0};
    std::atomic<bool> stop_{false};
    const std::function<void(int)> *fn_ = nullptr;
};

int build_threads() {
    if (const char *e = std::getenv("GMPGR_BUILD_THREADS")) {
        const int v = std::atoi(e);
        if (v >= 1) return v;
    }
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(hc, 64u));
}

}  // namespace

extern "C" int gr_hnsw_insert(int64_t n0, int64_t n1, int32_t dim, const double *vectors,
                              const int64_t *ids, const int32_t *levels, int32_t m,
                              int32_t ef_construction, int32_t max_layers, int select_heuristic,
                              int32_t *const *nbrs, int32_t *const *cnts, int64_t *stamps,
                              int64_t *stamp, int32_t *entry_slot, int32_t *top_level) {
    if (!vectors || !ids || !levels || !nbrs || !cnts || !stamps || !stamp || !entry_slot || !top_level)
        return GR_EINVAL;
    if (n0 < 0 || n1 < n0 || dim < 1 || m < 1 || ef_construction < 1 || max_layers < 1 ||
        max_layers > GR_MAX_GRAPH_LAYERS || n1 > 0x7fffffffLL)
        return GR_EINVAL;
    for (int64_t s = n0; s < n1; ++s)
        if (levels[s] < 0 || levels[s] >= max_layers) return GR_EINVAL;
    Builder B;
    // large builds work on huge-page copies of the vectors and adjacency (copied back below)
    const bool big = n1 >= (1 << 20);
    Huge<double> hvec;
    Huge<int32_t> hnb[GR_MAX_GRAPH_LAYERS], hct[GR_MAX_GRAPH_LAYERS];
    int32_t *wnb[GR_MAX_GRAPH_LAYERS], *wct[GR_MAX_GRAPH_LAYERS];
    auto capl = [&](int l) { return l == 0 ? 2 * (int64_t)m : (int64_t)m; };
    for (int l = 0; l < max_layers; ++l) { wnb[l] = nbrs[l]; wct[l] = cnts[l]; }
    if (big) {
        if (!hvec.alloc((size_t)n1 * dim)) return GR_ENOMEM;
        std::memcpy(hvec.p, vectors, (size_t)n1 * dim * 8);
        for (int l = 0; l < max_layers; ++l) {
            if (!hnb[l].alloc((size_t)n1 * capl(l)) || !hct[l].alloc((size_t)n1)) return GR_ENOMEM;
            std::memcpy(hnb[l].p, nbrs[l], (size_t)n1 * capl(l) * 4);
            std::memcpy(hct[l].p, cnts[l], (size_t)n1 * 4);
            wnb[l] = hnb[l].p;
            wct[l] = hct[l].p;
        }
    }
    B.vec = big ? hvec.p : vectors;
    B.dim = dim;
    B.ids = ids;
    B.levels = levels;
    B.m = m;
    B.efc = ef_construction;
    B.max_layers = max_layers;
    B.heuristic = select_heuristic != 0;
    B.nbrs = wnb;
    B.cnts = wct;
    B.diffs.resize(dim);

    int32_t entry = *entry_slot, top = *top_level;
    const int T = n1 - n0 >= 256 ? build_threads() : 1;
    if (!B.init_rowd(n0, n1, T)) return GR_ENOMEM;
    std::vector<Ctx> ctx(T);
    for (Ctx &c : ctx) {
        if (!c.stamps.alloc((size_t)n1)) return GR_ENOMEM;
        c.cand.reserve((size_t)n1 + 1);
        c.diffs.resize(dim);
    }
    // Pipeline: T - 1 planning threads run ahead of the committing thread by at most R
    // slots, each plan made against the live graph and stamped with the number of slots
    // committed when it started; the committing thread takes the plans in slot order,
    // re-plans the stale ones itself (it is the only writer, so its plans are exact) and
    // commits.
    const int R = T == 1 ? 1 : 2 * T;
    B.MR = R;
    B.modlog.assign(R, {});
    std::vector<Plan> plans(R);  // ring: slot s -> plans[s % R]
    std::vector<std::atomic<int64_t>> ready(R);  // slot whose plan is published in that entry
    for (auto &r : ready) r.store(-1);
    std::atomic<int64_t> committed{n0}, next_plan{n0};
    std::atomic<int32_t> a_entry{entry}, a_top{top};
    int64_t replans = 0, rounds = 0;
    std::atomic<int64_t> early_replans{0};
    double t_commit = 0.0;
    auto planner = [&](int t) {
        for (;;) {
            const int64_t s = next_plan.fetch_add(1);
            if (s >= n1) return;
            while (s >= committed.load(std::memory_order_acquire) + R) std::this_thread::yield();
            Plan &P = plans[s % R];
            int64_t base = committed.load(std::memory_order_acquire);
            B.plan(ctx[t], s, a_entry.load(std::memory_order_acquire), a_top.load(std::memory_order_acquire), P);
            // re-validate against the commits made while planning; re-plan here (off the
            // sequential commit path) while stale.  Commits [base, now) are complete and their
            // modlog entries stay untouched until slot s is committed.
            for (;;) {
                const int64_t now = committed.load(std::memory_order_acquire);
                P.base = base;
                if (B.still_exact(P, now, a_entry.load(std::memory_order_acquire),
                                  a_top.load(std::memory_order_acquire))) {
                    P.base = now;
                    break;
                }
                base = now;
                B.plan(ctx[t], s, a_entry.load(std::memory_order_acquire), a_top.load(std::memory_order_acquire), P);
                ++early_replans;
            }
            ready[s % R].store(s, std::memory_order_release);
        }
    };
    std::vector<std::thread> planners;
    for (int t = 1; t < T; ++t) planners.emplace_back(planner, t);
    for (int64_t s = n0; s < n1; ++s) {
        Plan &P = plans[s % R];
        if (T > 1) {
            while (ready[s % R].load(std::memory_order_acquire) != s) std::this_thread::yield();
        } else {
            B.plan(ctx[0], s, entry, top, P);
            P.base = s;
        }
        const auto tc0 = std::chrono::steady_clock::now();
        if (T > 1 && s + 1 < n1 && ready[(s + 1) % R].load(std::memory_order_acquire) == s + 1)
            B.prefetch_rows(plans[(s + 1) % R], top);  // next commit's rows, one commit ahead
        if (!B.still_exact(P, s, entry, top)) {
            B.plan(ctx[0], s, entry, top, P);
            ++replans;
        }
        B.commit(P, entry, top);
        a_entry.store(entry, std::memory_order_release);
        a_top.store(top, std::memory_order_release);
        ready[s % R].store(-1, std::memory_order_relaxed);
        committed.store(s + 1, std::memory_order_release);
        t_commit += std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count();
    }
    for (auto &th : planners) th.join();
    
    if (std::getenv("GMPGR_BUILD_STATS"))
        std::fprintf(stderr, "[gr_hnsw_insert] %lld inserts, %d threads, window %d, %lld re-planned by planners, %lld by the committer, "
                     "%.2f s in the sequential commit\n",
                     (long long)(n1 - n0), T, R, (long long)early_replans.load(), (long long)replans, t_commit);
    // the reference's shared stamp counter advances once per _search call; callers only
    // compare stamps for equality, so the native build keeps private stamps and leaves
    // the caller's array untouched
    if (big)
        for (int l = 0; l < max_layers; ++l) {
            std::memcpy(nbrs[l], hnb[l].p, (size_t)n1 * capl(l) * 4);
            std::memcpy(cnts[l], hct[l].p, (size_t)n1 * 4);
        }
    *entry_slot = entry;
    *top_level = top;
    return GR_OK;
}
