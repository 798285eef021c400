/*
 * CPU ORACLE — test infrastructure and the CPU-baseline leg of bench.py only.
 * Never linked into, loaded by, or called from the product path.
 *
 * Plain-C restatement of the reference HiPANNS hot path, pinned against the
 * reference's own outputs (tests/golden/ fixtures, tests/test_oracle_golden.py):
 *
 *   - relevance metric: /root/reference/pkg/src/nann/metric.py:102-154
 *     (forward_batch / relevance_batch), with numpy 2.3's fp32
 *     einsum('ij,kj->ik') reduction order (metric.py:30-32): four SSE lanes,
 *     per 16-element block  acc = a0*b0 + (a1*b1 + (a2*b2 + (a3*b3 + acc)))
 *     (separately rounded mul and add), zero-padded groups of four for the
 *     remainder, then (acc0 + acc1) + (acc2 + acc3).  _mm_mul_ps/_mm_add_ps
 *     are exactly those IEEE operations, so this is bit-exact by construction.
 *   - c_hipanns: /root/reference/pkg/src/nann/search.py:194-286, in its
 *     hop-synchronous lowest-searcher-owner form (SURVEY.md §8(a')):
 *     seeds = top-kp of everything scored (pool.py:49-55, search.py:239);
 *     per hop every searcher lists its frontier's rows (search.py:246-252);
 *     the lowest-index searcher listing an unclaimed node owns it
 *     (lock-step claim order, search.py:261-265); each searcher keeps the
 *     top-ef of its own fresh claims (search.py:258-259).
 *   - ordering key (score desc, item id asc) (pool.py:30-55, search.py:258).
 *
 * Build: oracle/Makefile  ->  oracle/_build/liboracle.so
 */
#include <emmintrin.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

#define OMAX_LAYERS 16
#define OMAX_MLP 8

typedef struct {
    int n_mlp;
    int dims[OMAX_MLP + 1];
    const float *W[OMAX_MLP];
    const float *b[OMAX_MLP];
    const float *A;
    int relu;
} omodel;

/* one einsum('ij,kj->ik') output: x[K] . w[K] in numpy's order */
static inline float edot(const float *x, const float *w, int K) {
    __m128 acc = _mm_setzero_ps();
    int nb = K / 16, p;
    for (int blk = 0; blk < nb; ++blk) {
        p = 16 * blk;
        __m128 s = _mm_add_ps(_mm_mul_ps(_mm_loadu_ps(x + p + 12), _mm_loadu_ps(w + p + 12)), acc);
        s = _mm_add_ps(_mm_mul_ps(_mm_loadu_ps(x + p + 8), _mm_loadu_ps(w + p + 8)), s);
        s = _mm_add_ps(_mm_mul_ps(_mm_loadu_ps(x + p + 4), _mm_loadu_ps(w + p + 4)), s);
        acc = _mm_add_ps(_mm_mul_ps(_mm_loadu_ps(x + p), _mm_loadu_ps(w + p)), s);
    }
    for (p = 16 * nb; p < K; p += 4) {
        float a[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
        int q = K - p < 4 ? K - p : 4;
        for (int t = 0; t < q; ++t) { a[t] = x[p + t]; b[t] = w[p + t]; }
        acc = _mm_add_ps(_mm_mul_ps(_mm_loadu_ps(a), _mm_loadu_ps(b)), acc);
    }
    float l[4];
    _mm_storeu_ps(l, acc);
    return (l[0] + l[1]) + (l[2] + l[3]);
}

/* relevance of one pair; returns 0 if the final layer output is non-finite */
static int relevance1(const omodel *m, const float *hu, const float *hv, int d, float *out,
                      float *buf0, float *buf1) {
    memcpy(buf0, hu, sizeof(float) * d);
    memcpy(buf0 + d, hv, sizeof(float) * d);
    float *x = buf0, *y = buf1;
    for (int l = 0; l < m->n_mlp; ++l) {
        int K = m->dims[l], O = m->dims[l + 1];
        const float *W = m->W[l], *b = m->b[l];
        for (int o = 0; o < O; ++o) {
            float v = edot(x, W + (size_t)o * K, K) + b[o];
            if (l < m->n_mlp - 1 && m->relu) v = v > 0.0f ? v : 0.0f; /* np.maximum(v, 0) */
            y[o] = v;
        }
        float *t = x; x = y; y = t;
    }
    int Z = m->dims[m->n_mlp];
    int finite = 1;
    for (int z = 0; z < Z; ++z) finite &= isfinite(x[z]) ? 1 : 0;
    *out = edot(x, m->A, Z);
    return finite;
}

static int max_width(const omodel *m) {
    int w = 0;
    for (int l = 0; l <= m->n_mlp; ++l) if (m->dims[l] > w) w = m->dims[l];
    return w + 16;
}

static void unpack_model(omodel *m, int n_mlp, const int32_t *dims, const float *const *W,
                         const float *const *b, const float *A, int relu) {
    m->n_mlp = n_mlp;
    for (int l = 0; l <= n_mlp; ++l) m->dims[l] = dims[l];
    for (int l = 0; l < n_mlp; ++l) { m->W[l] = W[l]; m->b[l] = b[l]; }
    m->A = A;
    m->relu = relu;
}

int oracle_relevance(int n_mlp, const int32_t *dims, const float *const *W, const float *const *b,
                     const float *A, int relu, const float *hu, int64_t hu_stride,
                     const float *hv, int64_t n, float *out, int nthreads) {
    omodel m;
    unpack_model(&m, n_mlp, dims, W, b, A, relu);
    int d = dims[0] / 2, bad = 0;
    int mw = max_width(&m);
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1) reduction(| : bad)
    {
        float *b0 = malloc(sizeof(float) * mw), *b1 = malloc(sizeof(float) * mw);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            if (!relevance1(&m, hu + i * hu_stride, hv + i * d, d, out + i, b0, b1)) bad |= 1;
        free(b0); free(b1);
    }
    return bad ? 2 : 0;
}

/* ---------------------------------------------------------------- search */

static inline uint32_t f32_orderable(float f) {
    if (f == 0.0f) f = 0.0f; /* canonicalise -0.0: Python compares -0.0 == 0.0 */
    uint32_t u;
    memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
static inline float orderable_f32(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

typedef struct { uint64_t key; int32_t slot; int32_t hop; } oent;

static int cmp_desc(const void *a, const void *b) {
    uint64_t x = ((const oent *)a)->key, y = ((const oent *)b)->key;
    return x < y ? 1 : (x > y ? -1 : 0);
}

typedef struct {
    int n_layers;
    int64_t n;
    const int32_t *nbrs[OMAX_LAYERS];
    int64_t stride[OMAX_LAYERS];
    const int32_t *cnts[OMAX_LAYERS];
    int32_t entry;
    const int64_t *ids;
    const uint32_t *rank; /* tie-break rank of ids[slot] (ascending id) */
} ograph;

typedef struct {
    uint32_t *claimed; /* epoch stamp */
    uint32_t *seen;    /* hop stamp */
    uint32_t epoch, hstamp;
    oent *scored;
    int64_t n_scored, cap_scored;
    int32_t *frontier, *fcount, *foff;      /* per searcher */
    int32_t *fresh, *fresh_cnt, *fresh_off; /* per searcher, concatenated */
    oent *tmp, *seeds;
    float *b0, *b1;
    int64_t cap_fresh;
} owork;

static void push_scored(owork *w, oent e) {
    if (w->n_scored == w->cap_scored) {
        w->cap_scored = w->cap_scored ? 2 * w->cap_scored : 4096;
        w->scored = realloc(w->scored, sizeof(oent) * w->cap_scored);
        w->tmp = realloc(w->tmp, sizeof(oent) * w->cap_scored);
    }
    w->scored[w->n_scored++] = e;
}

/* top-m of scored[] by key into out (sorted desc); returns count */
static int64_t topm(owork *w, int64_t m, oent *out) {
    int64_t n = w->n_scored;
    memcpy(w->tmp, w->scored, sizeof(oent) * n);
    qsort(w->tmp, n, sizeof(oent), cmp_desc);
    if (m > n) m = n;
    memcpy(out, w->tmp, sizeof(oent) * m);
    return m;
}

typedef struct { int k, kp, hops, ef; } oparams;

static void search1(const ograph *g, const omodel *m, const float *items, int d, const float *hu,
                    const oparams *P, owork *w, int64_t *out_ids, double *out_scores,
                    int32_t *out_n, int64_t *stats, int *bad) {
    int top = g->n_layers - 1;
    w->epoch++;
    w->n_scored = 0;
    int64_t evals = 0, per_layer[OMAX_LAYERS] = {0};
    int64_t rows = 0, nbr_ids = 0; /* _neighbors_of calls / ids returned (search.py:135-137) */
    int kp = P->kp, ef = P->ef;

#define SCORE_SLOT(s, hop)                                                                   \
    do {                                                                                     \
        float sc;                                                                            \
        if (!relevance1(m, hu, items + (size_t)g->ids[s] * d, d, &sc, w->b0, w->b1)) *bad = 1; \
        oent e = {((uint64_t)f32_orderable(sc) << 32) | (uint64_t)(~g->rank[s]), (s), (hop)}; \
        push_scored(w, e);                                                                   \
    } while (0)

    /* init: entry + its top-layer neighbourhood (search.py:235-236) */
    {
        int32_t s0 = g->entry;
        w->claimed[s0] = w->epoch;
        SCORE_SLOT(s0, 0);
        const int32_t *row = g->nbrs[top] + (size_t)s0 * g->stride[top];
        rows += 1;
        nbr_ids += g->cnts[top][s0];
        for (int j = 0; j < g->cnts[top][s0]; ++j) {
            int32_t v = row[j];
            if (w->claimed[v] == w->epoch) continue;
            w->claimed[v] = w->epoch;
            SCORE_SLOT(v, 0);
        }
        per_layer[top] += w->n_scored;
    }
    int hop = 0;
    oent *seeds = w->seeds;
    for (int layer = top; layer >= 0; --layer) {
        int64_t ns = topm(w, kp, seeds);
        int nsearch = (int)ns;
        for (int i = 0; i < nsearch; ++i) {
            w->foff[i] = i * ef;
            w->frontier[i * ef] = seeds[i].slot;
            w->fcount[i] = 1;
        }
        const int32_t *nb = g->nbrs[layer], *ct = g->cnts[layer];
        int64_t st = g->stride[layer];
        for (int t = 0; t < P->hops; ++t) {
            hop++;
            w->hstamp++;
            int64_t nf = 0;
            for (int i = 0; i < nsearch; ++i) {
                w->fresh_off[i] = (int32_t)nf;
                for (int f = 0; f < w->fcount[i]; ++f) {
                    int32_t s = w->frontier[w->foff[i] + f];
                    const int32_t *row = nb + (size_t)s * st;
                    rows += 1;
                    nbr_ids += ct[s];
                    for (int j = 0; j < ct[s]; ++j) {
                        int32_t v = row[j];
                        if (w->claimed[v] == w->epoch || w->seen[v] == w->hstamp) continue;
                        w->seen[v] = w->hstamp;
                        w->fresh[nf++] = v;
                    }
                }
                w->fresh_cnt[i] = (int32_t)(nf - w->fresh_off[i]);
            }
            for (int64_t j = 0; j < nf; ++j) w->claimed[w->fresh[j]] = w->epoch;
            per_layer[layer] += nf;
            for (int i = 0; i < nsearch; ++i) {
                int64_t base = w->n_scored;
                for (int j = 0; j < w->fresh_cnt[i]; ++j) SCORE_SLOT(w->fresh[w->fresh_off[i] + j], hop);
                int64_t cnt = w->n_scored - base;
                if (cnt > ef) {
                    memcpy(w->tmp, w->scored + base, sizeof(oent) * cnt);
                    qsort(w->tmp, cnt, sizeof(oent), cmp_desc);
                    for (int j = 0; j < ef; ++j) w->frontier[w->foff[i] + j] = w->tmp[j].slot;
                    w->fcount[i] = ef;
                } else {
                    for (int j = 0; j < cnt; ++j) w->frontier[w->foff[i] + j] = w->scored[base + j].slot;
                    w->fcount[i] = (int32_t)cnt;
                }
            }
        }
    }
    int64_t nr = topm(w, P->k, seeds);
    for (int64_t j = 0; j < nr; ++j) {
        out_ids[j] = g->ids[seeds[j].slot];
        out_scores[j] = (double)orderable_f32((uint32_t)(seeds[j].key >> 32));
    }
    *out_n = (int32_t)nr;
    evals = w->n_scored;
    stats[0] = evals;
    stats[1] = evals;
    stats[2] = nr ? seeds[0].hop : -1;
    stats[3] = rows;
    stats[4] = nbr_ids;
    for (int l = 0; l < g->n_layers; ++l) stats[5 + l] = per_layer[l];
#undef SCORE_SLOT
}

/*
 * Batched search, one query per OpenMP task.  Output layout:
 *   out_ids[Q, k] int64, out_scores[Q, k] f64, out_n[Q],
 *   stats[Q, 5 + n_layers] = evals, nodes_visited, hops_to_best, rows expanded,
 *   neighbour ids read, per-layer evals.
 * Returns 0, or 2 if any final-layer metric output was non-finite.
 */
int oracle_search(int n_layers, int64_t n, const int32_t *const *nbrs, const int64_t *stride,
                  const int32_t *const *cnts, int32_t entry, const int64_t *ids,
                  const uint32_t *rank, int n_mlp, const int32_t *dims, const float *const *W,
                  const float *const *b, const float *A, int relu, const float *items, int d,
                  const float *users, int64_t Q, int k, int kp, int hops, int ef, int nthreads,
                  int64_t *out_ids, double *out_scores, int32_t *out_n, int64_t *stats) {
    if (n_layers < 1 || n_layers > OMAX_LAYERS || n_mlp < 1 || n_mlp > OMAX_MLP) return 1;
    ograph g;
    g.n_layers = n_layers;
    g.n = n;
    for (int l = 0; l < n_layers; ++l) { g.nbrs[l] = nbrs[l]; g.stride[l] = stride[l]; g.cnts[l] = cnts[l]; }
    g.entry = entry;
    g.ids = ids;
    g.rank = rank;
    omodel m;
    unpack_model(&m, n_mlp, dims, W, b, A, relu);
    oparams P = {k, kp, hops, ef};
    int maxdeg = 0;
    for (int l = 0; l < n_layers; ++l) if (stride[l] > maxdeg) maxdeg = (int)stride[l];
    int64_t cap_fresh = (int64_t)kp * ef * maxdeg;
    if (cap_fresh > n) cap_fresh = n;
    cap_fresh += 64;
    int bad = 0;
    int nst = 5 + n_layers;
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1) reduction(| : bad)
    {
        owork w;
        memset(&w, 0, sizeof(w));
        w.claimed = calloc(n, sizeof(uint32_t));
        w.seen = calloc(n, sizeof(uint32_t));
        w.cap_fresh = cap_fresh;
        w.frontier = malloc(sizeof(int32_t) * (size_t)kp * ef);
        w.fcount = malloc(sizeof(int32_t) * kp);
        w.foff = malloc(sizeof(int32_t) * kp);
        w.fresh = malloc(sizeof(int32_t) * cap_fresh);
        w.fresh_cnt = malloc(sizeof(int32_t) * kp);
        w.fresh_off = malloc(sizeof(int32_t) * kp);
        w.b0 = malloc(sizeof(float) * max_width(&m));
        w.b1 = malloc(sizeof(float) * max_width(&m));
        w.seeds = malloc(sizeof(oent) * (size_t)(k + kp + 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t q = 0; q < Q; ++q) {
            int mybad = 0;
            search1(&g, &m, items, d, users + (size_t)q * d, &P, &w, out_ids + q * k,
                    out_scores + q * k, out_n + q, stats + q * nst, &mybad);
            bad |= mybad;
        }
        free(w.claimed); free(w.seen); free(w.frontier); free(w.fcount); free(w.foff);
        free(w.fresh); free(w.fresh_cnt); free(w.fresh_off); free(w.b0); free(w.b1);
        free(w.scored); free(w.tmp); free(w.seeds);
    }
    return bad ? 2 : 0;
}

int oracle_num_threads(void) { return omp_get_max_threads(); }
