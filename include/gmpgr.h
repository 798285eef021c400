/*
 * gmpgr.h — C ABI of the B200-native GMP-GR HiPANNS retrieval hot path.
 *
 * libgmpgr.so (paper_2502_11490_b200/csrc, built for sm_100a) exports exactly the
 * functions below.  Plain pointers and sizes only; no torch types.  Every entry
 * point returns GR_OK (0) or an error code; gr_last_error() gives the message
 * (thread-local).  The Python package maps codes to the reference's exception
 * classes (errors.py:8-59): GR_EINVAL -> InvalidArgumentError,
 * GR_ENUMERIC -> NumericError, GR_ECUDA/GR_ENOMEM -> RuntimeError/MemoryError.
 *
 * Reference interfaces each entry point replaces (file:line under
 * /root/reference/pkg/src/nann/):
 *   gr_model_create   <- MetricModel / RelevanceModel weights (metric.py:74-99, 192-226),
 *                        NANN-MODEL payload order (metric.py:310-399)
 *   gr_graph_create   <- GraphIndex.graph_view() (index.py:384-391), NANN-IDX (index.py:397-508)
 *   gr_items_create   <- model_scorer's item_embeddings (search.py:84-90)
 *   gr_score_pairs    <- ScoreFn (search.py:27) / RelevanceModel.score (metric.py:222-226) /
 *                        BatchEngine.evaluate (batching.py:67-109) / relevance_batch (metric.py:150-154)
 *   gr_search         <- c_hipanns(index, model_scorer(model, h_u, emb), SearchParams)
 *                        (search.py:194-286, 30-70), batched over Q user embeddings
 *   gr_brute_force    <- brute_force(model_scorer(...), ids, k) (search.py:93-108)
 *   gr_merge_topk     <- CandidatePool(k).push(...) over several result lists (pool.py:11-55)
 *   gr_scores_euclid  <- euclidean_scorer(query, item_vectors) (search.py:73-81), Q queries
 *   gr_scores_create  <- an arbitrary ScoreFn (search.py:27) tabulated as fp64 [Q, n_items]
 *   gr_search_scores  <- c_hipanns(index, <that ScoreFn>, SearchParams) (search.py:194-286)
 *
 * Pointer arguments documented "host-or-device" follow the `on_device` flag of
 * the call: 0 = host memory (the library copies in/out on `stream` and
 * synchronises), 1 = device memory on the handle's device (asynchronous on
 * `stream` except where a status must be read back; see each call).
 */
#ifndef GMPGR_H
#define GMPGR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    GR_OK = 0,
    GR_EINVAL = 1,   /* bad argument / contract violation */
    GR_ENUMERIC = 2, /* non-finite metric output (metric.py:134-135) */
    GR_ECUDA = 3,    /* CUDA runtime failure */
    GR_ENOMEM = 4,   /* device allocation failure */
    GR_EBAND = 5     /* tensor-core mode: an approximate score missed its exact value by more
                        than half the refinement band (async calls; gr_search re-runs exact) */
};

#define GR_ABI_VERSION 1

typedef struct gr_model gr_model;
typedef struct gr_graph gr_graph;
typedef struct gr_items gr_items;
typedef struct gr_searcher gr_searcher;
typedef struct gr_scores gr_scores;

/* Search knobs = SearchParams (search.py:30-49); ef is frontier_width (ef or 2k).
 * mode: GR_MODE_EXACT (every claim scored by the exact-fp32 CUDA-core scorer) or
 * GR_MODE_TC (tcgen05 split-bf16 scores; every item within band_rel*|T| + band_abs of a
 * selection threshold T is re-scored exactly, so ids, order and returned scores are the
 * exact ones whenever |approx - exact| < band/2).  band_* <= 0 selects the defaults. */
typedef struct {
    int32_t k;
    int32_t k_parallel;
    int32_t hops;
    int32_t ef;
    int32_t mode;
    float band_rel;
    float band_abs;
} gr_search_params;

enum { GR_MODE_EXACT = 0, GR_MODE_TC = 1 };

const char *gr_last_error(void);
int gr_abi_version(void);
/* number of CUDA devices visible (0 without a GPU; never fails) */
int gr_device_count(void);

/* Metric MLP.  n_mlp layers; dims[0] = 2*d_h (pair width), dims[m+1] = output width of
 * layer m, dims[n_mlp] = z_dim.  W[m]: host fp32 row-major [dims[m+1], dims[m]] (the
 * reference's (d_out, d_in) layout); b[m]: [dims[m+1]]; attention: [z_dim]; relu: 1 for
 * "relu" (ReLU between layers, never after the last), 0 for "identity".  fp16 models are
 * passed widened to fp32 (exact). */
int gr_model_create(int device, int n_mlp, const int32_t *dims, const float *const *W,
                    const float *const *b, const float *attention, int relu, gr_model **out);
int gr_model_destroy(gr_model *m);

/* Layered graph over n slots.  For layer l < n_layers: nbrs[l] host int32 rows of
 * row_stride[l] entries (the first cnts[l][s] of row s are neighbour SLOTS; the reference's
 * fixed-width _nbrs[l] arrays, index.py:78-79); levels host int32 [n] (node level, index.py:77);
 * entry_slot (index.py:68); ids host int64 [n] (item id per slot: output ids and the
 * (score desc, id asc) tie-break); rows host int32 [n] or NULL: embedding row per slot
 * (NULL -> rows = ids, the model_scorer convention search.py:88). */
int gr_graph_create(int device, int n_layers, int64_t n, const int32_t *const *nbrs,
                    const int64_t *row_stride, const int32_t *const *cnts, const int32_t *levels,
                    int32_t entry_slot, const int64_t *ids, const int32_t *rows, gr_graph **out);
/* Same, with the device slot order chosen by the caller: order int64 [n] lists the caller
 * slots in device-slot order (a permutation; NULL = the default breadth-first order from the
 * entry).  Device slot order is invisible to results (ids and the id-rank tie-break are
 * carried per slot); it sets the memory locality of the per-query visited state, the
 * adjacency rows and the slot-ordered embedding copy (e.g. cluster-contiguous orders). */
int gr_graph_create_ordered(int device, int n_layers, int64_t n, const int32_t *const *nbrs,
                            const int64_t *row_stride, const int32_t *const *cnts,
                            const int32_t *levels, int32_t entry_slot, const int64_t *ids,
                            const int32_t *rows, const int64_t *order, gr_graph **out);
int gr_graph_destroy(gr_graph *g);

/* Item embeddings fp32 [n, d] row-major (host or device pointer per emb_on_device). */
int gr_items_create(int device, const float *emb, int64_t n, int32_t d, int emb_on_device,
                    gr_items **out);
int gr_items_destroy(gr_items *it);

/* Relevance of n (user, item) pairs (relevance_batch bit-exact).  users fp32 [n_users, d_h];
 * user_index int32 [n] (NULL -> every pair uses users[0], the model_scorer broadcast);
 * item_ids int64 [n] (rows of the items handle); out fp64 [n].  host-or-device pointers.
 * Synchronous; returns GR_ENUMERIC if any final-layer output is non-finite. */
int gr_score_pairs(const gr_model *m, const gr_items *it, const float *users, int64_t n_users,
                   const int32_t *user_index, const int64_t *item_ids, int64_t n,
                   double *out_scores, int on_device, void *stream);

/* First-pass tensor-core (split-bf16 tcgen05) scores of one user (host fp32 [d_h]) against
 * item rows (host int64 [n]) -> host fp64 [n].  Diagnostic for the tc mode's refinement band:
 * compare with gr_score_pairs.  GR_EINVAL if the model has no tensor-core shape. */
int gr_score_items_approx(const gr_model *m, const gr_items *it, const float *user,
                          const int64_t *item_ids, int64_t n, double *out_scores);

/* Scratch owner for gr_search (visited state, frontiers, pools).  Calls on one searcher are
 * serialised (a mutex covers staging, scratch growth, launch and read-back; launches on
 * different streams are ordered by an event), so host threads may share it. */
int gr_searcher_create(int device, gr_searcher **out);
int gr_searcher_destroy(gr_searcher *s);

/* Batched C-HiPANNS, deterministic lock-step semantics; results identical to the exact fp32
 * scorer in both modes (see gr_search_params.mode).
 * users fp32 [Q, d_h].  Outputs: ids int64 [Q, k] (-1 padded), scores fp64 [Q, k],
 * count int32 [Q], stats int64 [Q, 5 + n_layers] = (metric_evaluations, nodes_visited,
 * hops_to_best or -1, adjacency rows expanded, neighbour ids read, per-layer evaluations
 * base layer first).  host-or-device pointers.
 * Synchronous (reads back the numeric flag); GR_ENUMERIC on a non-finite metric output. */
int gr_search(gr_searcher *s, const gr_graph *g, const gr_model *m, const gr_items *it,
              const float *users, int64_t Q, const gr_search_params *p, int64_t *out_ids,
              double *out_scores, int32_t *out_count, int64_t *out_stats, int on_device,
              void *stream);

/* Same as gr_search but asynchronous on `stream` with device pointers only; the numeric
 * flag and the tensor-core band certificate are accumulated in the searcher and returned
 * by gr_searcher_status (GR_ENUMERIC / GR_EBAND).  gr_search itself checks the
 * certificate and, if any approximate score missed its exact value by more than half the
 * band, searches the batch again in exact mode before returning. */
int gr_search_async(gr_searcher *s, const gr_graph *g, const gr_model *m, const gr_items *it,
                    const float *users, int64_t Q, const gr_search_params *p, int64_t *out_ids,
                    double *out_scores, int32_t *out_count, int64_t *out_stats, void *stream);
/* Synchronise `stream`, return GR_ENUMERIC if any async search saw a non-finite output
 * since the last call, GR_EBAND if a tensor-core band violation was seen (flags cleared),
 * else GR_OK. */
int gr_searcher_status(gr_searcher *s, void *stream);
/* kernel launches issued by this searcher so far (evidence counter for bench.py) */
int64_t gr_searcher_launches(const gr_searcher *s);
/* cumulative scoring counters of this searcher: out[0] = exact re-scores (tensor-core
 * mode), out[1] = tensor-core scores; when the searcher was created with
 * GMPGR_PHASE_TIMING=1 in the environment, out[2..9] = summed SM cycles per search phase
 * (init, seeds, expand, resolve, score, pool, frontier, output) and out[10..17] = cycles
 * of the duo kernel's tensor-core stage roles (epilogue layer-0 / layer-1 work, layer-0 /
 * layer-1 waits, epilogue total, issuer idle / issuing, loader stage waits); out[18] = band violations seen (exact re-scores whose approximate score was
 * farther than band/2 from the exact one), out[19] = largest |approx - exact| / band seen,
 * as f32 bits, out[20] = batches gr_search re-ran in exact mode, out[21] = resident search
 * units (CTA halves of 8 queries) of the last duo-kernel launch.  out must hold 22 values.
 * Synchronises the device. */
int gr_searcher_counters(gr_searcher *s, int64_t *out);

/* Exact top-k over ALL items of the handle for Q users (ground truth, search.py:93-108):
 * ids int64 [Q, k] (= item rows), scores fp64 [Q, k].  host-or-device pointers. */
int gr_brute_force(const gr_model *m, const gr_items *it, const float *users, int64_t Q,
                   int32_t k, int64_t *out_ids, double *out_scores, int on_device, void *stream);

/* Merge R per-shard top-k lists per query into one top-k by (score desc, id asc)
 * (CandidatePool.push of every entry, pool.py:30-55).  in_ids/in_scores [R, Q, k_in]
 * (-1 ids are empty slots), out [Q, k].  Device pointers, asynchronous. */
int gr_merge_topk(int device, const int64_t *in_ids, const double *in_scores, int32_t R,
                  int64_t Q, int32_t k_in, int32_t k, int64_t *out_ids, double *out_scores,
                  int32_t *out_count, void *stream);
/* Shard-merge wire format, 8 bytes per entry (one all-gather instead of id + score
 * gathers): gr_pack_topk packs n (id, score) entries as orderable(fp32 score) << 32 | id
 * (requires 0 <= id < 2^32; id -1 -> 0 = empty); gr_merge_topk_packed merges R packed
 * lists [R, Q, k_in] like gr_merge_topk.  Device pointers, asynchronous. */
int gr_pack_topk(int device, const int64_t *ids, const double *scores, int64_t n, uint64_t *out,
                 void *stream);
int gr_merge_topk_packed(int device, const uint64_t *in, int32_t R, int64_t Q, int32_t k_in,
                         int32_t k, int64_t *out_ids, double *out_scores, int32_t *out_count,
                         void *stream);

/* Traversal-only scorers (the reference's search tests: search.py:73-81 euclidean_scorer and
 * ad-hoc ScoreFns).  A score table holds fp64 scores [Q, n_items] indexed by ITEM ID (ids are
 * score-table columns, like euclidean_scorer's `item_vectors[ids]`, search.py:79).
 * gr_scores_create: host-or-device fp64 table.  GR_ENUMERIC if any score is NaN.
 * gr_scores_euclid: host fp64 vectors [n_items, dim] and queries [Q, dim]; computes
 *   -sqrt(einsum('ij,ij->i', v - q, v - q)) on the device in numpy's fp64 order (bit-exact).
 * gr_scores_read: copy the fp64 table to host memory [Q, n_items]. */
int gr_scores_create(int device, const double *table, int64_t Q, int64_t n_items, int on_device,
                     gr_scores **out);
int gr_scores_euclid(int device, const double *vectors, int64_t n_items, int32_t dim,
                     const double *queries, int64_t Q, gr_scores **out);
int gr_scores_read(const gr_scores *t, double *out);
int gr_scores_destroy(gr_scores *t);

/* Batched C-HiPANNS driven by a score table (query q of the batch = row q of the table):
 * same semantics, outputs and stats as gr_search (exact mode only); returned scores are the
 * table's fp64 values.  Every graph item id must be < n_items (GR_EINVAL otherwise).
 * host-or-device output pointers; synchronous for host outputs. */
int gr_search_scores(gr_searcher *s, const gr_graph *g, const gr_scores *t,
                     const gr_search_params *p, int64_t *out_ids, double *out_scores,
                     int32_t *out_count, int64_t *out_stats, int on_device, void *stream);

/* Sequential index construction, node-for-node identical to the reference's
 * GraphIndex.insert (index.py:283-319: layer descent with ef=1, ef_construction beam
 * search per layer (_chot.pyx:116-179), keep-M or heuristic _select (index.py:226-239),
 * symmetric _connect with capacity re-selection (index.py:250-281)).  Host code (no GPU).
 * Inserts slots [n0, n1) in order; the caller has stored vectors fp64 [cap][dim],
 * ids int64 [cap] and levels int32 [cap] (drawn from the reference's level stream,
 * index.py:196-209) for those slots.  nbrs[l]: int32 [cap][2m (l == 0) or m], cnts[l]:
 * int32 [cap] for l < max_layers (the reference's _nbrs/_cnts arrays, index.py:78-79),
 * stamps int64 [cap] (index.py:80), *stamp the last used stamp, *entry_slot / *top_level
 * (-1 when empty) are updated in place. */
#define GR_MAX_GRAPH_LAYERS 8
int gr_hnsw_insert(int64_t n0, int64_t n1, int32_t dim, const double *vectors, const int64_t *ids,
                   const int32_t *levels, int32_t m, int32_t ef_construction, int32_t max_layers,
                   int select_heuristic, int32_t *const *nbrs, int32_t *const *cnts,
                   int64_t *stamps, int64_t *stamp, int32_t *entry_slot, int32_t *top_level);

#ifdef __cplusplus
}
#endif

#endif /* GMPGR_H */
