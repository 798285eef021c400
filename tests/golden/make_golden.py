"""Generate golden vectors by running the REFERENCE ``nann`` package.

Run in the build container (the reference is not on the GPU box):

    REF_SRC=/root/reference/pkg/src python tests/golden/make_golden.py

``REF_SRC`` may point at a writable copy with the Cython kernel built
(``python setup.py build_ext --inplace``) — that only speeds up
``GraphIndex.build``; search and scoring never call it (search.py:12-25).

Every output is produced by the reference's own public API:
``create_model`` / ``relevance_batch`` (metric.py:150-154, 229-267),
``GraphIndex.build`` / ``graph_view`` / ``save`` (index.py:160-194, 384-429),
``c_hipanns`` with ``model_scorer`` or ``euclidean_scorer`` (search.py:73-90, 194-286),
``brute_force`` (search.py:93-108), ``save_model`` / ``quantize`` (metric.py:280-341).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = os.environ.get("REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)

import nann  # noqa: E402
from nann import (  # noqa: E402
    GraphIndex,
    SearchParams,
    brute_force,
    c_hipanns,
    create_model,
    euclidean_scorer,
    model_scorer,
    quantize,
    save_model,
)
from nann.bench import clustered_vectors  # noqa: E402
from nann.metric import relevance_batch  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def graph_arrays(index: GraphIndex) -> dict:
    ids, levels, layers, entry = index.graph_view()
    n = len(index)
    out = {"ids": np.asarray(ids[:n]), "levels": np.asarray(levels[:n]),
           "entry_slot": np.int64(entry), "n_layers": np.int64(len(layers)),
           "m": np.int64(index.m)}
    for l, (nb, ct) in enumerate(layers):
        out[f"nbrs{l}"] = np.ascontiguousarray(nb[:n])
        out[f"cnts{l}"] = np.ascontiguousarray(ct[:n])
    return out


def model_arrays(model, prefix="") -> dict:
    out = {}
    for m, (w, b) in enumerate(model.metric.layers):
        out[f"{prefix}W{m}"] = w
        out[f"{prefix}b{m}"] = b
    out[f"{prefix}A"] = model.metric.attention
    out[f"{prefix}n_mlp"] = np.int64(len(model.metric.layers))
    out[f"{prefix}relu"] = np.int64(model.metric.activation == "relu")
    return out


class WorkCounter:
    """Counts _neighbors_of calls / ids per query (SURVEY.md Appendix A count_work.py)."""

    def __init__(self):
        import nann.search as S
        self.S = S
        self.orig = S._neighbors_of
        self.rows = 0
        self.ids = 0

        def wrapped(layers, layer, slot):
            out = self.orig(layers, layer, slot)
            self.rows += 1
            self.ids += len(out)
            return out

        S._neighbors_of = wrapped

    def take(self):
        r = (self.rows, self.ids)
        self.rows = self.ids = 0
        return r


COUNTER = None


def run_counted(fn):
    """Run one c_hipanns call; returns (result, rows_expanded, neighbour_ids_read)."""
    COUNTER.take()
    r = fn()
    rows, ids = COUNTER.take()
    return r, rows, ids


def result_arrays(results, k) -> dict:
    Q = len(results)
    ids = np.full((Q, k), -1, dtype=np.int64)
    scores = np.full((Q, k), np.nan)
    n_items = np.zeros(Q, dtype=np.int64)
    evals = np.zeros(Q, dtype=np.int64)
    visited = np.zeros(Q, dtype=np.int64)
    best_hop = np.full(Q, -1, dtype=np.int64)
    per_layer = []
    rows = np.zeros(Q, dtype=np.int64)
    nbr = np.zeros(Q, dtype=np.int64)
    for q, (r, nr, ni) in enumerate(results):
        rows[q] = nr
        nbr[q] = ni
        n_items[q] = len(r.items)
        for j, (i, s) in enumerate(r.items):
            ids[q, j] = i
            scores[q, j] = s
        evals[q] = r.stats.metric_evaluations
        visited[q] = r.stats.nodes_visited
        best_hop[q] = -1 if r.stats.hops_to_best is None else r.stats.hops_to_best
        per_layer.append(r.stats.per_layer_evaluations)
    return {"res_ids": ids, "res_scores": scores, "res_n": n_items, "res_evals": evals,
            "res_visited": visited, "res_best_hop": best_hop, "res_rows": rows, "res_nbr_ids": nbr,
            "res_per_layer": np.asarray(per_layer, dtype=np.int64)}


def scorer_fixture():
    """relevance_batch at every config shape (+ odd d_h, fp16, identity, 1-layer)."""
    cases = [
        ("d6_z3_h16x16", dict(d_x=8, d_h=6, z_dim=3, hidden=(16, 16), seed=5)),
        ("d32_z2_h64x64", dict(d_x=32, d_h=32, z_dim=2, hidden=(64, 64), seed=1)),
        ("d64_z2_h64x64", dict(d_x=64, d_h=64, z_dim=2, hidden=(64, 64), seed=1)),
        ("d128_z3_h64x64", dict(d_x=128, d_h=128, z_dim=3, hidden=(64, 64), seed=1)),
        ("d128_z3_h64x64_fp16", dict(d_x=128, d_h=128, z_dim=3, hidden=(64, 64), seed=2)),
        ("d20_z5_h40_identity", dict(d_x=8, d_h=20, z_dim=5, hidden=(40,), seed=3,
                                      activation="identity")),
        ("d16_z1_h24x8x12", dict(d_x=8, d_h=16, z_dim=1, hidden=(24, 8, 12), seed=4)),
    ]
    out = {"cases": np.array([c for c, _ in cases])}
    rng = np.random.default_rng(99)
    for name, kw in cases:
        model = create_model(**kw)
        if name.endswith("fp16"):
            model = quantize(model)
        n = 301
        d_h = kw["d_h"]
        hu = (rng.normal(size=(n, d_h)) * 2).astype(np.float32)
        hv = (rng.normal(size=(n, d_h)) * 2).astype(np.float32)
        # a shared-user block too (the search path broadcasts one h_u)
        hu[200:] = hu[200]
        out.update(model_arrays(model, prefix=f"{name}/"))
        out[f"{name}/hu"] = hu
        out[f"{name}/hv"] = hv
        out[f"{name}/expect"] = relevance_batch(model.metric, hu, hv)
    np.savez_compressed(os.path.join(OUT, "scorer.npz"), **out)
    # reference-written model files for the NANN-MODEL loader
    m32 = create_model(d_x=5, d_h=4, z_dim=3, hidden=(8, 6), seed=11)
    save_model(m32, os.path.join(OUT, "model_fp32.nann"))
    save_model(quantize(m32), os.path.join(OUT, "model_fp16.nann"))


PARAMS = [
    dict(k=100, k_parallel=8, hops=3),            # reference defaults (evalharness.py:84-87)
    dict(k=10, k_parallel=2, hops=6, ef=8),
    dict(k=50, k_parallel=16, hops=4, ef=32),
    dict(k=20, k_parallel=20, hops=2, ef=3),
]


def search_fixture(name, n, d, z, m, n_clusters, n_queries, params, shuffle_ids=False,
                   heuristic=False, hidden=(64, 64)):
    model = create_model(d_x=d, d_h=d, z_dim=z, hidden=hidden, seed=1)
    feats = clustered_vectors(n, d, n_clusters, seed=0).astype(np.float32)
    emb = model.item_embeddings(feats)  # (n, d) fp32, row = item id
    if shuffle_ids:
        perm = np.random.default_rng(5).permutation(n).astype(np.int64)
        index = GraphIndex.build(emb[perm].astype(np.float64), ids=perm, m=m,
                                 ef_construction=2 * m, seed=0, select_heuristic=heuristic)
    else:
        index = GraphIndex.build(emb.astype(np.float64), m=m, ef_construction=2 * m, seed=0,
                                 select_heuristic=heuristic)
    index.validate()
    users = model.user_embedding(
        np.random.default_rng(7).normal(size=(n_queries, d)).astype(np.float32))
    out = {"emb": emb, "users": users}
    out.update(graph_arrays(index))
    out.update(model_arrays(model))
    for pi, p in enumerate(params):
        sp = SearchParams(**p)
        res = [run_counted(lambda q=q: c_hipanns(index, model_scorer(model, users[q], emb), sp))
               for q in range(n_queries)]
        for key, val in result_arrays(res, sp.k).items():
            out[f"p{pi}/{key}"] = val
        out[f"p{pi}/params"] = np.array([sp.k, sp.k_parallel, sp.hops, sp.frontier_width])
    # brute-force ground truth (recall oracle) for the first few queries
    gt = []
    for q in range(min(n_queries, 8)):
        r = brute_force(model_scorer(model, users[q], emb), np.arange(n), 100)
        gt.append(r.item_ids())
    out["gt100"] = np.asarray(gt, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(name, "layers", index.layer_node_counts(),
          "evals p0", out["p0/res_evals"][:4])


def euclid_fixture():
    n, d = 1200, 12
    rng = np.random.default_rng(3)
    centers = rng.normal(scale=4.0, size=(8, d))
    vectors = centers[rng.integers(0, 8, size=n)] + rng.normal(size=(n, d))
    index = GraphIndex.build(vectors, m=6, ef_construction=24, seed=3)
    index.save(os.path.join(OUT, "euclid_index.nann"))
    queries = vectors[rng.integers(0, n, size=16)] + 0.1 * rng.normal(size=(16, d))
    out = {"vectors": vectors, "queries": queries}
    out.update(graph_arrays(index))
    for pi, p in enumerate(PARAMS[1:] + [dict(k=10, k_parallel=4, hops=3)]):
        sp = SearchParams(**p)
        res = [run_counted(lambda q=q: c_hipanns(index, euclidean_scorer(queries[q], vectors), sp))
               for q in range(16)]
        for key, val in result_arrays(res, sp.k).items():
            out[f"p{pi}/{key}"] = val
        out[f"p{pi}/params"] = np.array([sp.k, sp.k_parallel, sp.hops, sp.frontier_width])
    np.savez_compressed(os.path.join(OUT, "euclid.npz"), **out)


def main():
    global COUNTER
    print("reference nann", nann.__version__, "from", nann.__file__)
    COUNTER = WorkCounter()
    scorer_fixture()
    euclid_fixture()
    search_fixture("search_d64_z2", n=3000, d=64, z=2, m=8, n_clusters=32, n_queries=24,
                   params=PARAMS)
    search_fixture("search_d128_z3", n=2000, d=128, z=3, m=16, n_clusters=64, n_queries=16,
                   params=PARAMS[:3])
    search_fixture("search_d32_shuffled", n=1500, d=32, z=3, m=6, n_clusters=16, n_queries=16,
                   params=PARAMS, shuffle_ids=True, heuristic=True, hidden=(48, 32))


if __name__ == "__main__":
    main()
