"""Golden vectors for the reference's own search tests, run on the REFERENCE ``nann``.

    python tests/golden/make_reftests.py        (build container only)

Re-creates the inputs of ``/root/reference/pkg/tests/test_search.py`` (TestCHipanns and
the brute-force cases: the ``clustered`` / ``line_index`` helpers, the same seeds, graphs
built by the reference ``GraphIndex.build``) and records what the reference returns for
``c_hipanns(index, euclidean_scorer(q, vectors), params)`` and ``brute_force`` — ids,
fp64 scores and evaluation counts — into ``tests/golden/reftests.npz``.  The GPU tests
(tests/test_gpu_reftests.py) replay each case through the device traversal
(score-table mode, gr_search_scores) and assert both the reference test's own property
and identity with these recorded results.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = os.environ.get("REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)

from nann import GraphIndex, SearchParams, brute_force, c_hipanns, euclidean_scorer  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def clustered(n, d, seed, n_clusters=8):  # test_search.py:17-20
    rng = np.random.default_rng(seed)
    centers = rng.normal(scale=4.0, size=(n_clusters, d))
    return centers[rng.integers(0, n_clusters, size=n)] + rng.normal(size=(n, d))


def line_index(n=10):  # test_search.py:33-53 (hand-wired path graph)
    vectors = np.array([[float(i)] for i in range(n)])
    index = GraphIndex(dim=1, m=2, ef_construction=4, max_layers=1, seed=0)
    index._reserve(n)
    index._n = n
    for i in range(n):
        index._vectors[i] = vectors[i]
        index._ids[i] = i
        index._levels[i] = 0
        index._slot_of[i] = i
    index._entry_slot = 0
    index._top_level = 0
    nbrs, cnts = index._nbrs[0], index._cnts[0]
    for i in range(n - 1):
        nbrs[i, cnts[i]] = i + 1
        cnts[i] += 1
        nbrs[i + 1, cnts[i + 1]] = i
        cnts[i + 1] += 1
    index.validate()
    return index, vectors


OUTD: dict = {}


def record(case: str, index, vectors, queries, params):
    ids, levels, layers, entry = index.graph_view()
    n = len(index)
    p = f"{case}/"
    OUTD[p + "vectors"] = np.asarray(vectors, dtype=np.float64)
    OUTD[p + "queries"] = np.asarray(queries, dtype=np.float64)
    OUTD[p + "ids"] = np.asarray(ids[:n])
    OUTD[p + "levels"] = np.asarray(levels[:n])
    OUTD[p + "entry_slot"] = np.int64(entry)
    OUTD[p + "n_layers"] = np.int64(len(layers))
    OUTD[p + "m"] = np.int64(index.m)
    for l, (nb, ct) in enumerate(layers):
        OUTD[p + f"nbrs{l}"] = np.ascontiguousarray(nb[:n])
        OUTD[p + f"cnts{l}"] = np.ascontiguousarray(ct[:n])
    for pi, kw in enumerate(params):
        sp = SearchParams(**kw)
        res = [c_hipanns(index, euclidean_scorer(q, vectors), sp) for q in queries]
        k = sp.k
        rid = np.full((len(res), k), -1, dtype=np.int64)
        rsc = np.full((len(res), k), np.nan)
        for qi, r in enumerate(res):
            for j, (i, s) in enumerate(r.items):
                rid[qi, j] = i
                rsc[qi, j] = s
        pp = f"{p}p{pi}/"
        OUTD[pp + "params"] = np.array([sp.k, sp.k_parallel, sp.hops, sp.frontier_width])
        OUTD[pp + "ids"] = rid
        OUTD[pp + "scores"] = rsc
        OUTD[pp + "n"] = np.array([len(r.items) for r in res])
        OUTD[pp + "evals"] = np.array([r.stats.metric_evaluations for r in res])
        OUTD[pp + "per_layer"] = np.array([r.stats.per_layer_evaluations for r in res])
        OUTD[pp + "best_hop"] = np.array([-1 if r.stats.hops_to_best is None else r.stats.hops_to_best
                                          for r in res])
    # brute-force ground truth over all items (search.py:93-108), k = min(n, 10)
    kb = min(n, 10)
    gt = [brute_force(euclidean_scorer(q, vectors), np.arange(n), kb) for q in queries]
    OUTD[p + "bf_ids"] = np.array([g.item_ids() for g in gt])
    OUTD[p + "bf_scores"] = np.array([[s for _, s in g.items] for g in gt])


def main():
    # test_path_graph_matches_greedy_with_equivalent_budget (test_search.py:146-152)
    index, vectors = line_index(10)
    record("path", index, vectors, np.array([[8.7]]), [dict(k=2, k_parallel=1, hops=9, ef=2)])
    # test_complete_base_layer_equals_brute_force (:154-163)
    n = 40
    vectors = clustered(n, 5, seed=13)
    index = GraphIndex.build(vectors, m=n, ef_construction=n, seed=13)
    record("complete", index, vectors, (vectors[0] + 0.3)[None, :],
           [dict(k=n, k_parallel=n, hops=1)])
    # test_never_scores_an_item_twice (:165-171)
    vectors = clustered(300, 6, seed=14)
    index = GraphIndex.build(vectors, m=8, ef_construction=32, seed=14)
    record("never_twice", index, vectors, (vectors[5] + 0.1)[None, :],
           [dict(k=10, k_parallel=4, hops=3)])
    # test_visited_grows_with_k_parallel (:173-184): 20 graphs
    for seed in range(20):
        vectors = clustered(300, 6, seed=seed + 50)
        index = GraphIndex.build(vectors, m=8, ef_construction=32, seed=seed)
        record(f"visited{seed}", index, vectors, np.zeros((1, 6)),
               [dict(k=8, k_parallel=1, hops=3), dict(k=8, k_parallel=4, hops=3)])
    # test_recall_monotone_in_hops_and_parallel_in_expectation (:186-199): 20 graphs
    for seed in range(20):
        vectors = clustered(400, 6, seed=seed + 80)
        index = GraphIndex.build(vectors, m=8, ef_construction=32, seed=seed)
        rng = np.random.default_rng(seed)
        q = vectors[rng.integers(0, 400)] + 0.2
        record(f"recall{seed}", index, vectors, q[None, :],
               [dict(k=10, k_parallel=kp, hops=h, ef=10) for kp, h in ((1, 1), (1, 3), (4, 3))])
    # test_desk_scale_recall_floor_smoke (:201-212)
    vectors = clustered(500, 8, seed=21, n_clusters=10)
    index = GraphIndex.build(vectors, m=16, ef_construction=64, seed=21)
    rng = np.random.default_rng(22)
    qs = np.array([vectors[rng.integers(0, 500)] + 0.1 * rng.normal(size=8) for _ in range(20)])
    record("desk", index, vectors, qs, [dict(k=10, k_parallel=8, hops=3, ef=20)])
    # test_deterministic_mode_reproducible (:214-226)
    vectors = clustered(250, 6, seed=23)
    index = GraphIndex.build(vectors, m=8, ef_construction=32, seed=23)
    record("deterministic", index, vectors, (vectors[17] + 0.05)[None, :],
           [dict(k=10, k_parallel=4, hops=3)])
    # test_result_strictly_descending_with_id_ties (:243-249)
    vectors = clustered(100, 4, seed=25)
    index = GraphIndex.build(vectors, m=6, ef_construction=24, seed=25)
    record("ties", index, vectors, vectors[0][None, :], [dict(k=10, k_parallel=2, hops=3)])
    # brute force: 1-D line query 2.2 -> [2, 3]; equal scores -> lower id first (:66-78)
    OUTD["bf_line/vectors"] = np.array([[float(i)] for i in range(10)])
    OUTD["bf_ties/vectors"] = np.array([[1.0], [-1.0], [3.0]])
    np.savez_compressed(os.path.join(OUT, "reftests.npz"), **OUTD)
    print("cases:", sorted({k.split("/")[0] for k in OUTD}))


if __name__ == "__main__":
    main()
