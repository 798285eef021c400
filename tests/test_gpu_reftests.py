"""The reference's own search tests (test_search.py TestCHipanns / TestBruteForce) on the GPU.

Each case re-creates a reference test's inputs (recorded by tests/golden/make_reftests.py
from the reference package: same helpers, seeds and reference-built graphs) and runs
``c_hipanns(index, euclidean_scorer(q, vectors), params)`` through the device traversal
(score-table mode: gr_scores_euclid + gr_search_scores).  Every case asserts the
reference test's own property AND identity with what the reference returned: ids,
fp64 scores (bit-exact: numpy's einsum order is reproduced on the device), evaluation
counts, per-layer counts and hops_to_best.
"""

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2502_11490_b200 as P
    from paper_2502_11490_b200 import _lib

    if _lib.lib().gr_device_count() < 1:
        pytest.fail("no CUDA device visible for a -m gpu test")
    return P


def index_of(P, c):
    return P.GraphIndex.from_arrays(c.ids, c.levels, c.layers, c.entry, m=c.m)


def run(P, c, q, params):
    return P.c_hipanns(index_of(P, c), P.euclidean_scorer(c.queries[q], c.vectors),
                       P.SearchParams(**params))


def assert_same_as_reference(c, pi, q, got):
    exp = c.expected(pi)
    n = int(exp["n"][q])
    assert got.item_ids() == list(exp["ids"][q, :n])
    assert [s for _, s in got.items] == list(exp["scores"][q, :n])  # bit-exact fp64
    assert got.stats.metric_evaluations == exp["evals"][q]
    assert got.stats.nodes_visited == exp["evals"][q]
    assert got.stats.per_layer_evaluations == list(exp["per_layer"][q])
    hb = int(exp["best_hop"][q])
    assert got.stats.hops_to_best == (None if hb < 0 else hb)


@pytest.mark.parametrize("case", G.ref_cases())
def test_every_recorded_case_identical(P, case):
    c = G.ref_case(case)
    for pi, p in c.params():
        for q in range(len(c.queries)):
            assert_same_as_reference(c, pi, q, run(P, c, q, p))


def test_batched_scores_table_equals_single_queries(P):
    c = G.ref_case("desk")
    (pi, p), = c.params()
    r = P.c_hipanns_scores_batch(index_of(P, c),
                                 P._lib.DeviceScores(vectors=c.vectors, queries=c.queries),
                                 P.SearchParams(**p))
    exp = c.expected(pi)
    assert np.array_equal(r.ids, exp["ids"])
    assert np.array_equal(r.scores, exp["scores"])
    assert np.array_equal(r.evals, exp["evals"])


def test_path_graph_matches_greedy_with_equivalent_budget(P):
    c = G.ref_case("path")  # test_search.py:146-152
    (pi, p), = c.params()
    assert run(P, c, 0, p).item_ids() == [9, 8]


def test_complete_base_layer_equals_brute_force(P):
    c = G.ref_case("complete")  # test_search.py:154-163
    (pi, p), = c.params()
    n = len(c.ids)
    fn = P.euclidean_scorer(c.queries[0], c.vectors)
    exact = P.brute_force(fn, np.arange(n), n)
    got = run(P, c, 0, p)
    assert got.items == exact.items


def test_never_scores_an_item_twice(P):
    c = G.ref_case("never_twice")  # test_search.py:165-171
    (pi, p), = c.params()
    got = run(P, c, 0, p)
    assert got.stats.nodes_visited == got.stats.metric_evaluations
    assert got.stats.metric_evaluations == c.expected(pi)["evals"][0]  # = reference's scorer calls


def test_visited_grows_with_k_parallel(P):
    wins = 0  # test_search.py:173-184
    for seed in range(20):
        c = G.ref_case(f"visited{seed}")
        (_, p1), (_, p4) = c.params()
        v1 = run(P, c, 0, p1).stats.nodes_visited
        v4 = run(P, c, 0, p4).stats.nodes_visited
        wins += v4 >= v1
    assert wins == 20


def test_recall_monotone_in_hops_and_parallel_in_expectation(P):
    rec = {0: [], 1: [], 2: []}  # (kp, hops) = (1,1), (1,3), (4,3); test_search.py:186-199
    for seed in range(20):
        c = G.ref_case(f"recall{seed}")
        gt = set(c.bf_ids[0].tolist())
        for pi, p in c.params():
            got = run(P, c, 0, p)
            rec[pi].append(len(set(got.item_ids()) & gt) / 10)
    assert np.mean(rec[1]) >= np.mean(rec[0])
    assert np.mean(rec[2]) >= np.mean(rec[1])


def test_desk_scale_recall_floor_smoke(P):
    c = G.ref_case("desk")  # test_search.py:201-212
    (pi, p), = c.params()
    recs = []
    for q in range(len(c.queries)):
        got = run(P, c, q, p)
        recs.append(len(set(got.item_ids()) & set(c.bf_ids[q].tolist())) / 10)
    assert np.mean(recs) >= 0.9


def test_deterministic_mode_reproducible(P):
    c = G.ref_case("deterministic")  # test_search.py:214-226
    (pi, p), = c.params()
    runs = [P.c_hipanns(index_of(P, c), P.euclidean_scorer(c.queries[0], c.vectors),
                        P.SearchParams(**p, deterministic=True, n_threads=t)) for t in (None, 1, 8)]
    assert runs[0].items == runs[1].items == runs[2].items


def test_reported_scores_are_true_scores(P):
    c = G.ref_case("deterministic")  # pool contract, test_search.py:228-241
    (pi, p), = c.params()
    fn = P.euclidean_scorer(c.queries[0], c.vectors)
    got = P.c_hipanns(index_of(P, c), fn, P.SearchParams(**p, deterministic=False, n_threads=4))
    scores = [s for _, s in got.items]
    assert scores == sorted(scores, reverse=True)
    for item, score in got.items:
        assert fn(np.array([item]))[0] == score


def test_result_strictly_descending_with_id_ties(P):
    c = G.ref_case("ties")  # test_search.py:243-249
    (pi, p), = c.params()
    got = run(P, c, 0, p)
    keys = [(-s, i) for i, s in got.items]
    assert keys == sorted(keys)


def test_brute_force_line_and_ties(P):
    z = G.load("reftests")  # test_search.py:66-78
    line = z["bf_line/vectors"]
    assert P.brute_force(P.euclidean_scorer(np.array([2.2]), line), np.arange(10), 2).item_ids() == [2, 3]
    ties = z["bf_ties/vectors"]
    assert P.brute_force(P.euclidean_scorer(np.array([0.0]), ties), np.arange(3), 2).item_ids() == [0, 1]


def test_euclid_table_bit_exact(P):
    for name in ("desk", "ties", "complete"):
        c = G.ref_case(name)
        t = P._lib.DeviceScores(vectors=c.vectors, queries=c.queries).read()
        for q in range(len(c.queries)):
            # brute force of the reference: fp64 scores of its top items
            assert list(t[q][c.bf_ids[q]]) == list(c.bf_scores[q])


def test_table_scorer_and_errors(P):
    c = G.ref_case("ties")
    (pi, p), = c.params()
    fn = P.euclidean_scorer(c.queries[0], c.vectors)
    table = fn(np.arange(len(c.vectors)))
    got = P.c_hipanns(index_of(P, c), P.table_scorer(table), P.SearchParams(**p))
    assert_same_as_reference(c, pi, 0, got)
    with pytest.raises(P.NumericError):
        P.c_hipanns(index_of(P, c), P.table_scorer(np.full(len(c.vectors), np.nan)),
                    P.SearchParams(**p))
    with pytest.raises(P.InvalidArgumentError):  # ids outside the table
        P.c_hipanns(index_of(P, c), P.table_scorer(table[:10]), P.SearchParams(**p))
    with pytest.raises(P.InvalidArgumentError):  # arbitrary callables have no device path
        P.c_hipanns(index_of(P, c), lambda ids: np.zeros(len(ids)), P.SearchParams(**p))
