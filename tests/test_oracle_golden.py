"""Pin the CPU oracle against the reference's own outputs (tests/golden/*).

CPU-only.  The oracle (oracle/hipanns_oracle.py and the C restatement
oracle/c/oracle.c) must reproduce ``relevance_batch`` bit-for-bit and
``c_hipanns`` item ids, scores and evaluation counts exactly.
"""

import numpy as np
import pytest

import golden_io as G
from oracle import hipanns_oracle as O


def test_einsum_emulation_matches_numpy_all_widths():
    rng = np.random.default_rng(0)
    for K in list(range(1, 40)) + [64, 127, 128, 256]:
        x = rng.normal(size=(9, K)).astype(np.float32)
        w = rng.normal(size=(3, K)).astype(np.float32)
        ref = np.einsum("ij,kj->ik", x, w, optimize=False)
        np.testing.assert_array_equal(O.einsum_rows_f32(x, w).view(np.uint32), ref.view(np.uint32))


def test_sqnorm_emulation_matches_numpy():
    rng = np.random.default_rng(1)
    for K in range(1, 40):
        d = rng.normal(size=(5, K))
        np.testing.assert_array_equal(O.sqnorm_rows_f64(d), np.einsum("ij,ij->i", d, d))


@pytest.mark.parametrize("case", list(G.load("scorer")["cases"]))
def test_relevance_bit_exact_vs_reference(case):
    z = G.load("scorer")
    layers, att, relu = G.model_layers(z, prefix=f"{case}/")
    model = O.OracleModel(layers, att, relu)
    got, finite = O.relevance_f32(model, z[f"{case}/hu"], z[f"{case}/hv"])
    assert finite
    exp = z[f"{case}/expect"]
    assert got.dtype == exp.dtype == np.float32
    np.testing.assert_array_equal(got.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("fixture", G.SEARCH_FIXTURES)
def test_hopsync_traversal_matches_reference(fixture):
    z = G.load(fixture)
    graph = O.OracleGraph(G.graph_layers(z), int(z["entry_slot"]), z["ids"])
    layers, att, relu = G.model_layers(z)
    model = O.OracleModel(layers, att, relu)
    emb, users, ids = z["emb"], z["users"], z["ids"]
    for pi, p in G.param_sets(z):
        exp = G.expected(z, pi)
        for q in range(len(users)):
            def score(slots, q=q):
                s, _ = O.relevance_f32(model, users[q], emb[ids[slots]])
                return s.astype(np.float64)
            r = O.c_hipanns(graph, score, **p)
            n = int(exp["n"][q])
            assert [i for i, _ in r["items"]] == list(exp["ids"][q, :n])
            assert [s for _, s in r["items"]] == list(exp["scores"][q, :n])
            assert r["evals"] == exp["evals"][q]
            assert r["per_layer"] == list(exp["per_layer"][q])
            assert r["hops_to_best"] == exp["best_hop"][q]


def test_euclid_traversal_matches_reference():
    z = G.load("euclid")
    graph = O.OracleGraph(G.graph_layers(z), int(z["entry_slot"]), z["ids"])
    vectors, queries = z["vectors"], z["queries"]
    for pi, p in G.param_sets(z):
        exp = G.expected(z, pi)
        for q in range(len(queries)):
            r = O.c_hipanns(graph, lambda s, q=q: O.neg_euclid_f64(vectors, queries[q], s), **p)
            n = int(exp["n"][q])
            assert [i for i, _ in r["items"]] == list(exp["ids"][q, :n])
            assert [s for _, s in r["items"]] == list(exp["scores"][q, :n])
            assert r["evals"] == exp["evals"][q]
            assert r["per_layer"] == list(exp["per_layer"][q])


# ---------------------------------------------------------------- C oracle

from oracle import oracle_c as OC  # noqa: E402


@pytest.mark.parametrize("case", list(G.load("scorer")["cases"]))
def test_c_oracle_relevance_bit_exact(case):
    z = G.load("scorer")
    layers, att, relu = G.model_layers(z, prefix=f"{case}/")
    got, finite = OC.relevance(layers, att, relu, z[f"{case}/hu"], z[f"{case}/hv"], nthreads=2)
    assert finite
    np.testing.assert_array_equal(got.view(np.uint32), z[f"{case}/expect"].view(np.uint32))


@pytest.mark.parametrize("fixture", G.SEARCH_FIXTURES)
def test_c_oracle_search_matches_reference(fixture):
    z = G.load(fixture)
    layers, att, relu = G.model_layers(z)
    for pi, p in G.param_sets(z):
        exp = G.expected(z, pi)
        r = OC.search(G.graph_layers(z), int(z["entry_slot"]), z["ids"], layers, att, relu,
                      z["emb"], z["users"], p["k"], p["k_parallel"], p["hops"], p["ef"],
                      nthreads=4)
        np.testing.assert_array_equal(r["n"], exp["n"])
        np.testing.assert_array_equal(r["ids"], exp["ids"])
        np.testing.assert_array_equal(r["scores"], exp["scores"])
        np.testing.assert_array_equal(r["evals"], exp["evals"])
        np.testing.assert_array_equal(r["visited"], exp["visited"])
        np.testing.assert_array_equal(r["best_hop"], exp["best_hop"])
        np.testing.assert_array_equal(r["per_layer"], exp["per_layer"])
        np.testing.assert_array_equal(r["rows"], exp["rows"])
        np.testing.assert_array_equal(r["nbr_ids"], exp["nbr_ids"])


@pytest.mark.parametrize("case", G.ref_cases())
def test_oracle_reproduces_reference_search_tests(case):
    """The reference's own test_search.py cases (make_reftests.py): the numpy oracle's
    euclidean scorer + hop-synchronous c_hipanns give the reference's items and counts."""
    c = G.ref_case(case)
    graph = O.OracleGraph(c.layers, c.entry, c.ids)
    for pi, p in c.params():
        exp = c.expected(pi)
        for q in range(len(c.queries)):
            r = O.c_hipanns(graph, lambda s, q=q: O.neg_euclid_f64(c.vectors, c.queries[q], s), **p)
            n = int(exp["n"][q])
            assert [i for i, _ in r["items"]] == list(exp["ids"][q, :n])
            assert [s for _, s in r["items"]] == list(exp["scores"][q, :n])
            assert r["evals"] == exp["evals"][q]
            assert r["per_layer"] == list(exp["per_layer"][q])
            assert r["hops_to_best"] == exp["best_hop"][q]
