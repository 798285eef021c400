"""GPU parity: libgmpgr.so (via the C ABI) vs the reference's recorded outputs and the oracle.

Bar (north_star): identical item ids, bit-identical fp32 scores (exact mode; the
1e-5 fp32 tolerance is therefore met with 0 error), identical evaluation counts.
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


def metric_of(P, z, prefix=""):
    layers, att, relu = G.model_layers(z, prefix=prefix)
    return P.MetricModel(list(layers), att, activation="relu" if relu else "identity")


def index_of(P, z):
    return P.GraphIndex.from_arrays(z["ids"], z["levels"], G.graph_layers(z), int(z["entry_slot"]),
                                    m=int(z["m"]))


@pytest.mark.parametrize("case", list(G.load("scorer")["cases"]))
def test_score_pairs_bit_exact(P, case):
    z = G.load("scorer")
    metric = metric_of(P, z, prefix=f"{case}/")
    got = P.relevance_batch(metric, z[f"{case}/hu"], z[f"{case}/hv"])
    exp = z[f"{case}/expect"]
    np.testing.assert_array_equal(got.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("case", list(G.load("scorer")["cases"]))
def test_batch_engine_bitwise_equals_direct(P, case):
    # test_batching.py:147-168: engine scores == direct relevance for the same pairs
    z = G.load("scorer")
    metric = metric_of(P, z, prefix=f"{case}/")
    hv = z[f"{case}/hv"]
    eng = P.GpuBatchEngine(metric, hv, batch_size=64)
    ids = np.arange(len(hv))[::-1].copy()
    got = eng.evaluate(z[f"{case}/hu"][ids], ids)
    exp = z[f"{case}/expect"][ids].astype(np.float64)
    np.testing.assert_array_equal(got, exp)
    assert eng.invocations == 1


@pytest.mark.parametrize("fixture", G.SEARCH_FIXTURES)
def test_search_matches_reference(P, fixture):
    z = G.load(fixture)
    metric = metric_of(P, z)
    index = index_of(P, z)
    for pi, p in G.param_sets(z):
        params = P.SearchParams(**p)
        r = P.c_hipanns_batch(index, metric, z["users"], z["emb"], params)
        exp = G.expected(z, pi)
        np.testing.assert_array_equal(r.count, exp["n"])
        np.testing.assert_array_equal(r.ids, exp["ids"])
        np.testing.assert_array_equal(r.scores, exp["scores"])
        np.testing.assert_array_equal(r.evals, exp["evals"])
        np.testing.assert_array_equal(r.per_layer, exp["per_layer"])
        np.testing.assert_array_equal(r.hops_to_best, exp["best_hop"])
        np.testing.assert_array_equal(r.rows_expanded, exp["rows"])
        np.testing.assert_array_equal(r.nbr_ids_read, exp["nbr_ids"])


def test_per_query_api_matches_reference(P):
    z = G.load("search_d64_z2")
    metric = metric_of(P, z)
    model = P.RelevanceModel(None, None, metric)
    index = index_of(P, z)
    pi, p = G.param_sets(z)[0]
    exp = G.expected(z, pi)
    for q in range(3):
        res = P.c_hipanns(index, P.model_scorer(model, z["users"][q], z["emb"]), P.SearchParams(**p))
        n = int(exp["n"][q])
        assert res.item_ids() == list(exp["ids"][q, :n])
        assert [s for _, s in res.items] == list(exp["scores"][q, :n])
        assert res.stats.metric_evaluations == exp["evals"][q]
        assert res.stats.nodes_visited == exp["visited"][q]
        assert res.stats.per_layer_evaluations == list(exp["per_layer"][q])


def test_scorer_callable_matches_reference_scores(P):
    z = G.load("search_d128_z3")
    metric = metric_of(P, z)
    fn = P.model_scorer(P.RelevanceModel(None, None, metric), z["users"][0], z["emb"])
    ids = np.array([5, 0, 17, 1999, 5], dtype=np.int64)
    from oracle import hipanns_oracle as O

    layers, att, relu = G.model_layers(z)
    exp, _ = O.relevance_f32(O.OracleModel(layers, att, relu), z["users"][0], z["emb"][ids])
    np.testing.assert_array_equal(fn(ids), exp.astype(np.float64))


def test_brute_force_matches_reference_ground_truth(P):
    z = G.load("search_d64_z2")
    metric = metric_of(P, z)
    gt = z["gt100"]
    ids, scores = P.brute_force_batch(metric, z["users"][: len(gt)], z["emb"], 100)
    np.testing.assert_array_equal(ids, gt)
    res = P.brute_force(P.model_scorer(P.RelevanceModel(None, None, metric), z["users"][0], z["emb"]),
                        np.arange(len(z["emb"])), 100)
    assert res.item_ids() == list(gt[0])


def test_merge_topk_equals_candidate_pool(P):
    import torch
    from paper_2502_11490_b200 import _lib

    rng = np.random.default_rng(0)
    R, Q, kin, k = 4, 9, 20, 25
    ids = rng.permutation(R * Q * kin).reshape(R, Q, kin).astype(np.int64)
    scores = rng.integers(0, 40, size=(R, Q, kin)).astype(np.float32).astype(np.float64)
    ids[1, 2, 5:] = -1  # ragged shard list
    ti, ts = torch.from_numpy(ids).cuda(), torch.from_numpy(scores).cuda()
    oi = torch.empty((Q, k), dtype=torch.int64, device="cuda")
    os_ = torch.empty((Q, k), dtype=torch.float64, device="cuda")
    oc = torch.empty(Q, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().gr_merge_topk(0, ti.data_ptr(), ts.data_ptr(), R, Q, kin, k,
                                        oi.data_ptr(), os_.data_ptr(), oc.data_ptr(), None))
    torch.cuda.synchronize()
    for q in range(Q):
        pool = P.CandidatePool(k)
        for r in range(R):
            for j in range(kin):
                if ids[r, q, j] >= 0:
                    pool.push(int(ids[r, q, j]), float(scores[r, q, j]))
        top = pool.top(k)
        assert int(oc[q]) == len(top)
        assert oi[q, : len(top)].cpu().tolist() == [i for i, _ in top]
        assert os_[q, : len(top)].cpu().tolist() == [s for _, s in top]


def test_nonfinite_raises_numeric_error(P):
    # test_metric.py:104-108
    m = P.create_model(d_x=4, d_h=3, z_dim=2, hidden=(6,), seed=1)
    m.metric.layers[0][0][:] = 1e38
    with pytest.raises(P.NumericError):
        P.relevance_batch(m.metric, np.full((1, 3), 1e5, np.float32), np.ones((1, 3), np.float32))


def test_invalid_arguments(P):
    z = G.load("search_d64_z2")
    metric = metric_of(P, z)
    index = index_of(P, z)
    with pytest.raises(P.InvalidArgumentError):
        P.c_hipanns(index, lambda ids: np.zeros(len(ids)), P.SearchParams(k=10))
    with pytest.raises(P.InvalidArgumentError):
        P.c_hipanns_batch(index, metric, z["users"][:, :10], z["emb"], P.SearchParams(k=10))
    bad = P.GpuBatchEngine(metric, z["emb"])
    with pytest.raises(P.InvalidArgumentError):
        bad.evaluate(z["users"][:2], np.array([0, len(z["emb"]) + 5]))


def test_large_generated_graph_matches_c_oracle(P):
    """50k items x 128-d, Z=3, GPU-built graph (m=16): GPU search == C oracle bitwise."""
    from oracle import oracle_c

    rng = np.random.default_rng(11)
    n, d = 50_000, 128
    model = P.create_model(d_x=d, d_h=d, z_dim=3, hidden=(64, 64), seed=1)
    centers = rng.normal(scale=4.0, size=(256, d))
    feats = (centers[rng.integers(0, 256, size=n)] + rng.normal(size=(n, d))).astype(np.float32)
    emb = model.item_embeddings(feats).astype(np.float32)
    index = P.GraphIndex.build(emb, m=16, seed=0)
    index.validate()
    users = model.user_embedding(rng.normal(size=(96, d)).astype(np.float32)).astype(np.float32)
    layers, att = model.metric.layers, model.metric.attention
    ids_v, lv, glayers, entry = index.graph_view()
    for kw in (dict(k=100, k_parallel=8, hops=3, ef=200), dict(k=32, k_parallel=32, hops=6, ef=48)):
        r = P.c_hipanns_batch(index, model, users, emb, P.SearchParams(**kw))
        o = oracle_c.search(glayers, entry, ids_v, layers, att, True, emb, users, **kw, nthreads=8)
        np.testing.assert_array_equal(r.ids, o["ids"])
        np.testing.assert_array_equal(r.scores, o["scores"])
        np.testing.assert_array_equal(r.evals, o["evals"])
        np.testing.assert_array_equal(r.rows_expanded, o["rows"])
        np.testing.assert_array_equal(r.nbr_ids_read, o["nbr_ids"])
        np.testing.assert_array_equal(r.per_layer, o["per_layer"])


@pytest.mark.parametrize("fixture", ["search_d64_z2", "search_d128_z3"])
def test_tensor_core_mode_matches_reference(P, fixture):
    """tcgen05 split-bf16 scoring + exact band refinement: same ids/scores/counts as exact."""
    z = G.load(fixture)
    metric = metric_of(P, z)
    index = index_of(P, z)
    for pi, p in G.param_sets(z):
        r = P.c_hipanns_batch(index, metric, z["users"], z["emb"], P.SearchParams(**p, mode="tc"))
        exp = G.expected(z, pi)
        np.testing.assert_array_equal(r.ids, exp["ids"])
        np.testing.assert_array_equal(r.scores, exp["scores"])
        np.testing.assert_array_equal(r.evals, exp["evals"])
        np.testing.assert_array_equal(r.per_layer, exp["per_layer"])
        np.testing.assert_array_equal(r.hops_to_best, exp["best_hop"])


def test_tensor_core_mode_large_graph_equals_exact(P):
    from paper_2502_11490_b200 import _lib

    rng = np.random.default_rng(12)
    n, d = 60_000, 128
    model = P.create_model(d_x=d, d_h=d, z_dim=3, hidden=(64, 64), seed=1)
    centers = rng.normal(scale=4.0, size=(256, d))
    feats = (centers[rng.integers(0, 256, size=n)] + rng.normal(size=(n, d))).astype(np.float32)
    emb = model.item_embeddings(feats).astype(np.float32)
    index = P.GraphIndex.build(emb, m=16, seed=0)
    users = model.user_embedding(rng.normal(size=(200, d)).astype(np.float32)).astype(np.float32)
    s = _lib.DeviceSearcher(0)
    for kw in (dict(k=100, k_parallel=8, hops=3, ef=200), dict(k=50, k_parallel=16, hops=5, ef=40)):
        ex = P.c_hipanns_batch(index, model, users, emb, P.SearchParams(**kw))
        tc = P.c_hipanns_batch(index, model, users, emb, P.SearchParams(**kw, mode="tc"), searcher=s)
        np.testing.assert_array_equal(tc.ids, ex.ids)
        np.testing.assert_array_equal(tc.scores, ex.scores)
        np.testing.assert_array_equal(tc.evals, ex.evals)
        np.testing.assert_array_equal(tc.hops_to_best, ex.hops_to_best)
    c = s.counters()
    assert c["tensor_scored"] > 0
    assert c["exact_rescored"] < 0.5 * c["tensor_scored"], c


def test_tc_first_pass_error_far_inside_refinement_band(P):
    """The tc mode is exact only if |approx - exact| < band/2 (band = 1e-3*|T| + 1e-3).
    Measure the split-bf16 tcgen05 first pass against the exact scorer on 1M pairs of the
    BASELINE model family (d_h 128, Z 3) and require a >= 10x margin."""
    import ctypes
    from paper_2502_11490_b200 import _lib

    rng = np.random.default_rng(21)
    n, d = 250_000, 128
    model = P.create_model(d_x=d, d_h=d, z_dim=3, hidden=(64, 64), seed=1)
    centers = rng.normal(scale=4.0, size=(1024, d))
    feats = (centers[rng.integers(0, 1024, size=n)] + rng.normal(size=(n, d))).astype(np.float32)
    emb = np.ascontiguousarray(model.item_embeddings(feats), dtype=np.float32)
    users = model.user_embedding(rng.normal(size=(4, d)).astype(np.float32)).astype(np.float32)
    dm = model.metric.device_model(0)
    it = _lib.DeviceItems(emb, 0)
    ids = np.arange(n, dtype=np.int64)
    worst = 0.0
    for u in users:
        u = np.ascontiguousarray(u)
        approx = np.empty(n)
        _lib.check(_lib.lib().gr_score_items_approx(dm.h, it.h, _lib.ptr(u), _lib.ptr(ids), n,
                                                    _lib.ptr(approx)))
        exact = np.empty(n)
        _lib.check(_lib.lib().gr_score_pairs(dm.h, it.h, _lib.ptr(u), 1, None, _lib.ptr(ids), n,
                                             _lib.ptr(exact), 0, None))
        band = 1e-3 * np.abs(exact) + 1e-3
        worst = max(worst, float(np.max(np.abs(approx - exact) / band)))
    print(f"max |approx-exact| / band = {worst:.3e}")
    assert worst < 0.05


@pytest.mark.parametrize("fixture", ["search_d64_z2", "search_d128_z3"])
def test_tensor_core_mode_large_batch_matches_reference(P, fixture):
    """Batches that fill every SM twice run 16 queries per CTA (launch_mq): the reference's
    recorded results must come back for every copy of every query."""
    z = G.load(fixture)
    metric = metric_of(P, z)
    index = index_of(P, z)
    nq = len(z["users"])
    reps = -(-5000 // nq)
    users = np.tile(z["users"], (reps, 1))
    pi, p = G.param_sets(z)[0]
    r = P.c_hipanns_batch(index, metric, users, z["emb"], P.SearchParams(**p, mode="tc"))
    exp = G.expected(z, pi)
    for rep in range(reps):
        sl = slice(rep * nq, (rep + 1) * nq)
        np.testing.assert_array_equal(r.ids[sl], exp["ids"])
        np.testing.assert_array_equal(r.scores[sl], exp["scores"])
        np.testing.assert_array_equal(r.evals[sl], exp["evals"])
        np.testing.assert_array_equal(r.hops_to_best[sl], exp["best_hop"])


def test_tensor_core_head_overflow_guard_path(P):
    """Head weights scaled so the epilogue's largest relu output often exceeds its no-overflow
    limit: those rows take the per-head path (non-finite check per head) instead of the
    collapsed dot product -- results still equal exact mode, and nothing is flagged."""
    rng = np.random.default_rng(13)
    n, d = 20_000, 128
    model = P.create_model(d_x=d, d_h=d, z_dim=3, hidden=(64, 64), seed=1)
    w2, b2 = model.metric.layers[-1]
    w2 *= np.float32(1e35)  # |z| ~ 1e36: finite, but h_max above the guard's limit (~15)
    centers = rng.normal(scale=4.0, size=(128, d))
    feats = (centers[rng.integers(0, 128, size=n)] + rng.normal(size=(n, d))).astype(np.float32)
    emb = model.item_embeddings(feats).astype(np.float32)
    index = P.GraphIndex.build(emb, m=16, seed=0)
    users = model.user_embedding(rng.normal(size=(64, d)).astype(np.float32)).astype(np.float32)
    kw = dict(k=100, k_parallel=8, hops=3, ef=200)
    ex = P.c_hipanns_batch(index, model, users, emb, P.SearchParams(**kw))
    tc = P.c_hipanns_batch(index, model, users, emb, P.SearchParams(**kw, mode="tc"))
    assert np.all(np.isfinite(ex.scores[ex.ids >= 0]))
    assert np.abs(ex.scores[ex.ids >= 0]).max() > 1e30
    np.testing.assert_array_equal(tc.ids, ex.ids)
    np.testing.assert_array_equal(tc.scores, ex.scores)
    np.testing.assert_array_equal(tc.evals, ex.evals)
