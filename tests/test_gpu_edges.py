"""Edge cases of the device search, checked against the C oracle (oracle/c, pinned to the
reference by test_oracle_golden.py): tiny / disconnected / single-node graphs, k larger
than the reachable set (-1 / NaN padding, count < k), an empty batch, hub nodes listed by
every frontier row (lowest-searcher claims), and both scorer modes on the multi-query
kernel (BASELINE model family) and the per-query kernel (generic model shape)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2502_11490_b200 as P
    from paper_2502_11490_b200 import _lib

    if _lib.lib().gr_device_count() < 1:
        pytest.fail("no CUDA device visible for a -m gpu test")
    return P


def random_graph(rng, n, deg, n_layers=2, p_up=0.2, isolate=()):
    """Symmetric random graph with an upper layer; nodes in `isolate` get no edges."""
    levels = np.zeros(n, dtype=np.int32)
    if n_layers > 1:
        levels[rng.random(n) < p_up] = 1
    for l in range(2, n_layers):
        levels[(levels == l - 1) & (rng.random(n) < 0.3)] = l
    entry = int(np.flatnonzero(levels == levels.max())[0])
    layers = []
    for l in range(n_layers):
        members = np.flatnonzero(levels >= l)
        cap = 2 * deg if l == 0 else deg
        nb = np.full((n, cap), -1, dtype=np.int32)
        ct = np.zeros(n, dtype=np.int32)
        adj = {int(v): set() for v in members}
        for v in members:
            if int(v) in isolate:
                continue
            for u in rng.choice(members, size=min(deg, len(members)), replace=False):
                u = int(u)
                if u == v or u in isolate or len(adj[v]) >= cap or len(adj[u]) >= cap:
                    continue
                adj[int(v)].add(u)
                adj[u].add(int(v))
        for v, s in adj.items():
            s = sorted(s)[:cap]
            nb[v, :len(s)] = s
            ct[v] = len(s)
        layers.append((nb, ct))
    return levels, layers, entry


def check(P, rng, n, deg, d, z, users_n, params, mode, isolate=(), hidden=(64, 64), n_layers=2):
    from oracle import oracle_c as OC

    model = P.create_model(d_x=d, d_h=d, z_dim=z, hidden=hidden, seed=3)
    emb = model.item_embeddings(rng.normal(size=(n, d)).astype(np.float32)).astype(np.float32)
    users = model.user_embedding(rng.normal(size=(users_n, d)).astype(np.float32)).astype(np.float32)
    levels, layers, entry = random_graph(rng, n, deg, n_layers=n_layers, isolate=isolate)
    ids = np.arange(n, dtype=np.int64)
    index = P.GraphIndex.from_arrays(ids, levels, layers, entry, m=deg)
    r = P.c_hipanns_batch(index, model, users, emb, P.SearchParams(**params, mode=mode))
    m = model.metric
    o = OC.search(layers, entry, ids, m.layers, m.attention, m.activation == "relu", emb, users,
                  params["k"], params["k_parallel"], params["hops"], params["ef"], nthreads=4)
    np.testing.assert_array_equal(r.count, o["n"])
    np.testing.assert_array_equal(r.ids, o["ids"])
    np.testing.assert_array_equal(r.scores, o["scores"])
    np.testing.assert_array_equal(r.evals, o["evals"])
    np.testing.assert_array_equal(r.per_layer, o["per_layer"])
    np.testing.assert_array_equal(r.hops_to_best, o["best_hop"])
    return r


@pytest.mark.parametrize("mode", ["exact", "tc"])
def test_k_larger_than_reachable_set_is_padded(P, mode):
    rng = np.random.default_rng(1)
    # 40 nodes, 12 of them isolated: at most 28 reachable, k = 64
    r = check(P, rng, 40, 4, 64, 2, 6, dict(k=64, k_parallel=4, hops=6, ef=16), mode,
              isolate=set(range(28, 40)))
    assert (r.count <= 28).all()
    for q in range(len(r.count)):
        c = int(r.count[q])
        assert (r.ids[q, c:] == -1).all() and np.isnan(r.scores[q, c:]).all()


@pytest.mark.parametrize("mode", ["exact", "tc"])
def test_single_node_graph(P, mode):
    rng = np.random.default_rng(2)
    r = check(P, rng, 1, 2, 128, 3, 3, dict(k=5, k_parallel=1, hops=2, ef=4), mode, n_layers=1)
    assert (r.count == 1).all() and (r.ids[:, 0] == 0).all() and (r.evals == 1).all()


@pytest.mark.parametrize("mode", ["exact", "tc"])
def test_hub_graph_lowest_searcher_claims(P, mode):
    """Dense small graph: every node is listed by many frontier rows of many searchers."""
    rng = np.random.default_rng(3)
    check(P, rng, 300, 24, 128, 3, 40, dict(k=100, k_parallel=32, hops=4, ef=64), mode)


@pytest.mark.parametrize("mode", ["exact", "tc"])
def test_many_queries_many_layers(P, mode):
    rng = np.random.default_rng(4)
    check(P, rng, 3000, 8, 64, 3, 700, dict(k=20, k_parallel=8, hops=3, ef=40), mode, n_layers=3)


def test_generic_model_shape_uses_per_query_kernel(P):
    """d_h = 20, one hidden layer: no fixed-shape kernel, the per-query kernel runs."""
    rng = np.random.default_rng(5)
    check(P, rng, 500, 6, 20, 2, 16, dict(k=10, k_parallel=4, hops=3, ef=20), "exact",
          hidden=(16,))


def test_empty_batch(P):
    rng = np.random.default_rng(6)
    d = 64
    model = P.create_model(d_x=d, d_h=d, z_dim=2, hidden=(64, 64), seed=3)
    emb = model.item_embeddings(rng.normal(size=(50, d)).astype(np.float32)).astype(np.float32)
    levels, layers, entry = random_graph(rng, 50, 4)
    index = P.GraphIndex.from_arrays(np.arange(50), levels, layers, entry, m=4)
    r = P.c_hipanns_batch(index, model, np.zeros((0, d), np.float32), emb, P.SearchParams(k=5))
    assert r.ids.shape == (0, 5) and r.count.shape == (0,)
