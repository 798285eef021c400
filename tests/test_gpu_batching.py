"""Q-HiPANNS with the device engine: Dispatcher/BatchQueue driving GpuBatchEngine
(= ModelBatchEngine), scores bit-identical to evaluating each request alone and to the
oracle's restatement of relevance_batch (reference test_batching.py:147-168, 290-312)."""

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


def oracle_scores(P, model, users, items):
    from oracle import hipanns_oracle as O

    om = O.OracleModel.from_metric(getattr(model, "metric", model))
    s, _ = O.relevance_f32(om, users, items)
    return s.astype(np.float64)


def test_engine_batched_bitwise_equal_direct_and_oracle(P):
    rng = np.random.default_rng(1)
    model = P.create_model(d_x=6, d_h=4, z_dim=2, hidden=(8,), seed=0)
    emb = model.item_embeddings(rng.normal(size=(500, 6)).astype(np.float32))
    eng = P.ModelBatchEngine(model, emb, batch_size=32)
    q = P.BatchQueue(capacity=32, flush_timeout_s=0.002)
    d = P.Dispatcher(q, eng).start()
    reqs = []
    for _ in range(60):
        n = int(rng.integers(1, 20))
        users = np.repeat(rng.normal(size=(1, 4)).astype(np.float32), n, axis=0)
        reqs.append(P.EvalRequest(users=users, item_ids=rng.integers(0, 500, size=n)))
    got = [h.wait(20.0) for h in [q.submit(r) for r in reqs]]
    d.stop()
    direct = P.ModelBatchEngine(model, emb, batch_size=32)
    for r, g in zip(reqs, got):
        np.testing.assert_array_equal(g, direct.evaluate(r.users, r.item_ids))
        np.testing.assert_array_equal(g, oracle_scores(P, model, r.users, emb[r.item_ids]))
    assert eng.invocations < len(reqs)  # aggregation happened


def test_pipeline_mode_with_device_engine(P):
    z = G.load("search_d128_z3")
    layers, att, relu = G.model_layers(z)
    metric = P.MetricModel(list(layers), att, activation="relu" if relu else "identity")
    emb, users = z["emb"], z["users"]
    rng = np.random.default_rng(7)
    eng = P.GpuBatchEngine(metric, emb, batch_size=256)
    q = P.BatchQueue(capacity=256, flush_timeout_s=0.002)
    d = P.run_dispatcher(q, eng, pipeline=True)
    reqs = []
    for i in range(200):
        n = int(rng.integers(1, 64))
        u = np.broadcast_to(users[i % len(users)], (n, users.shape[1]))
        reqs.append(P.EvalRequest(users=u, item_ids=rng.integers(0, len(emb), size=n)))
    got = [h.wait(20.0) for h in [q.submit(r) for r in reqs]]
    d.stop()
    for r, g in zip(reqs, got):
        np.testing.assert_array_equal(g, oracle_scores(P, metric, np.asarray(r.users), emb[r.item_ids]))
    rep = P.batching.stats(q)
    assert rep.total_pairs_dispatched == sum(len(r) for r in reqs)
    assert rep.mean_fill > 0.5


def test_batch_client_roundtrip_device(P):
    model = P.create_model(d_x=4, d_h=4, z_dim=2, hidden=(8,), seed=2)
    rng = np.random.default_rng(6)
    emb = model.item_embeddings(rng.normal(size=(50, 4)).astype(np.float32))
    eng = P.ModelBatchEngine(model, emb, batch_size=16)
    q = P.BatchQueue(capacity=16, flush_timeout_s=0.001)
    d = P.Dispatcher(q, eng).start()
    h_u = model.user_embedding(rng.normal(size=4).astype(np.float32))
    got = P.BatchClient(q, h_u)(np.arange(10))
    d.stop()
    np.testing.assert_array_equal(got, oracle_scores(P, model, h_u[None, :], emb[:10]))
