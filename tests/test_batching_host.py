"""Q-HiPANNS host logic (BatchQueue / Dispatcher / stats / BatchClient) on CPU.

Mirrors the reference's test_batching.py (TestSlicing / TestCorrectness / TestThroughput)
with a pure host stand-in engine (score = user[0] + item_id / 1000) that records batch
compositions; the device engine is exercised in test_gpu_batching.py.
"""

import threading
import time

import numpy as np
import pytest

from paper_2502_11490_b200.batching import (
    BatchClient,
    BatchEngine,
    BatchQueue,
    Dispatcher,
    EvalRequest,
    run_dispatcher,
    stats,
)
from paper_2502_11490_b200.errors import InvalidArgumentError, QueueShutdownError


class StubEngine(BatchEngine):
    def __init__(self, batch_size, fail_on=None, cost=(0.0, 0.0)):
        self.batch_size = batch_size
        self.invocations = 0
        self.batches = []
        self.fail_on = fail_on
        self.cost = cost
        self.simulated_seconds = 0.0

    def evaluate(self, users, item_ids):
        self.invocations += 1
        self.simulated_seconds += self.cost[0] + self.cost[1] * len(item_ids)
        self.batches.append([int(i) for i in item_ids])
        if self.fail_on == self.invocations:
            raise RuntimeError("injected engine failure")
        return users[:, 0].astype(np.float64) + item_ids.astype(np.float64) / 1000.0


def req(user, ids):
    ids = np.asarray(ids, dtype=np.int64)
    return EvalRequest(users=np.full((len(ids), 2), float(user)), item_ids=ids)


def expect(r):
    return r.users[:, 0].astype(np.float64) + r.item_ids.astype(np.float64) / 1000.0


def random_requests(rng, n, max_size):
    return [req(float(rng.normal()), rng.integers(0, 5000, size=int(s)))
            for s in rng.integers(1, max_size + 1, size=n)]


def test_exact_fit_is_one_invocation():
    eng, q = StubEngine(8), BatchQueue(capacity=8, flush_timeout_s=10.0)
    h = q.submit(req(1.0, range(8)))
    d = Dispatcher(q, eng).start()
    got = h.wait(5.0)
    d.stop()
    assert eng.invocations == 1
    np.testing.assert_array_equal(got, 1.0 + np.arange(8) / 1000.0)


def test_one_over_capacity_splits():
    eng, q = StubEngine(8), BatchQueue(capacity=8, flush_timeout_s=0.01)
    h = q.submit(req(2.0, range(9)))
    d = Dispatcher(q, eng).start()
    got = h.wait(5.0)
    d.stop()
    assert [len(b) for b in eng.batches] == [8, 1]
    np.testing.assert_array_equal(got, 2.0 + np.arange(9) / 1000.0)


def test_straddling_requests_are_sliced_fifo():
    eng, q = StubEngine(4), BatchQueue(capacity=4, flush_timeout_s=0.01)
    h1, h2 = q.submit(req(1.0, [10, 11, 12])), q.submit(req(2.0, [20, 21, 22]))
    d = Dispatcher(q, eng).start()
    s1, s2 = h1.wait(5.0), h2.wait(5.0)
    d.stop()
    assert eng.batches == [[10, 11, 12, 20], [21, 22]]
    np.testing.assert_array_equal(s1, 1.0 + np.array([10, 11, 12]) / 1000.0)
    np.testing.assert_array_equal(s2, 2.0 + np.array([20, 21, 22]) / 1000.0)


def test_singletons_fill_batches_and_drain_flushes_tail():
    eng, q = StubEngine(256), BatchQueue(capacity=256, flush_timeout_s=30.0)
    hs = [q.submit(req(0.5, [i])) for i in range(1000)]
    Dispatcher(q, eng).start().stop(drain=True)
    assert all(h.done for h in hs)
    rep = stats(q)
    assert eng.invocations == 4 and rep.timeout_flushes == 0 and rep.drain_flushes == 1
    assert rep.mean_fill >= 0.97 and sum(rep.batch_sizes) == 1000
    assert rep.total_pairs_submitted == 1000


def test_idle_dispatcher_never_invokes():
    eng, q = StubEngine(4), BatchQueue(capacity=4, flush_timeout_s=0.005)
    d = Dispatcher(q, eng).start()
    time.sleep(0.05)
    d.stop()
    assert eng.invocations == 0 and stats(q).invocations == 0


def test_argument_errors():
    with pytest.raises(InvalidArgumentError):
        BatchQueue(capacity=4).submit(req(0.0, []))
    with pytest.raises(InvalidArgumentError):
        BatchQueue(capacity=0)
    with pytest.raises(InvalidArgumentError):
        BatchQueue(capacity=8, max_pending_pairs=4)
    with pytest.raises(InvalidArgumentError):
        Dispatcher(BatchQueue(capacity=8), StubEngine(4))


def test_concurrent_submitters_match_direct_evaluation():
    rng = np.random.default_rng(0)
    reqs = random_requests(rng, 200, 32)
    eng, q = StubEngine(64), BatchQueue(capacity=64, flush_timeout_s=0.002)
    d = Dispatcher(q, eng).start()
    hs = [None] * len(reqs)

    def submit(lo, hi):
        for i in range(lo, hi):
            hs[i] = q.submit(reqs[i])

    ts = [threading.Thread(target=submit, args=(50 * i, 50 * i + 50)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    got = [h.wait(10.0) for h in hs]
    d.stop()
    for r, g in zip(reqs, got):
        np.testing.assert_array_equal(g, expect(r))


def test_conservation_and_invocation_bound():
    rng = np.random.default_rng(2)
    reqs = random_requests(rng, 300, 24)
    total = sum(len(r) for r in reqs)
    eng, q = StubEngine(128), BatchQueue(capacity=128, flush_timeout_s=0.001)
    d = Dispatcher(q, eng).start()
    for h in [q.submit(r) for r in reqs]:
        h.wait(10.0)
    d.stop()
    rep = stats(q)
    assert rep.total_pairs_dispatched == total == sum(rep.batch_sizes)
    assert rep.invocations <= int(np.ceil(total / 128)) + rep.timeout_flushes + rep.drain_flushes


def test_fifo_order_of_pairs():
    rng = np.random.default_rng(3)
    reqs = [req(i, rng.integers(0, 100, size=int(rng.integers(1, 30)))) for i in range(40)]
    eng, q = StubEngine(16), BatchQueue(capacity=16, flush_timeout_s=0.001)
    d = Dispatcher(q, eng).start()
    for h in [q.submit(r) for r in reqs]:
        h.wait(10.0)
    d.stop()
    assert [i for b in eng.batches for i in b] == [int(i) for r in reqs for i in r.item_ids]


def test_engine_failure_isolated_to_its_batch():
    eng, q = StubEngine(8, fail_on=2), BatchQueue(capacity=8, flush_timeout_s=0.01)
    d = Dispatcher(q, eng).start()
    h1, h2, h3 = (q.submit(req(u, range(8))) for u in (1.0, 2.0, 3.0))
    assert len(h1.wait(5.0)) == 8
    with pytest.raises(RuntimeError, match="injected"):
        h2.wait(5.0)
    assert len(h3.wait(5.0)) == 8
    d.stop()


def test_submit_after_shutdown_rejected():
    q = BatchQueue(capacity=4)
    Dispatcher(q, StubEngine(4)).start().stop()
    with pytest.raises(QueueShutdownError):
        q.submit(req(0.0, [1]))


def test_backpressure_blocks_then_releases():
    eng, q = StubEngine(4), BatchQueue(capacity=4, flush_timeout_s=0.001, max_pending_pairs=8)
    d = Dispatcher(q, eng).start()
    done = []

    def produce():
        for i in range(20):
            q.submit(req(i, [1, 2]))
        done.append(True)

    t = threading.Thread(target=produce)
    t.start()
    t.join(timeout=10.0)
    assert done
    d.stop()
    assert stats(q).total_pairs_dispatched == 40


def test_pipeline_mode_same_results():
    rng = np.random.default_rng(4)
    reqs = random_requests(rng, 100, 16)
    eng, q = StubEngine(32), BatchQueue(capacity=32, flush_timeout_s=0.002)
    d = run_dispatcher(q, eng, pipeline=True)
    got = [h.wait(10.0) for h in [q.submit(r) for r in reqs]]
    d.stop()
    for r, g in zip(reqs, got):
        np.testing.assert_array_equal(g, expect(r))


def test_modelled_invocation_reduction():
    rng = np.random.default_rng(5)
    sizes = rng.integers(1, 33, size=1000)
    overhead, per_pair = 2e-4, 1e-7
    eng, q = StubEngine(256, cost=(overhead, per_pair)), BatchQueue(capacity=256, flush_timeout_s=5.0)
    hs = [q.submit(req(0.0, rng.integers(0, 1000, size=int(s)))) for s in sizes]
    Dispatcher(q, eng).start().stop(drain=True)
    assert all(h.done for h in hs)
    total, rep = int(sizes.sum()), stats(q)
    assert rep.invocations <= int(np.ceil(total / 256)) + rep.timeout_flushes + 1
    per_request = 1000 * overhead + total * per_pair
    assert per_request / eng.simulated_seconds > 5


def test_idle_queue_stats_zero():
    rep = stats(BatchQueue(capacity=16))
    assert rep.invocations == 0 and rep.mean_fill == 0.0 and rep.total_pairs_submitted == 0
    assert rep.to_dict()["mean_request_latency_s"] == 0.0


def test_batch_client_roundtrip():
    eng, q = StubEngine(16), BatchQueue(capacity=16, flush_timeout_s=0.001)
    d = Dispatcher(q, eng).start()
    got = BatchClient(q, np.array([0.25, 9.0]))(np.arange(10))
    d.stop()
    np.testing.assert_array_equal(got, 0.25 + np.arange(10) / 1000.0)
