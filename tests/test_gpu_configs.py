"""BASELINE configs 1 and 2 on the reference's OWN inputs, through the C ABI, vs the
reference's recorded results (tests/golden/make_cfg_golden.py ran nann itself).

The box regenerates the inputs with numpy (workload.reference_inputs: the reference's
clustered_vectors / create_model / projector recipe, digests checked against the
reference's arrays) and the graph with the native exact build (digest checked against
the reference's GraphIndex.build), then every golden query must return the reference's
ids, bit-identical fp64 scores, evaluation counts, per-layer counts, hops_to_best, rows
expanded and neighbour ids read -- in exact AND tensor-core mode -- and recall@100 equals
the reference's.  Also here: thread safety of the shared searcher, the tc-mode band
certificate counters, and the world-1 NCCL sharded path vs per-shard search + pool merge.
"""

import hashlib
import os
import threading

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2502_11490_b200 as P
    from paper_2502_11490_b200 import _lib

    if _lib.lib().gr_device_count() < 1:
        pytest.skip("no GPU")
    return P


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


_WL = {}


def reference_workload(P, name):
    if name not in _WL:
        from paper_2502_11490_b200 import workload

        z = G.load(f"{name}_ref")
        model, emb, users = workload.reference_inputs(name)
        assert _sha(emb) == str(z["items_sha256"]), "items differ from the reference's"
        assert _sha(users) == str(z["users_sha256"]), "users differ from the reference's"
        idx = P.GraphIndex.build(emb.astype(np.float64), m=int(z["m"]), ef_construction=64, seed=0)
        assert workload.graph_digest(idx) == str(z["graph_sha256"]), "graph differs from the reference build"
        _WL[name] = (z, model, emb, users, idx)
    return _WL[name]


def check_against_golden(P, name, mode):
    z, model, emb, users, idx = reference_workload(P, name)
    for pi, p in G.param_sets(z):
        exp = G.expected(z, pi)
        nq = exp["ids"].shape[0]
        r = P.c_hipanns_batch(idx, model, users[:nq], emb, P.SearchParams(**p, mode=mode))
        np.testing.assert_array_equal(r.ids, exp["ids"])
        np.testing.assert_array_equal(r.scores, exp["scores"])
        np.testing.assert_array_equal(r.count, exp["n"])
        np.testing.assert_array_equal(r.evals, exp["evals"])
        np.testing.assert_array_equal(r.per_layer, exp["per_layer"])
        np.testing.assert_array_equal(r.hops_to_best, exp["best_hop"])
        np.testing.assert_array_equal(r.rows_expanded, exp["rows"])
        np.testing.assert_array_equal(r.nbr_ids_read, exp["nbr_ids"])
        gt = z["gt100"]
        ng = min(nq, gt.shape[0])
        rec = np.mean([len(set(r.ids[q]) & set(gt[q])) / 100.0 for q in range(ng)])
        assert rec == pytest.approx(float(z[f"p{pi}/recall100"]), abs=1e-12)


@pytest.mark.parametrize("mode", ["exact", "tc"])
def test_cfg1_reference_inputs_match_reference(P, mode):
    check_against_golden(P, "cfg1", mode)


def test_cfg1_brute_force_matches_reference(P):
    z, model, emb, users, idx = reference_workload(P, "cfg1")
    n = z["gt100"].shape[0]
    ids, scores = P.brute_force_batch(model, users[:n], emb, 100)
    np.testing.assert_array_equal(ids, z["gt100"])
    np.testing.assert_array_equal(scores, z["gt100_scores"])


@pytest.mark.skipif(os.environ.get("GMPGR_CFG2_TESTS") != "1",
                    reason="cfg2 (1M items) rebuilds the reference graph natively (minutes of host "
                           "time): opt in with GMPGR_CFG2_TESTS=1")
@pytest.mark.parametrize("mode", ["exact", "tc"])
def test_cfg2_reference_inputs_match_reference(P, mode):
    check_against_golden(P, "cfg2", mode)


def test_tc_band_certificate_counters(P):
    """tc mode on cfg1: every exact re-score compared its approximate score; no violation
    of |approx - exact| < band/2, so no exact re-run was needed."""
    from paper_2502_11490_b200 import _lib

    z, model, emb, users, idx = reference_workload(P, "cfg1")
    s = _lib.DeviceSearcher(0)
    P.c_hipanns_batch(idx, model, users, emb, P.SearchParams(k=100, k_parallel=8, hops=3, mode="tc"),
                      searcher=s)
    c = s.counters()
    assert c["exact_rescored"] > 0
    assert c["band_violations"] == 0 and c["exact_reruns"] == 0, c
    assert 0.0 < c["max_err_over_band"] < 0.5, c


def test_tc_band_violation_forces_exact_rerun(P):
    """A band far below the split-bf16 error makes the certificate fail: gr_search re-runs
    the batch in exact mode and returns the exact results (async callers get BandError)."""
    import ctypes

    import torch

    from paper_2502_11490_b200 import _lib

    z, model, emb, users, idx = reference_workload(P, "cfg1")
    p = dict(k=100, k_parallel=8, hops=3)
    s = _lib.DeviceSearcher(0)
    tiny = P.SearchParams(**p, mode="tc", band_rel=1e-12, band_abs=1e-12)
    r = P.c_hipanns_batch(idx, model, users[:64], emb, tiny, searcher=s)
    c = s.counters()
    assert c["band_violations"] > 0 and c["exact_reruns"] == 1, c
    exp = G.expected(z, 0)
    np.testing.assert_array_equal(r.ids, exp["ids"][:64])
    np.testing.assert_array_equal(r.scores, exp["scores"][:64])
    # async path: the violation is reported, never silently accepted
    dm, g = model.metric.device_model(0), idx.device_graph(0)
    from paper_2502_11490_b200.search import device_items

    it = device_items(emb, 0)
    Q, L = 64, g.n_layers
    u = torch.from_numpy(users[:Q]).cuda()
    o_i = torch.empty((Q, 100), dtype=torch.int64, device="cuda")
    o_s = torch.empty((Q, 100), dtype=torch.float64, device="cuda")
    o_c = torch.empty(Q, dtype=torch.int32, device="cuda")
    o_t = torch.empty((Q, 5 + L), dtype=torch.int64, device="cuda")
    pc = tiny._c()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(_lib.lib().gr_search_async(s.h, g.h, dm.h, it.h, u.data_ptr(), Q, ctypes.byref(pc),
                                          o_i.data_ptr(), o_s.data_ptr(), o_c.data_ptr(), o_t.data_ptr(), st))
    with pytest.raises(P.BandError):
        _lib.check(_lib.lib().gr_searcher_status(s.h, st))


def test_shared_searcher_is_thread_safe(P):
    """c_hipanns from several host threads shares one cached searcher; every
    thread must get its own query's results (reference evalharness.py:346-351 runs
    c_hipanns from a ThreadPoolExecutor)."""
    z, model, emb, users, idx = reference_workload(P, "cfg1")
    exp = G.expected(z, 0)
    params = P.SearchParams(k=100, k_parallel=8, hops=3, mode="tc")
    got = {}
    errors = []

    def worker(t):
        try:
            for q in range(t, 48, 6):
                r = P.c_hipanns(idx, P.model_scorer(model, users[q], emb), params)
                got[q] = r
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for q in range(48):
        r = got[q]
        assert [i for i, _ in r.items] == list(exp["ids"][q][: exp["n"][q]])
        assert [s for _, s in r.items] == list(exp["scores"][q][: exp["n"][q]])
        assert r.stats.metric_evaluations == exp["evals"][q]


def test_items_table_too_small_is_rejected(P):
    z, model, emb, users, idx = reference_workload(P, "cfg1")
    with pytest.raises(P.InvalidArgumentError):
        P.c_hipanns_batch(idx, model, users[:2], emb[:1000], P.SearchParams(k=10, k_parallel=2))


def _nccl_world1_worker(q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(29513)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        q.put(_sharded_check())
    except Exception as e:  # pragma: no cover
        q.put(repr(e))
    finally:
        dist.destroy_process_group()


def _sharded_check():
    """Two host-sliced shards of the cfg1 items searched by ShardedSearcher-style calls
    (local search + packed NCCL all-gather + device merge) == the restatement: per-shard
    c_hipanns (oracle) followed by CandidatePool(k).push of every shard result."""
    import torch

    import paper_2502_11490_b200 as P
    from oracle import oracle_c
    from paper_2502_11490_b200 import workload
    from paper_2502_11490_b200.distributed import ShardedSearcher, gather_packed, merge_packed, pack_lists

    model, emb, users = workload.reference_inputs("cfg1", n_queries=48)
    n = len(emb)
    half = n // 2
    params = dict(k=100, k_parallel=8, hops=3, ef=200)
    shard_out = []
    packed = []
    for lo, hi in ((0, half), (half, n)):
        idx = P.GraphIndex.build(emb[lo:hi].astype(np.float64), ids=np.arange(lo, hi, dtype=np.int64),
                                 m=16, ef_construction=64, seed=lo)
        idx.rows = np.arange(hi - lo, dtype=np.int32)
        ss = ShardedSearcher(idx, model, emb[lo:hi], device=0)
        u = torch.from_numpy(users).cuda()
        ids, sc, _, _ = ss.search_local(u, P.SearchParams(**params, mode="tc"))
        out = ss.search(u, P.SearchParams(**params))  # world 1: gather of one list + merge
        np.testing.assert_array_equal(out[0].cpu().numpy(), ids.cpu().numpy())
        packed.append(gather_packed(pack_lists(ids, sc)))
        ids_v, _, layers, entry = idx.graph_view()
        m = model.metric
        # the oracle reads items[id]: the full table with global ids = the shard's local rows
        o = oracle_c.search(layers, entry, ids_v, m.layers, m.attention, True, emb, users,
                            **params, nthreads=8)
        shard_out.append(o)
    mi, ms, mc = merge_packed(torch.cat(packed, 0), 100)
    mi, ms = mi.cpu().numpy(), ms.cpu().numpy()
    for q in range(len(users)):
        pool = P.CandidatePool(100)
        for o in shard_out:
            for i, s in zip(o["ids"][q], o["scores"][q]):
                if i >= 0:
                    pool.push(int(i), float(s))
        top = pool.top(100)
        if [i for i, _ in top] != list(mi[q]) or [s for _, s in top] != list(ms[q]):
            return f"query {q} differs"
    return "ok"


def test_sharded_world1_nccl_equals_per_shard_pool_merge(P):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1_worker, args=(q,))
    p.start()
    p.join(timeout=600)
    assert q.get(timeout=5) == "ok"


def test_failed_call_leaves_the_searcher_usable(P, monkeypatch):
    """SURVEY §5 failure isolation: a call that fails (allocation over the scratch budget,
    a contract violation) fails alone -- the next call on the same handles returns the
    reference's results."""
    from paper_2502_11490_b200 import _lib

    z, model, emb, users, idx = reference_workload(P, "cfg1")
    exp = G.expected(z, 0)
    s = _lib.DeviceSearcher(0)
    params = P.SearchParams(k=100, k_parallel=8, hops=3, mode="tc")
    monkeypatch.setenv("GMPGR_SCRATCH_GB", "0.000001")
    with pytest.raises(MemoryError):
        P.c_hipanns_batch(idx, model, users[:32], emb, params, searcher=s)
    monkeypatch.delenv("GMPGR_SCRATCH_GB")
    with pytest.raises(P.InvalidArgumentError):
        P.c_hipanns_batch(idx, model, users[:32, :10], emb, params, searcher=s)
    r = P.c_hipanns_batch(idx, model, users[:32], emb, params, searcher=s)
    np.testing.assert_array_equal(r.ids, exp["ids"][:32])
    np.testing.assert_array_equal(r.scores, exp["scores"][:32])


def test_streamed_host_call_equals_plain_path(P, monkeypatch):
    """gr_search with host buffers, >= 4096 queries and GMPGR_STREAM=1 streams users in and
    results out in chunks beside one persistent launch: identical results to the plain
    (copy, launch, copy) path and to the reference's goldens for the first queries."""
    from paper_2502_11490_b200 import workload

    z, model, emb, _, idx = reference_workload(P, "cfg1")
    _, _, users = workload.reference_inputs("cfg1", n_queries=6000)
    exp = G.expected(z, 0)
    params = P.SearchParams(k=100, k_parallel=8, hops=3, mode="tc")
    monkeypatch.setenv("GMPGR_STREAM", "1")
    a = P.c_hipanns_batch(idx, model, users, emb, params)
    monkeypatch.setenv("GMPGR_STREAM", "0")
    b = P.c_hipanns_batch(idx, model, users, emb, params)
    for f in ("ids", "scores", "count", "evals", "per_layer", "hops_to_best", "rows_expanded", "nbr_ids_read"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    n = exp["ids"].shape[0]
    np.testing.assert_array_equal(a.ids[:n], exp["ids"])
    np.testing.assert_array_equal(a.scores[:n], exp["scores"])
