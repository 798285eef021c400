"""C-HiPANNS search over the graph index — device path (mirror of nann.search).

Public surface of /root/reference/pkg/src/nann/search.py:27-286: ``SearchParams``,
``SearchStats``, ``SearchResult``, ``model_scorer``, ``c_hipanns``, ``brute_force``,
plus the batched entry points a GPU needs (``c_hipanns_batch``, ``brute_force_batch``)
because a per-query Python ScoreFn callback cannot feed a GPU.

``c_hipanns`` accepts the ScoreFn objects this package's ``model_scorer`` returns
(they carry model, user embedding and item embeddings) and runs the whole traversal
and scoring in ``libgmpgr.so``.  Any other callable raises InvalidArgumentError:
there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import time
import weakref
from dataclasses import asdict, dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import _lib
from .errors import InvalidArgumentError
from .index import GraphIndex

ScoreFn = Callable[[np.ndarray], np.ndarray]


@dataclass
class SearchParams:
    """Knobs of search.py:30-49 (same defaults, same validation)."""

    k: int = 10
    k_parallel: int = 1
    hops: int = 3
    ef: int | None = None
    deterministic: bool = True
    n_threads: int | None = None
    # device-only extras (not in the reference): scoring engine and refinement band
    mode: str = "exact"          # "exact": CUDA-core exact fp32 | "tc": tcgen05 + exact refinement
    band_rel: float = 0.0        # <= 0: library default (1e-3)
    band_abs: float = 0.0

    def __post_init__(self):
        if self.k < 1 or self.k_parallel < 1 or self.hops < 1:
            raise InvalidArgumentError("k, k_parallel, and hops must be >= 1")
        if self.k_parallel > self.k:
            raise InvalidArgumentError("k_parallel must not exceed k")
        if self.ef is not None and self.ef < 1:
            raise InvalidArgumentError("ef must be >= 1")
        if self.mode not in ("exact", "tc"):
            raise InvalidArgumentError("mode must be 'exact' or 'tc'")

    @property
    def frontier_width(self) -> int:
        return self.ef if self.ef is not None else 2 * self.k

    def _c(self) -> _lib.SearchParamsC:
        return _lib.SearchParamsC(self.k, self.k_parallel, self.hops, self.frontier_width,
                                  _lib.GR_MODE_TC if self.mode == "tc" else _lib.GR_MODE_EXACT,
                                  self.band_rel, self.band_abs)


@dataclass
class SearchStats:
    nodes_visited: int = 0
    metric_evaluations: int = 0
    per_layer_evaluations: list = field(default_factory=list)
    wall_time_s: float = 0.0
    hops_to_best: int | None = None

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass
class SearchResult:
    items: list  # (item_id, score), descending
    stats: SearchStats

    def item_ids(self) -> list:
        return [i for i, _ in self.items]


# ------------------------------------------------------------------ device caches
_items_cache: dict = {}


def device_items(emb, device: int | None = None) -> _lib.DeviceItems:
    """Upload (once) an item-embedding array; cached while the array object lives.

    The device copy is a SNAPSHOT taken at first use (the reference reads the live array on
    every call, search.py:88): after editing an embedding array in place, call
    ``invalidate_device_items(emb)`` (or pass a new array) so the next search re-uploads."""
    device = _lib.current_device() if device is None else device
    if isinstance(emb, np.ndarray):
        sig = (tuple(emb.shape), emb.dtype.str, emb.__array_interface__["data"][0])
    else:  # torch tensor (host or device)
        sig = (tuple(emb.shape), str(emb.dtype), emb.data_ptr())
    key = (id(emb), device)
    hit = _items_cache.get(key)
    if hit is not None and hit[0]() is emb and hit[2] == sig:
        return hit[1]
    h = _lib.DeviceItems(emb, device)
    _items_cache[key] = (weakref.ref(emb, lambda _r, k=key: _items_cache.pop(k, None)), h, sig)
    return h


def invalidate_device_items(emb) -> None:
    """Drop every cached device copy of ``emb`` (after in-place edits)."""
    for key in [k for k in _items_cache if k[0] == id(emb)]:
        _items_cache.pop(key, None)


class ModelScorer:
    """ScoreFn of ``model_scorer`` (search.py:84-90): scores item ids (= embedding rows)
    for one user on the GPU; ``c_hipanns`` recognises it and runs on the device."""

    def __init__(self, model, user_embedding, item_embeddings):
        self.model = model
        self.user = np.ascontiguousarray(user_embedding, dtype=np.float32).reshape(-1)
        self.items = item_embeddings

    @property
    def metric(self):
        return getattr(self.model, "metric", self.model)

    def __call__(self, ids: np.ndarray) -> np.ndarray:
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        out = np.empty(len(ids), dtype=np.float64)
        if len(ids) == 0:
            return out
        dm = self.metric.device_model()
        it = device_items(self.items, dm.device)
        _lib.check(_lib.lib().gr_score_pairs(dm.h, it.h, _lib.ptr(self.user), 1, None,
                                             _lib.ptr(ids), len(ids), _lib.ptr(out), 0, None))
        return out


def model_scorer(model, user_embedding: np.ndarray, item_embeddings: np.ndarray) -> ScoreFn:
    """Learned-metric scorer over precomputed item embeddings (dense ids)."""
    return ModelScorer(model, user_embedding, item_embeddings)


class EuclideanScorer:
    """ScoreFn of ``euclidean_scorer`` (search.py:73-81): -||v - q|| in fp64, item ids are
    row indexes.  Scores come from the device (gr_scores_euclid, numpy's fp64 einsum order,
    bit-exact); ``c_hipanns`` runs the traversal on the device over that score table."""

    def __init__(self, query, item_vectors):
        self.query = np.asarray(query, dtype=np.float64).reshape(-1)
        self.vectors = np.asarray(item_vectors)
        self._table = None

    def device_scores(self, device: int | None = None) -> _lib.DeviceScores:
        device = _lib.current_device() if device is None else device
        if self._table is None or self._table.device != device:
            self._table = _lib.DeviceScores(vectors=self.vectors, queries=self.query[None, :],
                                            device=device)
        return self._table

    def __call__(self, ids: np.ndarray) -> np.ndarray:
        ids = np.asarray(ids, dtype=np.int64)
        return self.device_scores().read()[0][ids]


def euclidean_scorer(query: np.ndarray, item_vectors: np.ndarray) -> ScoreFn:
    """Score = negated Euclidean distance; item ids must be row indexes."""
    return EuclideanScorer(query, item_vectors)


class TableScorer:
    """A ScoreFn given as its fp64 values over item ids 0..n-1 (``scores[id]``): the
    traversal-only form of an arbitrary ScoreFn (search.py:27) the device can run."""

    def __init__(self, scores):
        self.scores = np.ascontiguousarray(scores, dtype=np.float64).reshape(-1)
        self._table = None

    def device_scores(self, device: int | None = None) -> _lib.DeviceScores:
        device = _lib.current_device() if device is None else device
        if self._table is None or self._table.device != device:
            self._table = _lib.DeviceScores(self.scores[None, :], device=device)
        return self._table

    def __call__(self, ids: np.ndarray) -> np.ndarray:
        return self.scores[np.asarray(ids, dtype=np.int64)]


def table_scorer(scores: np.ndarray) -> ScoreFn:
    return TableScorer(scores)


# ------------------------------------------------------------------ batched search
@dataclass
class BatchSearchResult:
    """Arrays for Q queries: ids/scores [Q, k] (-1 / nan padded), count [Q], stats."""

    ids: np.ndarray
    scores: np.ndarray
    count: np.ndarray
    evals: np.ndarray
    rows_expanded: np.ndarray
    nbr_ids_read: np.ndarray
    hops_to_best: np.ndarray
    per_layer: np.ndarray
    wall_time_s: float = 0.0

    def result(self, q: int) -> SearchResult:
        n = int(self.count[q])
        items = [(int(i), float(s)) for i, s in zip(self.ids[q, :n], self.scores[q, :n])]
        hb = int(self.hops_to_best[q])
        st = SearchStats(nodes_visited=int(self.evals[q]), metric_evaluations=int(self.evals[q]),
                         per_layer_evaluations=[int(v) for v in self.per_layer[q]],
                         wall_time_s=self.wall_time_s / max(1, len(self.count)),
                         hops_to_best=None if hb < 0 else hb)
        return SearchResult(items=items, stats=st)

    def results(self) -> list:
        return [self.result(q) for q in range(len(self.count))]


_searchers: dict = {}


def _searcher(device: int) -> _lib.DeviceSearcher:
    s = _searchers.get(device)
    if s is None:
        s = _searchers[device] = _lib.DeviceSearcher(device)
    return s


def c_hipanns_batch(index: GraphIndex, model, users, item_embeddings,
                    params: SearchParams, device: int | None = None,
                    searcher: _lib.DeviceSearcher | None = None) -> BatchSearchResult:
    """C-HiPANNS for Q user embeddings at once (deterministic lock-step semantics,
    search.py:194-286), exact-fp32 scores; all traversal and scoring on the device."""
    if len(index) == 0:
        raise InvalidArgumentError("index is empty")
    metric = getattr(model, "metric", model)
    users = np.ascontiguousarray(np.atleast_2d(users), dtype=np.float32)
    device = _lib.current_device() if device is None else device
    dm = metric.device_model(device)
    if users.shape[1] != dm.d_h:
        raise InvalidArgumentError(f"user embedding dim {users.shape[1]} != d_h {dm.d_h}")
    g = index.device_graph(device, items=item_embeddings)
    it = device_items(item_embeddings, device)
    if it.d != dm.d_h:
        raise InvalidArgumentError("item embedding dim != model d_h")
    s = searcher or _searcher(device)
    Q, k, L = users.shape[0], params.k, g.n_layers
    ids = np.empty((Q, k), dtype=np.int64)
    scores = np.empty((Q, k), dtype=np.float64)
    count = np.empty(Q, dtype=np.int32)
    stats = np.empty((Q, 5 + L), dtype=np.int64)
    pc = params._c()
    t0 = time.perf_counter()
    _lib.check(_lib.lib().gr_search(s.h, g.h, dm.h, it.h, _lib.ptr(users), Q,
                                    ctypes.byref(pc),
                                    _lib.ptr(ids), _lib.ptr(scores), _lib.ptr(count),
                                    _lib.ptr(stats), 0, None))
    wall = time.perf_counter() - t0
    return BatchSearchResult(ids=ids, scores=scores, count=count, evals=stats[:, 0],
                             rows_expanded=stats[:, 3], nbr_ids_read=stats[:, 4],
                             hops_to_best=stats[:, 2], per_layer=stats[:, 5:], wall_time_s=wall)


def c_hipanns_scores_batch(index: GraphIndex, scores, params: SearchParams,
                           device: int | None = None,
                           searcher: _lib.DeviceSearcher | None = None) -> BatchSearchResult:
    """C-HiPANNS for every row of a score table (``DeviceScores`` or an fp64 array
    [Q, n_items] by item id): traversal-only mode used by the reference's search tests."""
    if len(index) == 0:
        raise InvalidArgumentError("index is empty")
    if params.mode != "exact":
        raise InvalidArgumentError("score tables run in exact mode only")
    device = _lib.current_device() if device is None else device
    if not isinstance(scores, _lib.DeviceScores):
        scores = _lib.DeviceScores(scores, device=device)
    g = index.device_graph(device)
    s = searcher or _searcher(device)
    Q, k, L = scores.Q, params.k, g.n_layers
    ids = np.empty((Q, k), dtype=np.int64)
    sc = np.empty((Q, k), dtype=np.float64)
    count = np.empty(Q, dtype=np.int32)
    stats = np.empty((Q, 5 + L), dtype=np.int64)
    pc = params._c()
    t0 = time.perf_counter()
    _lib.check(_lib.lib().gr_search_scores(s.h, g.h, scores.h, ctypes.byref(pc), _lib.ptr(ids),
                                           _lib.ptr(sc), _lib.ptr(count), _lib.ptr(stats), 0, None))
    wall = time.perf_counter() - t0
    return BatchSearchResult(ids=ids, scores=sc, count=count, evals=stats[:, 0],
                             rows_expanded=stats[:, 3], nbr_ids_read=stats[:, 4],
                             hops_to_best=stats[:, 2], per_layer=stats[:, 5:], wall_time_s=wall)


def c_hipanns(index: GraphIndex, score_fn: ScoreFn, params: SearchParams) -> SearchResult:
    """Breadth-parallel layered search with a shared candidate pool (search.py:194-286).

    ``score_fn`` must come from ``model_scorer``; the device runs the lock-step
    schedule (deterministic=True semantics) for either ``deterministic`` setting —
    one legal linearisation of the threaded mode, which the reference leaves
    unspecified (search.py:266-275).
    """
    if len(index) == 0:
        raise InvalidArgumentError("index is empty")
    if isinstance(score_fn, (EuclideanScorer, TableScorer)):
        return c_hipanns_scores_batch(index, score_fn.device_scores(), params).result(0)
    if not isinstance(score_fn, ModelScorer):
        raise InvalidArgumentError(
            "c_hipanns runs on the GPU: score_fn must come from model_scorer(...), "
            "euclidean_scorer(...) or table_scorer(...) "
            "(there is no CPU fallback for arbitrary callables)")
    r = c_hipanns_batch(index, score_fn.model, score_fn.user[None, :], score_fn.items, params)
    return r.result(0)


# ------------------------------------------------------------------ ground truth
def brute_force_batch(model, users, item_embeddings, k: int, device: int | None = None):
    """Exact top-k over all items for each user (search.py:93-108) -> (ids, scores)."""
    metric = getattr(model, "metric", model)
    users = np.ascontiguousarray(np.atleast_2d(users), dtype=np.float32)
    device = _lib.current_device() if device is None else device
    dm = metric.device_model(device)
    it = device_items(item_embeddings, device)
    if k > it.n:
        raise InvalidArgumentError(f"k={k} exceeds item count {it.n}")
    Q = users.shape[0]
    ids = np.empty((Q, k), dtype=np.int64)
    scores = np.empty((Q, k), dtype=np.float64)
    _lib.check(_lib.lib().gr_brute_force(dm.h, it.h, _lib.ptr(users), Q, k, _lib.ptr(ids),
                                         _lib.ptr(scores), 0, None))
    return ids, scores


def brute_force(score_fn: ScoreFn, item_ids: Sequence[int], k: int) -> SearchResult:
    """Exact top-k by exhaustive scoring; the ground-truth oracle (search.py:93-108)."""
    item_ids = np.asarray(item_ids, dtype=np.int64)
    if k > len(item_ids):
        raise InvalidArgumentError(f"k={k} exceeds item count {len(item_ids)}")
    if not isinstance(score_fn, (ModelScorer, EuclideanScorer, TableScorer)):
        raise InvalidArgumentError("brute_force runs on the GPU: use model_scorer(...), "
                                   "euclidean_scorer(...) or table_scorer(...)")
    t0 = time.perf_counter()
    n_items = score_fn.items.shape[0] if isinstance(score_fn, ModelScorer) else -1
    if isinstance(score_fn, ModelScorer) and len(item_ids) == n_items and \
            np.array_equal(item_ids, np.arange(n_items)):
        ids, scores = brute_force_batch(score_fn.model, score_fn.user[None, :], score_fn.items, k)
        items = [(int(i), float(s)) for i, s in zip(ids[0], scores[0])]
    else:
        import torch

        sc = torch.from_numpy(score_fn(item_ids)).cuda()
        idt = torch.from_numpy(item_ids).cuda()
        o1 = torch.argsort(idt, stable=True)
        o2 = torch.argsort(-sc[o1], stable=True)
        order = o1[o2][:k].cpu().numpy()
        items = [(int(item_ids[i]), float(v)) for i, v in
                 zip(order, sc.cpu().numpy()[order])]
    st = SearchStats(nodes_visited=len(item_ids), metric_evaluations=len(item_ids),
                     per_layer_evaluations=[len(item_ids)], wall_time_s=time.perf_counter() - t0)
    return SearchResult(items=items, stats=st)


# ------------------------------------------------------------------ metrics (evalharness.py:36-48)
def coverage(retrieved_ids, ground_truth_ids) -> float:
    gt = set(ground_truth_ids)
    if not gt:
        raise InvalidArgumentError("empty ground truth")
    return len(set(retrieved_ids) & gt) / len(gt)


def recall_at(k: int, retrieved_ids, ground_truth_ids) -> float:
    if k < 1:
        raise InvalidArgumentError("k must be >= 1")
    return len(set(list(retrieved_ids)[:k]) & set(list(ground_truth_ids)[:k])) / k
