"""CPU ORACLE — test infrastructure only, never the product path.

Plain numpy/Python restatement of the reference HiPANNS hot path:

* the exact fp32 reduction order of numpy's ``einsum('ij,kj->ik')`` that the
  reference uses for every MLP layer (``/root/reference/pkg/src/nann/metric.py:30-32``)
  and for the attention dot (``metric.py:150-154``);
* the fp64 ``einsum('ij,ij->i')`` order of ``euclidean_scorer``
  (``/root/reference/pkg/src/nann/search.py:73-81``);
* ``c_hipanns`` (``search.py:194-286``) restated in its hop-synchronous,
  lowest-searcher-owner form (SURVEY.md §8(a'), H2), and ``brute_force``
  (``search.py:93-108``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may
import this module, and only as the checker.  Parity of this restatement is pinned
against outputs of the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference`` and records ``nann.c_hipanns`` / ``relevance_batch`` results in
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks every vector).
"""

from __future__ import annotations

import numpy as np

F32 = np.float32


# ---------------------------------------------------------------------------
# numpy einsum reduction order (fp32, 'ij,kj->ik'; 4 SSE lanes, 4x unrolled)
# ---------------------------------------------------------------------------

def einsum_rows_f32(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Bit-exact emulation of ``np.einsum('ij,kj->ik', x, w)`` for fp32.

    numpy 2.3's ``sum_of_products_contig_contig_outstride0_two`` (the reduction
    the reference's ``_affine`` hits, metric.py:32) keeps four accumulator lanes;
    for every 16-element block p it computes, per lane l (terms t = 0..3 take
    element p+4t+l), ``acc = a0*b0 + (a1*b1 + (a2*b2 + (a3*b3 + acc)))`` with a
    separately rounded multiply and add; the <16 remainder is consumed in
    zero-padded groups of four (``acc += a*b``); the result is
    ``(acc0 + acc1) + (acc2 + acc3)``.
    """
    x = np.ascontiguousarray(x, dtype=F32)
    w = np.ascontiguousarray(w, dtype=F32)
    n, K = x.shape
    m = w.shape[0]
    out = np.empty((n, m), dtype=F32)
    nb = K // 16
    for o in range(m):
        acc = np.zeros((n, 4), dtype=F32)
        for blk in range(nb):
            p = 16 * blk
            s = x[:, p + 12:p + 16] * w[o, p + 12:p + 16] + acc
            s = x[:, p + 8:p + 12] * w[o, p + 8:p + 12] + s
            s = x[:, p + 4:p + 8] * w[o, p + 4:p + 8] + s
            acc = x[:, p:p + 4] * w[o, p:p + 4] + s
        p = 16 * nb
        while p < K:
            q = min(p + 4, K)
            a = np.zeros((n, 4), dtype=F32)
            b = np.zeros(4, dtype=F32)
            a[:, : q - p] = x[:, p:q]
            b[: q - p] = w[o, p:q]
            acc = a * b + acc
            p += 4
        out[:, o] = (acc[:, 0] + acc[:, 1]) + (acc[:, 2] + acc[:, 3])
    return out


def sqnorm_rows_f64(d: np.ndarray) -> np.ndarray:
    """Bit-exact emulation of ``np.einsum('ij,ij->i', d, d)`` for fp64.

    Two SSE2 lanes, blocks of 8 with the same nested 4x unroll, zero-padded
    pairs for the remainder, result ``acc0 + acc1`` (search.py:79).
    """
    d = np.ascontiguousarray(d, dtype=np.float64)
    n, K = d.shape
    acc = np.zeros((n, 2))
    nb = K // 8
    for blk in range(nb):
        p = 8 * blk
        s = d[:, p + 6:p + 8] * d[:, p + 6:p + 8] + acc
        s = d[:, p + 4:p + 6] * d[:, p + 4:p + 6] + s
        s = d[:, p + 2:p + 4] * d[:, p + 2:p + 4] + s
        acc = d[:, p:p + 2] * d[:, p:p + 2] + s
    p = 8 * nb
    while p < K:
        q = min(p + 2, K)
        a = np.zeros((n, 2))
        a[:, : q - p] = d[:, p:q]
        acc = a * a + acc
        p += 2
    return acc[:, 0] + acc[:, 1]


# ---------------------------------------------------------------------------
# relevance metric (metric.py:102-154)
# ---------------------------------------------------------------------------

class OracleModel:
    """Weights of a ``MetricModel``: layers [(W[out,in], b[out])], attention[Z]."""

    def __init__(self, layers, attention, relu: bool = True):
        # fp16 storage is widened exactly to fp32 (metric.py:35-37,127-131)
        self.layers = [(np.asarray(w).astype(F32), np.asarray(b).astype(F32)) for w, b in layers]
        self.attention = np.asarray(attention).astype(F32)
        self.relu = relu

    @classmethod
    def from_metric(cls, metric):
        return cls(metric.layers, metric.attention, metric.activation == "relu")


def relevance_f32(model: OracleModel, hu: np.ndarray, hv: np.ndarray):
    """Scores for n (user, item) pairs; returns (scores fp32[n], finite_z bool)."""
    hu = np.atleast_2d(hu)
    hv = np.atleast_2d(hv)
    x = np.concatenate([np.broadcast_to(hu, hv.shape), hv], axis=1).astype(F32)
    last = len(model.layers) - 1
    for m, (w, b) in enumerate(model.layers):
        x = einsum_rows_f32(x, w) + b
        if m < last and model.relu:
            # np.maximum(x, 0): max(-0.0, 0) is +0.0 on this numpy
            x = np.where(x > 0, x, F32(0.0)).astype(F32)
    finite = bool(np.isfinite(x).all())
    s = einsum_rows_f32(x, model.attention[None, :])[:, 0]
    return s, finite


def neg_euclid_f64(vectors: np.ndarray, query: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """``euclidean_scorer`` (search.py:73-81): -sqrt(einsum fp64)."""
    diffs = vectors[ids] - np.asarray(query, dtype=np.float64)
    return -np.sqrt(sqnorm_rows_f64(diffs))


# ---------------------------------------------------------------------------
# traversal (search.py:194-286), hop-synchronous restatement
# ---------------------------------------------------------------------------

class OracleGraph:
    """Layers as (nbrs[rows, cap], cnts[rows]) over slots; ``ids`` per slot."""

    def __init__(self, layers, entry_slot: int, ids: np.ndarray):
        self.layers = [(np.asarray(nb), np.asarray(ct)) for nb, ct in layers]
        self.entry = int(entry_slot)
        self.ids = np.asarray(ids, dtype=np.int64)

    @property
    def n_layers(self):
        return len(self.layers)

    def nbrs(self, layer: int, slot: int):
        nb, ct = self.layers[layer]
        return [int(s) for s in nb[slot, : ct[slot]]]


def c_hipanns(graph: OracleGraph, score_slots, k: int, k_parallel: int, hops: int, ef: int):
    """Hop-synchronous C-HiPANNS.

    ``score_slots(slots: list[int]) -> float64 array`` scores a batch of slots.
    Returns dict(items=[(id, score)], evals, per_layer, hops_to_best).

    Per layer (search.py:238-265): seeds = top-kp of everything scored so far
    (the pool is the top-k of all pushes, search.py:239 / pool.py:49-55); every
    searcher's candidate list is the first-occurrence concatenation of its
    frontier's rows (search.py:246-252); a node goes to the lowest-index searcher
    listing it (lock-step claim order, search.py:261-265); fresh claims are scored
    and each searcher keeps the top-ef of its own fresh set (search.py:258-259).
    """
    ids = graph.ids
    top = graph.n_layers - 1
    scores: dict[int, float] = {}
    eval_hop: dict[int, int] = {}
    per_layer = [0] * graph.n_layers
    claimed: set[int] = set()

    def key(s):
        return (-scores[s], int(ids[s]))

    def score(slots, layer, hop):
        if not slots:
            return
        vals = np.asarray(score_slots(list(slots)), dtype=np.float64)
        for s, v in zip(slots, vals):
            scores[s] = float(v)
            eval_hop[s] = hop
        per_layer[layer] += len(slots)

    init = []
    for s in [graph.entry] + graph.nbrs(top, graph.entry):
        if s not in claimed:
            claimed.add(s)
            init.append(s)
    score(init, top, 0)

    hop = 0
    for layer in range(top, -1, -1):
        seeds = sorted(scores, key=key)[:k_parallel]
        frontiers = [[s] for s in seeds]
        for _ in range(hops):
            hop += 1
            owner: dict[int, int] = {}
            for i, fr in enumerate(frontiers):
                for s in fr:
                    for v in graph.nbrs(layer, s):
                        if v not in claimed and v not in owner:
                            owner[v] = i
            fresh = [[] for _ in frontiers]
            for v, i in owner.items():
                fresh[i].append(v)
            flat = [v for f in fresh for v in f]
            claimed.update(flat)
            score(flat, layer, hop)
            frontiers = [sorted(f, key=key)[:ef] for f in fresh]
    ranked = sorted(scores, key=key)[:k]
    items = [(int(ids[s]), scores[s]) for s in ranked]
    best = eval_hop[ranked[0]] if ranked else None
    return dict(items=items, evals=len(scores), per_layer=per_layer, hops_to_best=best)


def brute_force(scores: np.ndarray, item_ids: np.ndarray, k: int):
    """Exact top-k by (score desc, id asc) (search.py:93-108)."""
    order = np.lexsort((item_ids, -scores))[:k]
    return [(int(item_ids[i]), float(scores[i])) for i in order]
