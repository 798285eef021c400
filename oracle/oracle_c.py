"""ctypes front-end of the C oracle (oracle/c/oracle.c) — CPU ORACLE, test/baseline only.

``build()`` compiles it with ``make -C oracle``; nothing in the product package
imports this module.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.oracle_num_threads.restype = C.c_int
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _ptr_array(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def rank_of(ids: np.ndarray) -> np.ndarray:
    """Tie-break rank per slot: position of ids[slot] in ascending id order."""
    ids = np.asarray(ids, dtype=np.int64)
    rank = np.empty(len(ids), dtype=np.uint32)
    rank[np.argsort(ids, kind="stable")] = np.arange(len(ids), dtype=np.uint32)
    return rank


class _Model:
    def __init__(self, layers, attention, relu):
        self.W = [np.ascontiguousarray(np.asarray(w).astype(np.float32)) for w, _ in layers]
        self.b = [np.ascontiguousarray(np.asarray(b).astype(np.float32)) for _, b in layers]
        self.A = np.ascontiguousarray(np.asarray(attention).astype(np.float32))
        self.dims = np.array([self.W[0].shape[1]] + [w.shape[0] for w in self.W], dtype=np.int32)
        self.relu = int(bool(relu))


def relevance(layers, attention, relu, hu, hv, nthreads=None):
    """fp32 scores of (hu[i], hv[i]) pairs; hu may be one row (broadcast)."""
    m = _Model(layers, attention, relu)
    hv = np.ascontiguousarray(hv, dtype=np.float32)
    hu = np.ascontiguousarray(hu, dtype=np.float32)
    n = hv.shape[0]
    stride = 0 if hu.ndim == 1 or hu.shape[0] == 1 else hu.shape[1]
    out = np.empty(n, dtype=np.float32)
    rc = lib().oracle_relevance(
        C.c_int(len(m.W)), _ptr(m.dims), _ptr_array(m.W), _ptr_array(m.b), _ptr(m.A),
        C.c_int(m.relu), _ptr(hu), C.c_int64(stride), _ptr(hv), C.c_int64(n), _ptr(out),
        C.c_int(nthreads or 1))
    return out, rc == 0


def search(layers, entry_slot, ids, model_layers, attention, relu, items, users,
           k, k_parallel, hops, ef, nthreads=None):
    """Batched hop-synchronous c_hipanns.  Returns dict of arrays."""
    m = _Model(model_layers, attention, relu)
    nbrs = [np.ascontiguousarray(nb, dtype=np.int32) for nb, _ in layers]
    cnts = [np.ascontiguousarray(ct, dtype=np.int32) for _, ct in layers]
    stride = np.array([nb.shape[1] for nb in nbrs], dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    rank = rank_of(ids)
    items = np.ascontiguousarray(items, dtype=np.float32)
    users = np.ascontiguousarray(users, dtype=np.float32)
    Q = users.shape[0]
    L = len(layers)
    out_ids = np.full((Q, k), -1, dtype=np.int64)
    out_scores = np.full((Q, k), np.nan)
    out_n = np.zeros(Q, dtype=np.int32)
    stats = np.zeros((Q, 5 + L), dtype=np.int64)
    rc = lib().oracle_search(
        C.c_int(L), C.c_int64(len(ids)), _ptr_array(nbrs), _ptr(stride), _ptr_array(cnts),
        C.c_int32(int(entry_slot)), _ptr(ids), _ptr(rank),
        C.c_int(len(m.W)), _ptr(m.dims), _ptr_array(m.W), _ptr_array(m.b), _ptr(m.A),
        C.c_int(m.relu), _ptr(items), C.c_int(items.shape[1]), _ptr(users), C.c_int64(Q),
        C.c_int(k), C.c_int(k_parallel), C.c_int(hops), C.c_int(ef),
        C.c_int(nthreads or lib().oracle_num_threads()),
        _ptr(out_ids), _ptr(out_scores), _ptr(out_n), _ptr(stats))
    if rc == 1:
        raise ValueError("oracle_search: bad arguments")
    return dict(ids=out_ids, scores=out_scores, n=out_n, evals=stats[:, 0], visited=stats[:, 1],
                best_hop=stats[:, 2], rows=stats[:, 3], nbr_ids=stats[:, 4],
                per_layer=stats[:, 5:], finite=rc == 0)
