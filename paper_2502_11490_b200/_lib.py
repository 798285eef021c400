"""ctypes binding of libgmpgr.so (include/gmpgr.h) and RAII handle wrappers.

The library is the product path: there is no fallback.  If it is missing or no
CUDA device is present, every compute call raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import BandError, DeviceError, InvalidArgumentError, NumericError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GMPGR_LIB") or os.path.join(HERE, "libgmpgr.so")

GR_OK, GR_EINVAL, GR_ENUMERIC, GR_ECUDA, GR_ENOMEM, GR_EBAND = 0, 1, 2, 3, 4, 5

# every symbol include/gmpgr.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "gr_last_error", "gr_abi_version", "gr_device_count",
    "gr_model_create", "gr_model_destroy",
    "gr_graph_create", "gr_graph_create_ordered", "gr_graph_destroy",
    "gr_items_create", "gr_items_destroy",
    "gr_score_pairs", "gr_score_items_approx",
    "gr_searcher_create", "gr_searcher_destroy",
    "gr_search", "gr_search_async", "gr_searcher_status", "gr_searcher_launches",
    "gr_searcher_counters",
    "gr_brute_force", "gr_merge_topk",
    "gr_scores_create", "gr_scores_euclid", "gr_scores_read", "gr_scores_destroy",
    "gr_search_scores",
    "gr_hnsw_insert", "gr_pack_topk", "gr_merge_topk_packed",
)


GR_MODE_EXACT, GR_MODE_TC = 0, 1


class SearchParamsC(C.Structure):
    _fields_ = [("k", C.c_int32), ("k_parallel", C.c_int32), ("hops", C.c_int32),
                ("ef", C.c_int32), ("mode", C.c_int32), ("band_rel", C.c_float),
                ("band_abs", C.c_float)]


_lib = None
_lock = threading.Lock()
vp = C.c_void_p


def _declare(lib):
    i32, i64 = C.c_int32, C.c_int64
    sig = {
        "gr_last_error": (C.c_char_p, []),
        "gr_abi_version": (C.c_int, []),
        "gr_device_count": (C.c_int, []),
        "gr_model_create": (C.c_int, [C.c_int, C.c_int, vp, vp, vp, vp, C.c_int, vp]),
        "gr_model_destroy": (C.c_int, [vp]),
        "gr_graph_create": (C.c_int, [C.c_int, C.c_int, i64, vp, vp, vp, vp, i32, vp, vp, vp]),
        "gr_graph_create_ordered": (C.c_int, [C.c_int, C.c_int, i64, vp, vp, vp, vp, i32, vp, vp, vp, vp]),
        "gr_graph_destroy": (C.c_int, [vp]),
        "gr_items_create": (C.c_int, [C.c_int, vp, i64, i32, C.c_int, vp]),
        "gr_items_destroy": (C.c_int, [vp]),
        "gr_score_pairs": (C.c_int, [vp, vp, vp, i64, vp, vp, i64, vp, C.c_int, vp]),
        "gr_score_items_approx": (C.c_int, [vp, vp, vp, vp, i64, vp]),
        "gr_searcher_create": (C.c_int, [C.c_int, vp]),
        "gr_searcher_destroy": (C.c_int, [vp]),
        "gr_search": (C.c_int, [vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, C.c_int, vp]),
        "gr_search_async": (C.c_int, [vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp]),
        "gr_searcher_status": (C.c_int, [vp, vp]),
        "gr_searcher_launches": (i64, [vp]),
        "gr_searcher_counters": (C.c_int, [vp, vp]),
        "gr_brute_force": (C.c_int, [vp, vp, vp, i64, i32, vp, vp, C.c_int, vp]),
        "gr_merge_topk": (C.c_int, [C.c_int, vp, vp, i32, i64, i32, i32, vp, vp, vp, vp]),
        "gr_scores_create": (C.c_int, [C.c_int, vp, i64, i64, C.c_int, vp]),
        "gr_scores_euclid": (C.c_int, [C.c_int, vp, i64, i32, vp, i64, vp]),
        "gr_scores_read": (C.c_int, [vp, vp]),
        "gr_scores_destroy": (C.c_int, [vp]),
        "gr_search_scores": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, vp]),
        "gr_pack_topk": (C.c_int, [C.c_int, vp, vp, i64, vp, vp]),
        "gr_merge_topk_packed": (C.c_int, [C.c_int, vp, i32, i64, i32, i32, vp, vp, vp, vp]),
        "gr_hnsw_insert": (C.c_int, [i64, i64, i32, vp, vp, vp, i32, i32, i32, C.c_int, vp, vp,
                                     vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


def lib():
    """Load libgmpgr.so (never builds at import time on the product path)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise DeviceError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import "
                        f"__graft_entry__ as g; g.build()'` (nvcc, sm_100a); there is no CPU path")
                l = C.CDLL(LIB_PATH)
                _declare(l)
                _lib = l
    return _lib


def check(rc: int):
    if rc == GR_OK:
        return
    msg = lib().gr_last_error().decode(errors="replace")
    if rc == GR_EINVAL:
        raise InvalidArgumentError(msg)
    if rc == GR_ENUMERIC:
        raise NumericError(msg)
    if rc == GR_EBAND:
        raise BandError(msg)
    if rc == GR_ENOMEM:
        raise MemoryError(msg)
    raise DeviceError(msg)


def require_device():
    if lib().gr_device_count() < 1:
        raise DeviceError("no CUDA device visible: the GMP-GR hot path runs only on the GPU")


def current_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover - torch is plumbing only
        pass
    return 0


def ptr(a) -> int:
    """Address of a numpy array or torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def ptr_array(arrs):
    return (C.c_void_p * len(arrs))(*[ptr(a) for a in arrs])


class _Handle:
    _destroy = None

    def __init__(self, h: C.c_void_p, device: int):
        self.h = h
        self.device = device

    def __del__(self):
        try:
            if self.h and self._destroy:
                getattr(lib(), self._destroy)(self.h)
                self.h = None
        except Exception:
            pass


class DeviceModel(_Handle):
    """gr_model: metric MLP in processing order (metric.py:74-99)."""
    _destroy = "gr_model_destroy"

    def __init__(self, layers, attention, relu: bool, device: int | None = None):
        require_device()
        device = current_device() if device is None else device
        self.W = [np.ascontiguousarray(np.asarray(w).astype(np.float32)) for w, _ in layers]
        self.b = [np.ascontiguousarray(np.asarray(b).astype(np.float32)) for _, b in layers]
        self.A = np.ascontiguousarray(np.asarray(attention).astype(np.float32))
        dims = [self.W[0].shape[1]] + [w.shape[0] for w in self.W]
        for m, w in enumerate(self.W):
            if w.shape != (dims[m + 1], dims[m]) or self.b[m].shape != (dims[m + 1],):
                raise InvalidArgumentError(f"layer {m}: inconsistent weight shapes")
        if self.A.shape != (dims[-1],):
            raise InvalidArgumentError("attention length != z_dim")
        self.dims = np.asarray(dims, dtype=np.int32)
        self.d_h = dims[0] // 2
        h = C.c_void_p()
        check(lib().gr_model_create(device, len(self.W), ptr(self.dims), ptr_array(self.W),
                                    ptr_array(self.b), ptr(self.A), int(bool(relu)), C.byref(h)))
        super().__init__(h, device)


class DeviceGraph(_Handle):
    """gr_graph: device layout of GraphIndex.graph_view() (index.py:384-391)."""
    _destroy = "gr_graph_destroy"

    def __init__(self, layers, levels, entry_slot, ids, rows=None, device: int | None = None,
                 order=None):
        require_device()
        device = current_device() if device is None else device
        n = len(ids)
        nbrs = [np.ascontiguousarray(nb[:n], dtype=np.int32) for nb, _ in layers]
        cnts = [np.ascontiguousarray(ct[:n], dtype=np.int32) for _, ct in layers]
        stride = np.asarray([nb.shape[1] for nb in nbrs], dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        levels = None if levels is None else np.ascontiguousarray(levels[:n], dtype=np.int32)
        rows = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
        self.n = n
        self.n_layers = len(layers)
        order = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
        if order is not None and order.shape != (n,):
            raise InvalidArgumentError("order must list every slot once")
        h = C.c_void_p()
        check(lib().gr_graph_create_ordered(device, len(layers), n, ptr_array(nbrs), ptr(stride),
                                            ptr_array(cnts), ptr(levels), int(entry_slot), ptr(ids),
                                            ptr(rows), ptr(order), C.byref(h)))
        super().__init__(h, device)


class DeviceItems(_Handle):
    """gr_items: fp32 item embeddings (model_scorer's item_embeddings, search.py:84-90)."""
    _destroy = "gr_items_destroy"

    def __init__(self, emb, device: int | None = None):
        require_device()
        device = current_device() if device is None else device
        on_dev = not isinstance(emb, np.ndarray)
        if not on_dev:
            emb = np.ascontiguousarray(emb, dtype=np.float32)
        else:
            emb = emb.contiguous()
        if emb.ndim != 2:
            raise InvalidArgumentError("item embeddings must be (n, d)")
        self.n, self.d = int(emb.shape[0]), int(emb.shape[1])
        h = C.c_void_p()
        check(lib().gr_items_create(device, ptr(emb), self.n, self.d, int(on_dev), C.byref(h)))
        super().__init__(h, device)


class DeviceScores(_Handle):
    """gr_scores: traversal-only fp64 score table [Q, n_items] by item id (test scorers)."""
    _destroy = "gr_scores_destroy"

    def __init__(self, table=None, *, vectors=None, queries=None, device: int | None = None):
        require_device()
        device = current_device() if device is None else device
        h = C.c_void_p()
        if table is not None:
            table = np.ascontiguousarray(np.atleast_2d(table), dtype=np.float64)
            self.Q, self.n = table.shape
            check(lib().gr_scores_create(device, ptr(table), self.Q, self.n, 0, C.byref(h)))
        else:
            vectors = np.ascontiguousarray(vectors, dtype=np.float64)
            if vectors.ndim == 1:
                vectors = vectors[:, None]
            queries = np.ascontiguousarray(queries, dtype=np.float64).reshape(-1, vectors.shape[1])
            self.Q, self.n = queries.shape[0], vectors.shape[0]
            check(lib().gr_scores_euclid(device, ptr(vectors), self.n, vectors.shape[1],
                                         ptr(queries), self.Q, C.byref(h)))
        super().__init__(h, device)

    def read(self) -> np.ndarray:
        out = np.empty((self.Q, self.n), dtype=np.float64)
        check(lib().gr_scores_read(self.h, ptr(out)))
        return out


class DeviceSearcher(_Handle):
    """gr_searcher: per-stream scratch for gr_search."""
    _destroy = "gr_searcher_destroy"

    def __init__(self, device: int | None = None):
        require_device()
        device = current_device() if device is None else device
        h = C.c_void_p()
        check(lib().gr_searcher_create(device, C.byref(h)))
        super().__init__(h, device)

    @property
    def launches(self) -> int:
        return int(lib().gr_searcher_launches(self.h))

    def counters(self) -> dict:
        out = np.zeros(22, dtype=np.int64)
        check(lib().gr_searcher_counters(self.h, ptr(out)))
        d = {"exact_rescored": int(out[0]), "tensor_scored": int(out[1]),
             "band_violations": int(out[18]),
             "max_err_over_band": float(np.array([out[19]], dtype=np.uint32).view(np.float32)[0]),
             "exact_reruns": int(out[20]), "resident_units": int(out[21])}
        if out[2:10].any():
            names = ("init", "seeds", "expand", "resolve", "score", "pool", "frontier", "output")
            tot = float(out[2:10].sum())
            d["phase_share"] = {k: round(float(v) / tot, 4) for k, v in zip(names, out[2:10])}
            if out[10:18].any():
                sub = ("e_epi0", "e_epi1", "e_d0full_wait", "e_d1full_wait", "e_total",
                       "is_idle", "is_issuing", "ld_empty_wait")
                d["pipe_share"] = {k: round(float(v) / tot, 4) for k, v in zip(sub, out[10:18])}
            elif out[10:15].any():
                sub = ("tc_gather", "tc_mma0", "tc_epi0", "tc_mma1", "tc_epi1")
                d["score_sub_share"] = {k: round(float(v) / tot, 4) for k, v in zip(sub, out[10:15])}
        return d
