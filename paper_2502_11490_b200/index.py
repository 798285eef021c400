"""Layered item graph: NANN-IDX persistence, searcher views, device upload.

Mirror of ``nann.index.GraphIndex`` (/root/reference/pkg/src/nann/index.py:30-508) on
the read side the hot path consumes: same storage (per-layer fixed-width int32 rows of
cap 2m / m plus counts, index.py:67-85), same ``graph_view()`` (index.py:384-391), same
NANN-IDX format (index.py:24-27, 397-508), same ``validate()`` invariants
(index.py:325-358).  ``build``/``insert`` default to the native exact restatement of the
reference's sequential insert (csrc/hnsw_build.cpp, ``gr_hnsw_insert``): the graph is
identical node for node to ``nann.GraphIndex.build``.  ``build(method="gpu")`` is the
bulk GPU producer (builder.py) for catalogs the sequential build cannot reach in
minutes (10M+).  Stream admission (index.py:511-592) is outside the hot path.
"""

from __future__ import annotations

import struct

import numpy as np

from . import _lib
from .errors import FileFormatError, InvalidArgumentError

INDEX_MAGIC = b"NANN-IDX"
INDEX_VERSION = 1
_HEAD_FMT = "<IIIIdBqQIIq"  # version, L, m, efc, p, heuristic, seed, ordinal, n, dim, entry
LOCALITY_MIN = 1 << 16  # slots below this: breadth-first device order (fits caches anyway)


class GraphIndex:
    """L-layer navigable graph with symmetric adjacency and capped degrees."""

    def __init__(self, dim: int, m: int = 16, ef_construction: int = 64,
                 level_prob: float = 1.0 / 17.0, max_layers: int = 4, seed: int = 0,
                 select_heuristic: bool = False, kernel_backend: str | None = None):
        if dim < 1:
            raise InvalidArgumentError("dim must be >= 1")
        if m < 2:
            raise InvalidArgumentError("m must be >= 2")
        if ef_construction < 1:
            raise InvalidArgumentError("ef_construction must be >= 1")
        if not 0.0 < level_prob < 1.0:
            raise InvalidArgumentError("level_prob must be in (0, 1)")
        if max_layers < 1:
            raise InvalidArgumentError("max_layers must be >= 1")
        self.dim, self.m, self.ef_construction = dim, m, ef_construction
        self.level_prob, self.max_layers, self.seed = level_prob, max_layers, seed
        self.select_heuristic = select_heuristic
        self._n = 0
        self._entry_slot = -1
        self._top_level = -1
        self._level_draws = 0
        self._vectors = np.empty((0, dim), dtype=np.float64)
        self._ids = np.empty(0, dtype=np.int64)
        self._levels = np.empty(0, dtype=np.int32)
        self._nbrs = [np.empty((0, self._deg_cap(l)), dtype=np.int32) for l in range(max_layers)]
        self._cnts = [np.empty(0, dtype=np.int32) for _ in range(max_layers)]
        self._slot_map = None
        self._dev = {}
        self._stamps = np.empty(0, dtype=np.int64)
        self._stamp = 0
        self._level_rng = None
        # embedding row per slot; None = the item id (model_scorer convention, search.py:88).
        # Catalog shards set it to the local row while ids stay global.
        self.rows = None

    def _deg_cap(self, layer: int) -> int:
        return 2 * self.m if layer == 0 else self.m

    # ---------------------------------------------------------------- introspection
    def __len__(self) -> int:
        return self._n

    @property
    def _slot_of(self) -> dict:
        if self._slot_map is None:
            self._slot_map = {int(i): s for s, i in enumerate(self._ids[: self._n])}
        return self._slot_map

    def __contains__(self, item_id: int) -> bool:
        return item_id in self._slot_of

    @property
    def entry_point(self):
        return None if self._entry_slot < 0 else int(self._ids[self._entry_slot])

    @property
    def n_layers(self) -> int:
        return self._top_level + 1

    def item_ids(self) -> np.ndarray:
        return self._ids[: self._n].copy()

    def vector(self, item_id: int) -> np.ndarray:
        return self._vectors[self._slot_of[item_id]].copy()

    def level_of(self, item_id: int) -> int:
        return int(self._levels[self._slot_of[item_id]])

    def layer_node_counts(self) -> list:
        lv = self._levels[: self._n]
        return [int((lv >= l).sum()) for l in range(self.n_layers)]

    def neighbors(self, layer: int, item_id: int) -> list:
        s = self._slot_of[item_id]
        return sorted(int(self._ids[t]) for t in self._nbrs[layer][s, : self._cnts[layer][s]])

    def graph_view(self):
        """(ids, levels, [(nbrs, cnts)] per populated layer, entry_slot) — index.py:384-391."""
        return (self._ids[: self._n], self._levels[: self._n],
                [(self._nbrs[l], self._cnts[l]) for l in range(self.n_layers)], self._entry_slot)

    # ---------------------------------------------------------------- construction
    @classmethod
    def from_arrays(cls, ids, levels, layers, entry_slot, vectors=None, m=None, **kw):
        """Wrap existing adjacency (e.g. another index's graph_view()) without rebuilding."""
        ids = np.asarray(ids, dtype=np.int64)
        n = len(ids)
        layers = [(np.asarray(nb), np.asarray(ct)) for nb, ct in layers]
        if m is None:
            m = max(2, layers[1][0].shape[1] if len(layers) > 1 else layers[0][0].shape[1] // 2)
        dim = 1 if vectors is None else np.asarray(vectors).shape[1]
        idx = cls(dim=dim, m=m, max_layers=max(len(layers), kw.pop("max_layers", 1)), **kw)
        idx._n = n
        idx._ids = ids.copy()
        idx._levels = np.asarray(levels, dtype=np.int32)[:n].copy()
        idx._vectors = (np.zeros((n, 1)) if vectors is None
                        else np.ascontiguousarray(vectors, dtype=np.float64)[:n])
        for l in range(idx.max_layers):
            cap = idx._deg_cap(l)
            nb = np.zeros((n, cap), dtype=np.int32)
            ct = np.zeros(n, dtype=np.int32)
            if l < len(layers):
                src_nb, src_ct = layers[l]
                w = min(cap, src_nb.shape[1])
                if int(np.max(src_ct[:n], initial=0)) > cap:
                    raise InvalidArgumentError(f"layer {l}: degree exceeds cap {cap}")
                nb[:, :w] = src_nb[:n, :w]
                ct[:] = src_ct[:n]
            idx._nbrs[l] = nb
            idx._cnts[l] = ct
        idx._entry_slot = int(entry_slot)
        idx._top_level = int(idx._levels.max()) if n else -1
        return idx

    @classmethod
    def build(cls, vectors, ids=None, m: int = 16, ef_construction: int = 64,
              level_prob: float = 1.0 / 17.0, max_layers: int = 4, seed: int = 0,
              select_heuristic: bool = False, kernel_backend: str | None = None,
              device=None, method: str = "exact") -> "GraphIndex":
        """Index a batch of vectors.

        ``method="exact"`` (default): iterated :meth:`insert` through the native
        restatement of the reference build (index.py:160-194) -- same graph as
        ``nann.GraphIndex.build`` for the same arguments.  ``method="gpu"``: the bulk
        GPU producer (builder.py; reference level draws and entry point, k-NN edges).
        """
        if method == "exact":
            vec = np.ascontiguousarray(np.asarray(vectors), dtype=np.float64)
            if vec.ndim != 2 or vec.shape[0] < 1:
                raise InvalidArgumentError("vectors must be a nonempty (n, d) array")
            n = vec.shape[0]
            ids = np.arange(n, dtype=np.int64) if ids is None else np.asarray(ids, dtype=np.int64)
            if len(ids) != n:
                raise InvalidArgumentError("ids and vectors differ in length")
            if len(np.unique(ids)) != len(ids):
                raise InvalidArgumentError("duplicate item ids")
            idx = cls(dim=vec.shape[1], m=m, ef_construction=ef_construction,
                      level_prob=level_prob, max_layers=max_layers, seed=seed,
                      select_heuristic=select_heuristic, kernel_backend=kernel_backend)
            idx._insert_batch(ids, vec)
            return idx
        if method != "gpu":
            raise InvalidArgumentError(f"unknown build method {method!r}")
        from .builder import build_layers

        vec = vectors if not isinstance(vectors, np.ndarray) else np.ascontiguousarray(
            vectors, dtype=np.float64)
        if vec.ndim != 2 or vec.shape[0] < 1:
            raise InvalidArgumentError("vectors must be a nonempty (n, d) array")
        n = vec.shape[0]
        ids = np.arange(n, dtype=np.int64) if ids is None else np.asarray(ids, dtype=np.int64)
        if len(np.unique(ids)) != len(ids):
            raise InvalidArgumentError("duplicate item ids")
        g = build_layers(vec, m=m, level_prob=level_prob, max_layers=max_layers, seed=seed,
                         device=device)
        host_vec = vec if isinstance(vec, np.ndarray) else None
        idx = cls.from_arrays(ids, g["levels"], list(zip(g["nbrs"], g["cnts"])),
                              g["entry_slot"], vectors=host_vec, m=m, max_layers=max_layers,
                              ef_construction=ef_construction, level_prob=level_prob, seed=seed,
                              select_heuristic=select_heuristic)
        if host_vec is None:
            idx.dim = vec.shape[1]
        idx._level_draws = n
        return idx

    # ---------------------------------------------------------------- exact insert
    def _reserve(self, n: int) -> None:
        """Grow the slot arrays (index.py:91-116; same doubling, zero fill)."""
        cap = len(self._ids)
        if n <= cap and len(self._stamps) >= cap:
            return
        cap = max(n, 2 * cap, 16)
        k = self._n
        def grow(a, shape, dtype):
            new = np.zeros(shape, dtype=dtype)
            c = min(k, len(a))  # loaded / wrapped indexes carry no stamps
            new[:c] = a[:c]
            return new
        self._vectors = grow(self._vectors, (cap, self.dim), np.float64)
        self._ids = grow(self._ids, cap, np.int64)
        self._levels = grow(self._levels, cap, np.int32)
        self._stamps = grow(self._stamps, cap, np.int64)
        for l in range(self.max_layers):
            self._nbrs[l] = grow(self._nbrs[l], (cap, self._deg_cap(l)), np.int32)
            self._cnts[l] = grow(self._cnts[l], cap, np.int32)

    def _draw_levels(self, count: int) -> np.ndarray:
        """Next ``count`` levels of the persistent level stream (index.py:196-209): one
        uniform per insert from default_rng(seed), replayed to ``_level_draws``."""
        if self._level_rng is None:
            self._level_rng = np.random.default_rng(self.seed)
            if self._level_draws:
                self._level_rng.random(self._level_draws)
        u = self._level_rng.random(count)
        self._level_draws += count
        with np.errstate(divide="ignore"):
            lv = np.log(u) / np.log(self.level_prob)
        top = self.max_layers - 1
        return np.where(u <= 0.0, top, np.minimum(np.trunc(lv), top)).astype(np.int32)

    def _insert_batch(self, ids: np.ndarray, vectors: np.ndarray) -> None:
        ids = np.asarray(ids, dtype=np.int64)
        vectors = np.ascontiguousarray(vectors, dtype=np.float64).reshape(len(ids), self.dim)
        if self._n:
            present = self._slot_of
            for i in ids:
                if int(i) in present:
                    raise InvalidArgumentError(f"item id {int(i)} already present")
        n0, n1 = self._n, self._n + len(ids)
        self._reserve(n1)
        self._vectors[n0:n1] = vectors
        self._ids[n0:n1] = ids
        self._levels[n0:n1] = self._draw_levels(len(ids))
        stamp = np.array([self._stamp], dtype=np.int64)
        entry = np.array([self._entry_slot], dtype=np.int32)
        top = np.array([self._top_level], dtype=np.int32)
        _lib.check(_lib.lib().gr_hnsw_insert(
            n0, n1, self.dim, _lib.ptr(self._vectors), _lib.ptr(self._ids), _lib.ptr(self._levels),
            self.m, self.ef_construction, self.max_layers, int(bool(self.select_heuristic)),
            _lib.ptr_array(self._nbrs), _lib.ptr_array(self._cnts), _lib.ptr(self._stamps),
            _lib.ptr(stamp), _lib.ptr(entry), _lib.ptr(top)))
        self._n = n1
        self._stamp = int(stamp[0])
        self._entry_slot, self._top_level = int(entry[0]), int(top[0])
        if self._slot_map is not None:
            self._slot_map.update((int(i), n0 + j) for j, i in enumerate(ids))
        self._dev = {}

    def insert(self, item_id: int, vector) -> None:
        """Add one item (index.py:283-319), exact native restatement; invariants hold on return."""
        vector = np.asarray(vector, dtype=np.float64)
        if vector.shape != (self.dim,):
            raise InvalidArgumentError(f"vector shape {vector.shape} != ({self.dim},)")
        self._insert_batch(np.array([item_id], dtype=np.int64), vector[None, :])

    # ---------------------------------------------------------------- invariants
    def validate(self) -> None:
        """Vectorised sweep of the reference invariants (index.py:325-358)."""
        n = self._n
        if n == 0:
            return
        lv = self._levels[:n]
        if self._entry_slot < 0:
            raise AssertionError("nonempty index without entry point")
        if lv[self._entry_slot] != self._top_level:
            raise AssertionError("entry point is not on the top layer")
        if int(lv.max()) != self._top_level:
            raise AssertionError("top level out of sync with node levels")
        for l in range(self.n_layers):
            cap = self._deg_cap(l)
            member = lv >= l
            ct = self._cnts[l][:n]
            if (ct[member] > cap).any():
                raise AssertionError(f"layer {l}: degree > {cap}")
            s = np.repeat(np.nonzero(member)[0], ct[member])
            nb = self._nbrs[l][:n]
            mask = np.arange(nb.shape[1])[None, :] < ct[:, None]
            mask &= member[:, None]
            t = nb[mask].astype(np.int64)
            if len(t) == 0:
                continue
            if (t == s).any():
                raise AssertionError(f"layer {l}: self loop")
            if not member[t].all():
                raise AssertionError(f"layer {l}: neighbor not on layer (nesting)")
            fwd = s * n + t
            if len(np.unique(fwd)) != len(fwd):
                raise AssertionError(f"layer {l}: duplicate neighbor")
            if not np.array_equal(np.sort(fwd), np.sort(t * n + s)):
                raise AssertionError(f"layer {l}: missing reverse edge")

    # ---------------------------------------------------------------- persistence
    def save(self, path: str) -> None:
        """NANN-IDX v1 writer (index.py:397-429)."""
        n = self._n
        with open(path, "wb") as f:
            f.write(INDEX_MAGIC)
            f.write(struct.pack(_HEAD_FMT, INDEX_VERSION, self.max_layers, self.m,
                                self.ef_construction, self.level_prob,
                                1 if self.select_heuristic else 0, self.seed, self._level_draws,
                                n, self.dim, self._entry_slot))
            f.write(self._ids[:n].astype("<i8").tobytes())
            f.write(self._levels[:n].astype("<i4").tobytes())
            vec = self._vectors[:n]
            if vec.shape != (n, self.dim):
                vec = np.zeros((n, self.dim))
            f.write(np.ascontiguousarray(vec, dtype="<f8").tobytes())
            for l in range(self.max_layers):
                ct = self._cnts[l][:n] if l < len(self._cnts) else np.zeros(n, np.int32)
                indptr = np.zeros(n + 1, dtype="<u8")
                indptr[1:] = np.cumsum(ct, dtype=np.uint64)
                f.write(indptr.tobytes())
                nb = self._nbrs[l][:n]
                mask = np.arange(nb.shape[1])[None, :] < ct[:, None]
                f.write(nb[mask].astype("<i4").tobytes())

    @classmethod
    def load(cls, path: str) -> "GraphIndex":
        """NANN-IDX v1 reader (index.py:431-508), same FileFormatError cases."""
        with open(path, "rb") as f:
            raw = f.read()
        if raw[: len(INDEX_MAGIC)] != INDEX_MAGIC:
            raise FileFormatError("not an index file (bad magic)", path=path)
        off = len(INDEX_MAGIC)
        hs = struct.calcsize(_HEAD_FMT)
        if len(raw) < off + hs:
            raise FileFormatError("truncated index header", path=path)
        (version, max_layers, m, efc, p, heur, seed, draws, n, dim,
         entry) = struct.unpack_from(_HEAD_FMT, raw, off)
        off += hs
        if version != INDEX_VERSION:
            raise FileFormatError(f"unsupported index version {version}", path=path)

        def take(dt, count):
            nonlocal off
            dt = np.dtype(dt)
            nb = dt.itemsize * count
            if len(raw) < off + nb:
                raise FileFormatError(f"truncated block at byte {off}", path=path)
            a = np.frombuffer(raw, dtype=dt, count=count, offset=off)
            off += nb
            return a

        ids = take("<i8", n).astype(np.int64)
        levels = take("<i4", n).astype(np.int32)
        vectors = take("<f8", n * dim).astype(np.float64).reshape(n, dim)
        idx = cls(dim=dim, m=m, ef_construction=efc, level_prob=p, max_layers=max_layers,
                  seed=seed, select_heuristic=bool(heur))
        idx._n, idx._ids, idx._levels, idx._vectors = n, ids, levels, vectors
        idx._level_draws, idx._entry_slot = draws, entry
        idx._top_level = int(levels.max()) if n else -1
        for l in range(max_layers):
            indptr = take("<u8", n + 1).astype(np.int64)
            total = int(indptr[-1]) if n else 0
            targets = take("<i4", total)
            cap = idx._deg_cap(l)
            ct = np.diff(indptr).astype(np.int64)
            if (ct > cap).any():
                s = int(np.argmax(ct > cap))
                raise FileFormatError(f"layer {l} slot {s}: degree {ct[s]} > cap {cap}", path=path)
            nb = np.zeros((n, cap), dtype=np.int32)
            rows = np.repeat(np.arange(n), ct)
            cols = np.arange(total) - np.repeat(indptr[:-1], ct)
            nb[rows, cols] = targets
            idx._nbrs[l] = nb
            idx._cnts[l] = ct.astype(np.int32)
        if off != len(raw):
            raise FileFormatError(f"{len(raw) - off} trailing bytes", path=path)
        return idx

    # ---------------------------------------------------------------- device
    def device_graph(self, device: int | None = None, items=None) -> _lib.DeviceGraph:
        """Cached gr_graph upload of graph_view() (invalidated by no mutation: read side only).

        With the item embeddings at hand (the search entry points pass them) and at least
        LOCALITY_MIN slots, device slots are grouped by embedding cluster (locality.py);
        otherwise breadth-first from the entry.  GMPGR_ORDER=bfs forces the latter."""
        import os

        device = _lib.current_device() if device is None else device
        h = self._dev.get(device)
        if h is None:
            if self._n == 0:
                raise InvalidArgumentError("index is empty")
            ids, levels, layers, entry = self.graph_view()
            order = None
            if (items is not None and self._n >= LOCALITY_MIN
                    and os.environ.get("GMPGR_ORDER", "cluster") != "bfs"):
                from .locality import cluster_order

                rows = self.rows if self.rows is not None else ids
                if int(np.max(rows)) < len(items):
                    order = cluster_order(items, slot_rows=rows, device=device)
            h = _lib.DeviceGraph(layers, levels, entry, ids, rows=self.rows, device=device, order=order)
            self._dev[device] = h
        return h
