"""Synthetic workloads of the BASELINE.json shapes (bench.py, scaling runs).

Same recipe as the reference's benchmark inputs: clustered item
features (``nann.bench.clustered_vectors``: centres N(0, 4^2), unit noise,
bench.py:24-28) projected by ``create_model(d, d, Z, (64, 64), seed=1)``'s item tower,
user embeddings from the user tower over N(0, 1) features, graph over the item
embeddings with degree cap 2m.  At 10M items the generation runs on the GPU with
torch (seeded) — identical bytes on every rank — instead of numpy.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .index import GraphIndex
from .metric import RelevanceModel, create_model

CONFIGS = {
    # name: (n_items, d, m, n_clusters, Z, queries per GPU)
    "cfg1": (100_000, 64, 16, 256, 2, 1_000),
    "cfg2": (1_000_000, 128, 16, 1024, 3, 10_000),
    "cfg3": (10_000_000, 128, 24, 4096, 3, 65_536),
    "small": (200_000, 128, 24, 512, 3, 8_192),
}


@dataclass
class Workload:
    name: str
    model: RelevanceModel
    items: "object"        # torch fp32 [N, d] on the device
    items_host: np.ndarray | None
    users: np.ndarray      # fp32 [Q, d] (host)
    index: GraphIndex
    build_s: float


def clustered_vectors(n: int, d: int, n_clusters: int, seed: int) -> np.ndarray:
    """The reference's synthetic item features (nann/bench.py:24-28), same numpy stream."""
    rng = np.random.default_rng(seed)
    centers = rng.normal(scale=4.0, size=(n_clusters, d))
    assign = rng.integers(0, n_clusters, size=n)
    return centers[assign] + rng.normal(size=(n, d))


def reference_inputs(name: str, n_queries: int | None = None):
    """(model, item embeddings, user embeddings) of BASELINE config 1/2 exactly as the
    reference recipe makes them: create_model(d, d, Z, (64, 64), seed=1),
    items = item_embeddings(clustered_vectors(N, d, C, seed=0) as fp32), users =
    user_embedding(default_rng(7).normal(size=(Q, d)) as fp32).  Bit-identical to the
    reference's arrays (digests in tests/golden/cfg*_ref.npz)."""
    N, d, m, C, Z, Q = CONFIGS[name]
    model = create_model(d_x=d, d_h=d, z_dim=Z, hidden=(64, 64), seed=1)
    emb = model.item_embeddings(clustered_vectors(N, d, C, seed=0).astype(np.float32))
    users = model.user_embedding(
        np.random.default_rng(7).normal(size=(n_queries or Q, d)).astype(np.float32))
    return model, np.ascontiguousarray(emb), np.ascontiguousarray(users)


def graph_digest(index: GraphIndex) -> str:
    """sha256 over ids, levels, entry and every layer's rows in stored order (the same
    digest tests/golden/make_cfg_golden.py records for the reference's build)."""
    import hashlib

    ids, levels, layers, entry = index.graph_view()
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(ids, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(levels, dtype="<i4").tobytes())
    h.update(np.int64(entry).tobytes())
    n = len(ids)
    for nb, ct in layers:
        ct = np.asarray(ct[:n], dtype="<i4")
        h.update(ct.tobytes())
        mask = np.arange(nb.shape[1])[None, :] < ct[:, None]
        h.update(np.asarray(nb[:n], dtype="<i4")[mask].tobytes())
    return h.hexdigest()


def make_reference(name: str, device: int | None = 0, n_queries: int | None = None) -> Workload:
    """Config 1/2 on the reference's own inputs and graph: the index is the native exact
    build (GraphIndex.build, identical to nann.GraphIndex.build(m=16, ef_construction=64,
    seed=0)); items stay on the host too (CPU restatement / fixtures); device=None keeps
    everything on the host (the reference arm)."""
    import torch

    t0 = time.perf_counter()
    N, d, m, C, Z, Q = CONFIGS[name]
    model, emb, users = reference_inputs(name, n_queries)
    index = GraphIndex.build(emb.astype(np.float64), m=m, ef_construction=64, seed=0)
    items = emb if device is None else torch.from_numpy(emb).to(torch.device("cuda", device))
    return Workload(name, model, items, emb, users, index, time.perf_counter() - t0)


def make(name: str, rank: int = 0, device: int = 0, host_items: bool = False,
         n_queries: int | None = None, n_items: int | None = None, graph: str = "gpu") -> Workload:
    """Synthetic workload of a BASELINE shape.  graph="gpu": bulk GPU producer (builder.py);
    graph="exact": the reference's own sequential construction algorithm (native exact
    parallel build, GraphIndex.build(method="exact"), m and ef_construction=64 as the
    reference defaults) over the same items."""
    import torch

    N, d, m, C, Z, Q = CONFIGS[name]
    N = n_items or N
    Q = n_queries or Q
    t0 = time.perf_counter()
    dev = torch.device("cuda", device)
    model = create_model(d_x=d, d_h=d, z_dim=Z, hidden=(64, 64), seed=1)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    centers = torch.randn(C, d, generator=g, device=dev) * 4.0
    assign = torch.randint(0, C, (N,), generator=g, device=dev)
    w_item = torch.from_numpy(model.item_projector.weight.astype(np.float32)).to(dev)
    items = torch.empty((N, d), dtype=torch.float32, device=dev)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    for s in range(0, N, 1 << 20):
        e = min(N, s + (1 << 20))
        feats = centers[assign[s:e]] + torch.randn(e - s, d, generator=g, device=dev)
        items[s:e] = feats @ w_item
    gu = torch.Generator(device=dev)
    gu.manual_seed(7 + 1000 * rank)
    w_user = torch.from_numpy(model.user_projector.weight.astype(np.float32)).to(dev)
    users = (torch.randn(Q, d, generator=gu, device=dev) @ w_user).cpu().numpy()
    torch.backends.cuda.matmul.allow_tf32 = prev
    del centers, assign
    if graph == "exact":
        index = exact_graph(name, items, m, rank)
    elif graph == "random":  # memory/scale tests only: random fixed-degree layers, no quality
        from .builder import draw_levels

        levels = draw_levels(N, 1.0 / 17.0, 4, 0)
        rng = np.random.default_rng(0)
        layers = []
        for l in range(int(levels.max()) + 1):
            cap = 2 * m if l == 0 else m
            members = np.nonzero(levels >= l)[0]
            nb = np.zeros((N, cap), dtype=np.int32)
            ct = np.zeros(N, dtype=np.int32)
            if len(members) > 1:
                nb[members] = members[rng.integers(0, len(members), size=(len(members), cap))]
                ct[members] = cap
            layers.append((nb, ct))
        index = GraphIndex.from_arrays(np.arange(N, dtype=np.int64), levels, layers,
                                       int(np.argmax(levels)), m=m, max_layers=4)
    else:
        index = GraphIndex.build(items, m=m, seed=0, device=dev, method="gpu")
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()  # hand the builder's cached blocks back before the search scratch
    items_host = items.cpu().numpy() if host_items else None
    return Workload(name, model, items, items_host, np.ascontiguousarray(users, np.float32), index,
                    time.perf_counter() - t0)


def exact_graph(name: str, items, m: int, rank: int = 0) -> GraphIndex:
    """GraphIndex.build(items, m, ef_construction=64, seed=0) -- the reference's own
    construction algorithm (native exact parallel build) -- cached on local disk
    (GMPGR_CACHE, default /tmp/gmpgr_cache) keyed by the items' digest, so the ranks of one
    box and the benchmark's two arms build it once: rank 0 builds, the others wait for the
    file."""
    import hashlib
    import os

    N, d = items.shape
    probe = items[:: max(1, N // 8192)].double().cpu().numpy()
    key = hashlib.sha256(probe.tobytes()).hexdigest()[:16]
    cache = os.environ.get("GMPGR_CACHE", "/tmp/gmpgr_cache")
    path = os.path.join(cache, f"{name}_{N}x{d}_m{m}_ef64_{key}_v2.npz")
    failed = path + ".failed"
    if not os.path.exists(path):
        if rank == 0:
            if os.path.exists(failed):  # a marker left by an earlier run
                os.remove(failed)
            index = GraphIndex.build(items.double().cpu().numpy(), m=m, ef_construction=64, seed=0)
            ids, levels, layers, entry = index.graph_view()
            try:
                os.makedirs(cache, exist_ok=True)
                arrs = {"ids": ids, "levels": levels, "entry": np.int64(entry), "m": np.int64(index.m),
                        "max_layers": np.int64(index.max_layers)}
                for l, (nb, ct) in enumerate(layers):  # upper layers: member rows only
                    rows = np.arange(N) if l == 0 else np.nonzero(levels[:N] >= l)[0]
                    arrs[f"rows{l}"], arrs[f"nb{l}"], arrs[f"ct{l}"] = rows, nb[rows], ct[rows]
                tmp = path + f".tmp{os.getpid()}.npz"
                np.savez(tmp, **arrs)
                os.replace(tmp, path)
            except OSError:  # no room for the cache: the other ranks build their own copy
                try:
                    open(failed, "w").close()
                except OSError:
                    pass
            return index
        t0 = time.time()
        while not os.path.exists(path):
            if os.path.exists(failed) or time.time() - t0 > 3600:
                return GraphIndex.build(items.double().cpu().numpy(), m=m, ef_construction=64, seed=0)
            time.sleep(2.0)
    z = np.load(path)
    nl = sum(1 for f in z.files if f.startswith("nb"))
    layers = []
    for l in range(nl):
        rows, nbm, ctm = z[f"rows{l}"], z[f"nb{l}"], z[f"ct{l}"]
        nb = np.zeros((N, nbm.shape[1]), dtype=np.int32)
        ct = np.zeros(N, dtype=np.int32)
        nb[rows], ct[rows] = nbm, ctm
        layers.append((nb, ct))
    return GraphIndex.from_arrays(z["ids"], z["levels"], layers, int(z["entry"]), m=int(z["m"]),
                                  max_layers=int(z["max_layers"]))


def make_shard(rank: int, world: int, shard_n: int = 12_500_000, d: int = 128, m: int = 24,
               Z: int = 3, n_queries: int = 65_536, device: int = 0) -> Workload:
    """BASELINE config 4: a catalog of shard_n * world items split in contiguous global-id
    ranges; this rank's shard is an independent graph over items [rank*shard_n, ...) with
    GLOBAL ids (slot order = id order) and local embedding rows.  Cluster centres and users
    are shared by all ranks; per-shard items come from a rank-seeded stream."""
    import torch

    t0 = time.perf_counter()
    dev = torch.device("cuda", device)
    model = create_model(d_x=d, d_h=d, z_dim=Z, hidden=(64, 64), seed=1)
    C = 4096  # n_clusters 4096 for configs 3 and 4
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    centers = torch.randn(C, d, generator=g, device=dev) * 4.0
    gs = torch.Generator(device=dev)
    gs.manual_seed(1_000_003 * (rank + 1))
    assign = torch.randint(0, C, (shard_n,), generator=gs, device=dev)
    w_item = torch.from_numpy(model.item_projector.weight.astype(np.float32)).to(dev)
    items = torch.empty((shard_n, d), dtype=torch.float32, device=dev)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    for s0 in range(0, shard_n, 1 << 20):
        e = min(shard_n, s0 + (1 << 20))
        items[s0:e] = (centers[assign[s0:e]] + torch.randn(e - s0, d, generator=gs, device=dev)) @ w_item
    gu = torch.Generator(device=dev)
    gu.manual_seed(7)
    w_user = torch.from_numpy(model.user_projector.weight.astype(np.float32)).to(dev)
    users = (torch.randn(n_queries, d, generator=gu, device=dev) @ w_user).cpu().numpy()
    torch.backends.cuda.matmul.allow_tf32 = prev
    del centers, assign
    lo = rank * shard_n
    index = GraphIndex.build(items, ids=np.arange(lo, lo + shard_n, dtype=np.int64), m=m,
                             seed=rank, device=dev, method="gpu")
    index.rows = np.arange(shard_n, dtype=np.int32)
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    return Workload("cfg4", model, items, None, np.ascontiguousarray(users, np.float32), index,
                    time.perf_counter() - t0)
