"""GPU producer of NANN-IDX-valid layered graphs.

The reference builds by sequential HNSW-style insertion (index.py:160-319), ~1k
inserts/s on CPU, which cannot produce the 10M/100M graphs of BASELINE configs 3-4.
This producer keeps everything the search path consumes identical in *contract*:

* layer membership and entry point are the reference's exactly: one uniform draw
  per item from ``default_rng(seed)``, ``level = min(trunc(log u / log p), L-1)``
  (``u <= 0`` -> top), entry = first slot of the maximum level (index.py:196-209,
  302-319 — the sequential stream is a vectorised draw of the same numbers);
* degree caps 2m on layer 0 and m above (index.py:84-85), no self loops, no
  duplicates, every edge symmetric, neighbours on the same layer (nesting) — the
  ``GraphIndex.validate`` invariants (index.py:325-358).

Only the edge selection differs: each layer is a symmetrised approximate k-NN graph
(Euclidean on the item vectors, like the reference's construction metric) pruned so
an edge survives only if it is within the degree cap of BOTH endpoints' nearest
incident edges.  k-NN: exact blocked GEMM for small layers, an IVF partition (k-means
centroids, multi-probe) for large ones.  torch/cuBLAS does the GEMMs: this is input
preparation for the hot path, not the hot path.
"""

from __future__ import annotations

import math

import numpy as np


def draw_levels(n: int, level_prob: float, max_layers: int, seed: int) -> np.ndarray:
    u = np.random.default_rng(seed).random(n)
    with np.errstate(divide="ignore"):
        lv = np.log(u) / np.log(level_prob)
    lv = np.where(u <= 0.0, max_layers - 1, np.minimum(np.trunc(lv), max_layers - 1))
    return lv.astype(np.int32)


def _torch():
    import torch
    return torch


def _sqnorm(x):
    return (x * x).sum(1)


def knn_exact(x, K: int, block: int = 8192):
    """Exact K nearest (excluding self) by blocked GEMM; returns (idx int64, d2 fp32)."""
    torch = _torch()
    M = x.shape[0]
    K = min(K, M - 1)
    nx = _sqnorm(x)
    idx = torch.empty((M, K), dtype=torch.int64, device=x.device)
    dd = torch.empty((M, K), dtype=torch.float32, device=x.device)
    ar = torch.arange(M, device=x.device)
    for s in range(0, M, block):
        e = min(M, s + block)
        d2 = nx[s:e, None] + nx[None, :] - 2.0 * (x[s:e] @ x.T)
        d2[torch.arange(e - s, device=x.device), ar[s:e]] = float("inf")
        v, i = torch.topk(d2, K, dim=1, largest=False)
        idx[s:e] = i
        dd[s:e] = v
    return idx, dd


def _kmeans(x, C: int, iters: int, seed: int):
    torch = _torch()
    g = torch.Generator(device=x.device)
    g.manual_seed(seed)
    M = x.shape[0]
    samp = x[torch.randperm(M, generator=g, device=x.device)[: min(M, 64 * C)]]
    cent = samp[torch.randperm(samp.shape[0], generator=g, device=x.device)[:C]].clone()
    for _ in range(iters):
        a = _assign(samp, cent, 1)[:, 0]
        s = torch.zeros_like(cent).index_add_(0, a, samp)
        c = torch.bincount(a, minlength=C).clamp_min(1).to(x.dtype)
        cent = s / c[:, None]
    return cent


def _assign(x, cent, P: int, block: int = 65536):
    torch = _torch()
    nc = _sqnorm(cent)
    out = torch.empty((x.shape[0], P), dtype=torch.int64, device=x.device)
    for s in range(0, x.shape[0], block):
        d2 = nc[None, :] - 2.0 * (x[s:s + block] @ cent.T)
        out[s:s + block] = torch.topk(d2, P, dim=1, largest=False).indices
    return out


def knn_ivf(x, K: int, seed: int = 0, probes: int = 3):
    """Approximate K-NN: k-means partition, each point searches its `probes` nearest cells."""
    torch = _torch()
    M, dev = x.shape[0], x.device
    C = max(16, int(2 ** round(math.log2(max(16.0, math.sqrt(M) * 1.3)))))
    cent = _kmeans(x, C, iters=6, seed=seed)
    probe = _assign(x, cent, probes)            # [M, P]
    prim = probe[:, 0]
    order = torch.argsort(prim)
    counts = torch.bincount(prim, minlength=C)
    starts = torch.cumsum(counts, 0) - counts
    qcell = probe.reshape(-1)                   # (point, probe) pairs
    qorder = torch.argsort(qcell)
    qcounts = torch.bincount(qcell, minlength=C)
    qstarts = torch.cumsum(qcounts, 0) - qcounts
    cand_i = torch.full((M * probes, K), -1, dtype=torch.int64, device=dev)
    cand_d = torch.full((M * probes, K), float("inf"), dtype=torch.float32, device=dev)
    nx = _sqnorm(x)
    counts_h, starts_h = counts.tolist(), starts.tolist()
    qcounts_h, qstarts_h = qcounts.tolist(), qstarts.tolist()
    for c in range(C):
        nm, nq = counts_h[c], qcounts_h[c]
        if nm == 0 or nq == 0:
            continue
        mem = order[starts_h[c]:starts_h[c] + nm]
        qp = qorder[qstarts_h[c]:qstarts_h[c] + nq]  # flat (point*P + probe) indices
        qpt = qp // probes
        for s in range(0, nq, 16384):
            qs = qpt[s:s + 16384]
            d2 = nx[qs, None] + nx[None, mem] - 2.0 * (x[qs] @ x[mem].T)
            d2[qs[:, None] == mem[None, :]] = float("inf")
            kk = min(K, nm)
            v, i = torch.topk(d2, kk, dim=1, largest=False)
            cand_i[qp[s:s + 16384], :kk] = mem[i]
            cand_d[qp[s:s + 16384], :kk] = v
    cand_i = cand_i.view(M, probes * K)
    cand_d = cand_d.view(M, probes * K)
    v, j = torch.topk(cand_d, K, dim=1, largest=False)
    return torch.gather(cand_i, 1, j), v


def knn_backward_exact(x, K: int, block: int = 4096):
    """K nearest among EARLIER members (j < i): the neighbours an HNSW insertion in slot
    order would see (index.py:283-319 inserts in id order and links the new node to its
    nearest already-inserted nodes, keep-M selection index.py:226-239)."""
    torch = _torch()
    M = x.shape[0]
    nx = _sqnorm(x)
    idx = torch.full((M, K), -1, dtype=torch.int64, device=x.device)
    dd = torch.full((M, K), float("inf"), dtype=torch.float32, device=x.device)
    for s in range(1, M, block):
        e = min(M, s + block)
        d2 = nx[s:e, None] + nx[None, :e] - 2.0 * (x[s:e] @ x[:e].T)
        mask = torch.arange(e, device=x.device)[None, :] >= torch.arange(s, e, device=x.device)[:, None]
        d2 = d2.masked_fill(mask, float("inf"))
        kk = min(K, e)
        v, i = torch.topk(d2, kk, dim=1, largest=False)
        i = torch.where(torch.isfinite(v), i, torch.full_like(i, -1))
        idx[s:e, :kk] = i
        dd[s:e, :kk] = v
    return idx, dd


def knn_backward_ivf(x, K: int, seed: int = 0, probes: int = 4, exact_prefix: int = 131072):
    """Backward K-NN at scale: exact for the first `exact_prefix` nodes, then geometric
    stages [P, 2P) whose IVF index covers only the prefix [0, 2P) (so at least half of every
    cell is eligible), masked to j < i."""
    torch = _torch()
    M, dev = x.shape[0], x.device
    P0 = min(M, exact_prefix)
    idx = torch.full((M, K), -1, dtype=torch.int64, device=dev)
    dd = torch.full((M, K), float("inf"), dtype=torch.float32, device=dev)
    i0, d0 = knn_backward_exact(x[:P0], K)
    idx[:P0], dd[:P0] = i0, d0
    lo = P0
    nx = _sqnorm(x)
    while lo < M:
        hi = min(M, 2 * lo)
        pre = x[:hi]
        C = max(16, int(2 ** round(math.log2(max(16.0, math.sqrt(hi) * 1.3)))))
        cent = _kmeans(pre, C, iters=5, seed=seed + lo)
        prim = _assign(pre, cent, 1)[:, 0]
        order = torch.argsort(prim)
        counts = torch.bincount(prim, minlength=C)
        starts = torch.cumsum(counts, 0) - counts
        q = torch.arange(lo, hi, device=dev)
        probe = _assign(x[lo:hi], cent, probes)  # [nq, P]
        qcell = probe.reshape(-1)
        qorder = torch.argsort(qcell)
        qcounts = torch.bincount(qcell, minlength=C)
        qstarts = torch.cumsum(qcounts, 0) - qcounts
        nq = hi - lo
        ci = torch.full((nq * probes, K), -1, dtype=torch.int64, device=dev)
        cd = torch.full((nq * probes, K), float("inf"), dtype=torch.float32, device=dev)
        ch, sh, qch, qsh = counts.tolist(), starts.tolist(), qcounts.tolist(), qstarts.tolist()
        for c in range(C):
            nm, nqc = ch[c], qch[c]
            if nm == 0 or nqc == 0:
                continue
            mem = order[sh[c]:sh[c] + nm]
            qp = qorder[qsh[c]:qsh[c] + nqc]
            qpt = q[qp // probes]
            for s in range(0, nqc, 8192):
                qs = qpt[s:s + 8192]
                d2 = nx[qs, None] + nx[None, mem] - 2.0 * (x[qs] @ x[mem].T)
                d2 = d2.masked_fill(mem[None, :] >= qs[:, None], float("inf"))
                kk = min(K, nm)
                v, i = torch.topk(d2, kk, dim=1, largest=False)
                ci[qp[s:s + 8192], :kk] = torch.where(torch.isfinite(v), mem[i], -1)
                cd[qp[s:s + 8192], :kk] = v
        v, j = torch.topk(cd.view(nq, probes * K), K, dim=1, largest=False)
        idx[lo:hi] = torch.gather(ci.view(nq, probes * K), 1, j)
        dd[lo:hi] = v
        lo = hi
    return idx, dd


def symmetric_prune(idx, dd, cap: int):
    """Undirected union of k-NN edges, keep (u,v) iff it is within the `cap` nearest
    incident edges of both u and v -> symmetric rows with degree <= cap."""
    torch = _torch()
    M, K = idx.shape
    dev = idx.device
    src = torch.arange(M, device=dev).repeat_interleave(K)
    dst = idx.reshape(-1)
    d = dd.reshape(-1)
    ok = (dst >= 0) & torch.isfinite(d) & (dst != src)
    src, dst, d = src[ok], dst[ok], d[ok]
    u = torch.minimum(src, dst)
    v = torch.maximum(src, dst)
    key = u * M + v
    key, inv = torch.unique(key, return_inverse=True)
    dmin = torch.full((key.shape[0],), float("inf"), device=dev).scatter_reduce_(
        0, inv, d, reduce="amin")
    u = key // M
    v = key % M
    E = key.shape[0]
    # rank of every edge among each endpoint's incident edges (by distance, then other id)
    end = torch.cat([u, v])
    oth = torch.cat([v, u])
    dist = torch.cat([dmin, dmin])
    eid = torch.arange(E, device=dev).repeat(2)
    o1 = torch.argsort(oth, stable=True)
    o2 = torch.argsort(dist[o1], stable=True)
    o = o1[o2]
    o3 = torch.argsort(end[o], stable=True)
    o = o[o3]
    end_s = end[o]
    cnt = torch.bincount(end_s, minlength=M)
    first = torch.cumsum(cnt, 0) - cnt
    rank = torch.arange(end_s.shape[0], device=dev) - first[end_s]
    ok_inc = rank < cap
    keep = torch.zeros(E, dtype=torch.int32, device=dev)
    keep.index_add_(0, eid[o], ok_inc.to(torch.int32))
    kept = keep == 2
    # rows: incident kept edges per node, nearest first
    sel = kept[eid[o]]
    end_k = end_s[sel]
    oth_k = oth[o][sel]
    deg = torch.bincount(end_k, minlength=M)
    first = torch.cumsum(deg, 0) - deg
    pos = torch.arange(end_k.shape[0], device=dev) - first[end_k]
    rows = torch.full((M, cap), -1, dtype=torch.int32, device=dev)
    rows[end_k, pos] = oth_k.to(torch.int32)
    return rows, deg.to(torch.int32)


def long_links(x, n_links: int, seed: int, n_random: int = 256, block: int = 8192):
    """Navigability links (the role HNSW's early insertions play): every node links to the
    nearest members of its OWN random subset of the layer (n_random draws).  Nearest-of-a-
    sparse-random-sample edges span the gaps a k-NN graph leaves between clusters, and since
    every node draws a different subset no node becomes a hub that symmetric pruning would
    strip."""
    torch = _torch()
    M, dev = x.shape[0], x.device
    g = torch.Generator(device=dev)
    g.manual_seed(seed + 7919)
    S = min(n_random, M - 1)
    K = min(n_links, S)
    idx = torch.empty((M, K), dtype=torch.int64, device=dev)
    dd = torch.empty((M, K), dtype=torch.float32, device=dev)
    for s in range(0, M, block):
        e = min(M, s + block)
        cand = torch.randint(0, M, (e - s, S), generator=g, device=dev)
        d2 = ((x[s:e, None, :] - x[cand]) ** 2).sum(-1)
        d2 = torch.where(cand == torch.arange(s, e, device=dev)[:, None], float("inf"), d2)
        v, i = torch.topk(d2, K, dim=1, largest=False)
        idx[s:e] = torch.gather(cand, 1, i)
        dd[s:e] = v
    return idx, dd


def merge_rows(r1, c1, r2, c2, cap: int):
    """Union of two symmetric row sets (degree caps add up to <= cap), duplicates dropped."""
    torch = _torch()
    M = r1.shape[0]
    both = torch.cat([r1, r2], 1).long()
    valid = torch.cat([torch.arange(r1.shape[1], device=r1.device)[None, :] < c1[:, None],
                       torch.arange(r2.shape[1], device=r1.device)[None, :] < c2[:, None]], 1)
    both = torch.where(valid, both, torch.full_like(both, M))
    both, _ = torch.sort(both, 1)
    dup = torch.zeros_like(valid)
    dup[:, 1:] = both[:, 1:] == both[:, :-1]
    both = torch.where(dup, torch.full_like(both, M), both)
    both, _ = torch.sort(both, 1)
    cnt = (both < M).sum(1)
    rows = torch.where(both < M, both, torch.full_like(both, -1))[:, :cap].to(torch.int32)
    return rows, cnt.to(torch.int32)


def build_layers(vectors, m: int = 16, level_prob: float = 1.0 / 17.0, max_layers: int = 4,
                 seed: int = 0, device=None, exact_limit: int = 200_000, long_frac: float = 0.0,
                 n_random: int = 64, mode: str = "hnsw"):
    """Return dict(levels, entry_slot, n_layers, nbrs=[(n, cap_l) int32], cnts=[(n,) int32])."""
    torch = _torch()
    dev = torch.device(device if device is not None else "cuda")
    x = vectors if not isinstance(vectors, np.ndarray) else torch.from_numpy(
        np.ascontiguousarray(vectors, dtype=np.float32))
    x = x.to(dev, dtype=torch.float32)
    n = x.shape[0]
    levels = draw_levels(n, level_prob, max_layers, seed)
    top = int(levels.max())
    entry = int(np.argmax(levels))
    nbrs, cnts = [], []
    lv_t = torch.from_numpy(levels).to(dev)
    for l in range(top + 1):
        cap = 2 * m if l == 0 else m
        mem = torch.nonzero(lv_t >= l).squeeze(1)
        M = mem.shape[0]
        rows = np.full((n, cap), 0, dtype=np.int32)
        cnt = np.zeros(n, dtype=np.int32)
        if M >= 2:
            xm = x[mem]
            K = min(cap, M - 1)
            if mode == "hnsw":  # backward (insertion-order) k-NN, m per node like keep-M
                Kb = min(m, M - 1)
                idx, dd = (knn_backward_exact(xm, Kb) if M <= exact_limit
                           else knn_backward_ivf(xm, Kb, seed=seed + l))
            elif M <= exact_limit:
                idx, dd = knn_exact(xm, K)
            else:
                idx, dd = knn_ivf(xm, K, seed=seed + l)
            c_long = int(cap * long_frac) if M > 4 * cap else 0
            r, c = symmetric_prune(idx, dd, cap - c_long)
            ll = long_links(xm, c_long, seed + 31 * l, n_random) if c_long else None
            if ll is not None:
                rl, cl = symmetric_prune(ll[0], ll[1], c_long)
                r, c = merge_rows(r, c, rl, cl, cap)
            glob = torch.where(r >= 0, mem[r.clamp_min(0).long()].to(torch.int32),
                               torch.zeros_like(r))
            mem_h = mem.cpu().numpy()
            rows[mem_h] = glob.cpu().numpy()
            cnt[mem_h] = c.cpu().numpy()
        nbrs.append(rows)
        cnts.append(cnt)
    return dict(levels=levels, entry_slot=entry, n_layers=top + 1, nbrs=nbrs, cnts=cnts)
