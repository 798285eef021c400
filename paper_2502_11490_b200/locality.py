"""Device slot order for memory locality (input preparation for the device graph).

The search kernels keep per-query visited bitsets indexed by device slot, gather adjacency
rows by slot and read a slot-ordered copy of the item embeddings.  Graph neighbours that
sit far apart in slot space dirty one 32-byte sector each per touch; neighbours that sit
in a contiguous slot range share sectors.  ``cluster_order`` groups slots by a k-means
clustering of their embedding rows (clusters of ~``per_cluster`` items; graph edges of a
learned-metric k-NN/HNSW graph stay mostly inside such clusters), breadth-first order is
the fallback when no embeddings are at hand.  Results never depend on the order (ids and
the id-rank tie-break travel with the slots, gr_graph_create_ordered).
"""

from __future__ import annotations

import numpy as np


def cluster_order(emb, slot_rows=None, per_cluster: int | None = None, iters: int = 5, seed: int = 0,
                  device: int = 0) -> np.ndarray:
    """int64 permutation: caller slots grouped by k-means cluster of their embedding row."""
    import os

    import torch

    if per_cluster is None:
        per_cluster = int(os.environ.get("GMPGR_CLUSTER", "2048"))

    dev = torch.device("cuda", device)
    x = emb if isinstance(emb, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(emb))
    x = x.to(dev, dtype=torch.float32)
    if slot_rows is not None:
        x = x[torch.from_numpy(np.asarray(slot_rows, dtype=np.int64)).to(dev)]
    n, d = x.shape
    K = max(1, n // per_cluster)
    if K == 1:
        return np.arange(n, dtype=np.int64)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    samp = x[torch.randperm(n, generator=g, device=dev)[: min(n, 32 * K)]]
    cent = samp[:K].clone()

    def assign(v, c, block=1 << 16):
        cn = (c * c).sum(1)
        out = torch.empty(v.shape[0], dtype=torch.int64, device=dev)
        for s in range(0, v.shape[0], block):
            e = min(v.shape[0], s + block)
            out[s:e] = torch.argmin(cn[None, :] - 2.0 * (v[s:e] @ c.T), dim=1)
        return out

    for _ in range(iters):
        a = assign(samp, cent)
        sums = torch.zeros_like(cent).index_add_(0, a, samp)
        cnt = torch.bincount(a, minlength=K).to(sums.dtype)[:, None]
        cent = torch.where(cnt > 0, sums / cnt.clamp_min(1.0), cent)
    lab = assign(x, cent)
    import os

    if K >= 16 and os.environ.get("GMPGR_ORDER2", "0") != "0":
        # second level: clusters grouped by a k-means of their centroids (~sqrt(K) groups),
        # so clusters that share graph edges also sit near each other in slot space
        K2 = max(2, int(round(K ** 0.5)))
        c2 = cent[torch.randperm(K, generator=g, device=dev)[:K2]].clone()
        for _ in range(iters):
            a2 = assign(cent, c2)
            s2 = torch.zeros_like(c2).index_add_(0, a2, cent)
            n2 = torch.bincount(a2, minlength=K2).to(s2.dtype)[:, None]
            c2 = torch.where(n2 > 0, s2 / n2.clamp_min(1.0), c2)
        sup = assign(cent, c2)
        lab = sup[lab] * K + lab
    order = torch.sort(lab, stable=True).indices
    return order.cpu().numpy().astype(np.int64)
