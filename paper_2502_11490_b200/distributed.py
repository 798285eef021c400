"""Multi-GPU execution of the hot path (one process per GPU, torch.distributed plumbing).

Two modes:

* **query partition** (cfg3/cfg5): every rank holds a replica of the index and searches
  a contiguous block of the query batch — queries never interact (evalharness.py:322-351),
  so there is no data-path collective.
* **catalog shards** (cfg4): rank r holds a contiguous item-id range as an independent
  graph with GLOBAL ids (slot order = id order, so tie-breaks agree); every rank searches
  all queries on its shard, the per-shard top-k lists are packed to 8 bytes per entry
  (fp32 score | u32 id), all-gathered in ONE collective (NCCL over NVLink) and merged on
  the device by ``gr_merge_topk_packed`` with the reference pool's
  (score desc, id asc) order — the restatement of "CandidatePool(k).push every shard
  result" (pool.py:30-55).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import InvalidArgumentError
from .index import GraphIndex
from .search import SearchParams, device_items


def block_range(n: int, world: int, rank: int) -> tuple:
    """Contiguous [lo, hi) block of n units for `rank` (first n % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidArgumentError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_packed(packed, group=None):
    """All-gather per-rank packed [Q, k] lists (int64 view of the 8-byte wire format,
    ``gr_pack_topk``) -> [R, Q, k] on every rank: ONE collective of 8 B per entry over the
    process group's backend (NCCL over NVLink on GPUs; gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return packed[None]  # single process: one shard
    world = dist.get_world_size(group)
    out = torch.empty((world * packed.shape[0],) + tuple(packed.shape[1:]), dtype=packed.dtype,
                      device=packed.device)
    dist.all_gather_into_tensor(out, packed.contiguous(), group=group)
    return out.view((world,) + tuple(packed.shape))


def pack_lists(ids, scores):
    """Device [Q, k] (ids int64, scores f64) -> packed int64 [Q, k] (gr_pack_topk)."""
    import torch

    dev = ids.device
    out = torch.empty(ids.shape, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().gr_pack_topk(dev.index or 0, ids.data_ptr(), scores.data_ptr(),
                                       ids.numel(), out.data_ptr(), ctypes.c_void_p(stream)))
    return out


def merge_packed(all_packed, k: int):
    """Device merge of packed [R, Q, k_in] lists -> (ids [Q, k], scores [Q, k], count [Q])."""
    import torch

    R, Q, kin = all_packed.shape
    dev = all_packed.device
    out_i = torch.empty((Q, k), dtype=torch.int64, device=dev)
    out_s = torch.empty((Q, k), dtype=torch.float64, device=dev)
    out_c = torch.empty(Q, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().gr_merge_topk_packed(dev.index or 0, all_packed.data_ptr(), R, Q, kin, k,
                                               out_i.data_ptr(), out_s.data_ptr(), out_c.data_ptr(),
                                               ctypes.c_void_p(stream)))
    return out_i, out_s, out_c


def gather_lists(ids, scores, group=None):
    """Pack this rank's device [Q, k] lists and all-gather them -> packed [R, Q, k]."""
    return gather_packed(pack_lists(ids, scores), group)


def merge_lists(all_ids, all_scores, k: int):
    """Device merge of unpacked [R, Q, k_in] lists -> (ids [Q, k], scores [Q, k], count [Q])."""
    import torch

    R, Q, kin = all_ids.shape
    dev = all_ids.device
    out_i = torch.empty((Q, k), dtype=torch.int64, device=dev)
    out_s = torch.empty((Q, k), dtype=torch.float64, device=dev)
    out_c = torch.empty(Q, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().gr_merge_topk(dev.index or 0, all_ids.data_ptr(), all_scores.data_ptr(),
                                        R, Q, kin, k, out_i.data_ptr(), out_s.data_ptr(),
                                        out_c.data_ptr(), ctypes.c_void_p(stream)))
    return out_i, out_s, out_c


class ShardedSearcher:
    """Catalog-sharded C-HiPANNS: local shard search + NCCL all-gather + device merge."""

    def __init__(self, shard_index: GraphIndex, model, shard_items, group=None,
                 device: int | None = None):
        self.index = shard_index
        self.metric = getattr(model, "metric", model)
        self.device = _lib.current_device() if device is None else device
        self.dm = self.metric.device_model(self.device)
        self.graph = shard_index.device_graph(self.device, items=shard_items)
        self.items = device_items(shard_items, self.device)
        self.searcher = _lib.DeviceSearcher(self.device)
        self.group = group
        ids = shard_index.item_ids()
        if len(ids) and (ids.min() < 0 or ids.max() >= 1 << 32):
            raise InvalidArgumentError("shard item ids must lie in [0, 2^32) (8-byte merge format)")

    def search_local(self, users_d, params: SearchParams):
        import torch

        Q, k, L = users_d.shape[0], params.k, self.graph.n_layers
        dev = users_d.device
        ids = torch.empty((Q, k), dtype=torch.int64, device=dev)
        sc = torch.empty((Q, k), dtype=torch.float64, device=dev)
        cnt = torch.empty(Q, dtype=torch.int32, device=dev)
        st = torch.empty((Q, 5 + L), dtype=torch.int64, device=dev)
        pc = params._c()
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        _lib.check(_lib.lib().gr_search_async(self.searcher.h, self.graph.h, self.dm.h,
                                              self.items.h, users_d.data_ptr(), Q,
                                              ctypes.byref(pc), ids.data_ptr(), sc.data_ptr(),
                                              cnt.data_ptr(), st.data_ptr(), stream))
        return ids, sc, cnt, st

    def search(self, users_d, params: SearchParams):
        """Global top-k for every query (identical on all ranks) + this shard's stats."""
        ids, sc, _, st = self.search_local(users_d, params)
        out = merge_packed(gather_lists(ids, sc, self.group), params.k)
        return out + (st,)


def shard_index(full_levels, shard_layers, entry_slot, lo: int, n: int, m: int) -> GraphIndex:
    """Wrap one shard's graph: slots 0..n-1 hold global ids lo..lo+n-1, embedding rows local."""
    idx = GraphIndex.from_arrays(np.arange(lo, lo + n, dtype=np.int64), full_levels, shard_layers,
                                 entry_slot, m=m)
    idx.rows = np.arange(n, dtype=np.int32)
    return idx
