"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

Query partition: disjoint contiguous blocks covering the batch.  Catalog shards: each
rank computes its shard's exact top-k (brute force over global ids, scored by the C
oracle), packed to the 8-byte wire format (fp32 score | u32 id, gr_pack_topk's layout) and
all-gathered with the same single-collective `gather_packed` the NCCL path uses, and
merging them with the reference pool semantics (CandidatePool) equals the global top-k.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _orderable(f32):
    u = f32.view(np.uint32)
    return np.where(u & 0x80000000, ~u, u | 0x80000000).astype(np.uint64)


def pack_wire(ids, scores):
    """Host statement of gr_pack_topk's format: orderable(fp32) << 32 | u32 id; 0 = empty."""
    key = (_orderable(scores.astype(np.float32)) << np.uint64(32)) | ids.astype(np.uint64) & np.uint64(0xFFFFFFFF)
    return np.where(ids < 0, np.uint64(0), key).view(np.int64)


def unpack_wire(packed):
    p = packed.view(np.uint64)
    hi = (p >> np.uint64(32)).astype(np.uint32)
    u = np.where(hi & 0x80000000, hi & 0x7FFFFFFF, ~hi).astype(np.uint32)
    ids = np.where(p == 0, -1, (p & np.uint64(0xFFFFFFFF)).astype(np.int64))
    return ids, u.view(np.float32).astype(np.float64)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle_c
        from paper_2502_11490_b200.distributed import block_range, gather_packed
        from paper_2502_11490_b200 import CandidatePool, create_model

        rng = np.random.default_rng(0)
        N, d, Q, k = 997, 16, 5, 10
        model = create_model(d_x=d, d_h=d, z_dim=3, hidden=(32, 32), seed=2)
        emb = rng.normal(size=(N, d)).astype(np.float32)
        users = rng.normal(size=(Q, d)).astype(np.float32)
        ml = model.metric
        lo, hi = block_range(N, world, rank)
        ids = torch.full((Q, k), -1, dtype=torch.int64)
        sc = torch.full((Q, k), float("nan"), dtype=torch.float64)
        for qq in range(Q):
            s, _ = oracle_c.relevance(ml.layers, ml.attention, True, users[qq], emb[lo:hi])
            order = np.lexsort((np.arange(lo, hi), -s.astype(np.float64)))[:k]
            ids[qq, : len(order)] = torch.from_numpy(order + lo)
            sc[qq, : len(order)] = torch.from_numpy(s[order].astype(np.float64))
        all_p = gather_packed(torch.from_numpy(pack_wire(ids.numpy(), sc.numpy())))
        assert tuple(all_p.shape) == (world, Q, k)
        all_i, all_s = unpack_wire(all_p.numpy())
        ok = True
        for qq in range(Q):
            pool = CandidatePool(k)
            for r in range(world):
                for j in range(k):
                    if all_i[r, qq, j] >= 0:
                        pool.push(int(all_i[r, qq, j]), float(all_s[r, qq, j]))
            s, _ = oracle_c.relevance(ml.layers, ml.attention, True, users[qq], emb)
            gt = np.lexsort((np.arange(N), -s.astype(np.float64)))[:k]
            ok &= [i for i, _ in pool.top(k)] == gt.tolist()
        blocks = [block_range(1000, world, r) for r in range(world)]
        ok &= blocks[0][0] == 0 and blocks[-1][1] == 1000
        ok &= all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_sharded_merge_equals_global_topk_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
