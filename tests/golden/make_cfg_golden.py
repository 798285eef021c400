"""Golden results for BASELINE configs 1 and 2 from the REFERENCE package itself.

Run in the build container (the reference is not on the GPU box):

    REF_SRC=/tmp/refbuild/src python tests/golden/make_cfg_golden.py cfg1 [cfg2]

(``REF_SRC`` = a writable copy of /root/reference/pkg with ``_chot`` built in place,
``python setup.py build_ext --inplace``; it only speeds up ``GraphIndex.build``.)

Inputs are the reference's own recipe:
items = ``model.item_embeddings(clustered_vectors(N, d, C, seed=0).astype(f32))``,
model = ``create_model(d, d, Z, (64, 64), seed=1)``,
users = ``model.user_embedding(default_rng(7).normal(size=(Q, d)).astype(f32))``,
graph = ``GraphIndex.build(items.astype(f64), m=16, ef_construction=64, seed=0)``.

The fixture stores no bulk arrays: digests of the items / users / graph (so the GPU box,
which regenerates the items with numpy and the graph with the native exact builder,
can prove it searched the SAME inputs) plus the reference's ``c_hipanns`` results
(ids, scores, evaluation counts, per-layer counts, hops_to_best, rows expanded,
neighbour ids read) and ``brute_force`` top-100 for the first queries.
The reference-built NANN-IDX file is written to ``$REF_GRAPHS`` (default
/tmp/refgraphs) for local comparisons; it is too large to commit.
"""

from __future__ import annotations

import hashlib
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REF_SRC = os.environ.get("REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)

from nann import GraphIndex, SearchParams, brute_force, c_hipanns, create_model, model_scorer  # noqa: E402
from nann.bench import clustered_vectors  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import WorkCounter, result_arrays  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
REF_GRAPHS = os.environ.get("REF_GRAPHS", "/tmp/refgraphs")

# name: N, d, Z, m, clusters, batch Q, golden queries per parameter set, gt queries
CFGS = {
    "cfg1": (100_000, 64, 2, 16, 256, 1_000, [(dict(k=100, k_parallel=8, hops=3), 128),
                                               (dict(k=100, k_parallel=32, hops=10), 64)], 128),
    "cfg2": (1_000_000, 128, 3, 16, 1024, 10_000, [(dict(k=100, k_parallel=8, hops=3), 96),
                                                    (dict(k=100, k_parallel=32, hops=10), 24)], 96),
}


def graph_digest(ids, levels, layers, entry) -> str:
    """sha256 over ids, levels, entry and every layer's rows in stored order."""
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


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


_G = {}


def _search_one(args):
    q, p = args
    index, model, users, emb, counter = _G["index"], _G["model"], _G["users"], _G["emb"], _G["counter"]
    counter.take()
    r = c_hipanns(index, model_scorer(model, users[q], emb), SearchParams(**p))
    rows, ids = counter.take()
    return r, rows, ids


def _bf_one(q):
    model, users, emb = _G["model"], _G["users"], _G["emb"]
    r = brute_force(model_scorer(model, users[q], emb), np.arange(len(emb)), 100)
    return np.asarray(r.item_ids(), dtype=np.int64), np.asarray([s for _, s in r.items])


def make(name: str, procs: int) -> None:
    N, d, Z, m, C, Q, psets, n_gt = CFGS[name]
    t0 = time.time()
    model = create_model(d_x=d, d_h=d, z_dim=Z, hidden=(64, 64), seed=1)
    emb = model.item_embeddings(clustered_vectors(N, d, C, seed=0).astype(np.float32))
    users = model.user_embedding(np.random.default_rng(7).normal(size=(Q, d)).astype(np.float32))
    os.makedirs(REF_GRAPHS, exist_ok=True)
    path = os.path.join(REF_GRAPHS, f"{name}.nann")
    if os.path.exists(path):
        index = GraphIndex.load(path)
        print(f"{name}: loaded {path}", flush=True)
    else:
        index = GraphIndex.build(emb.astype(np.float64), m=m, ef_construction=64, seed=0)
        index.save(path)
        print(f"{name}: reference build {time.time() - t0:.1f}s", flush=True)
    ids, levels, layers, entry = index.graph_view()
    out = {"N": np.int64(N), "d": np.int64(d), "Z": np.int64(Z), "m": np.int64(m),
           "clusters": np.int64(C), "Q": np.int64(Q),
           "items_sha256": np.array(digest(emb)), "users_sha256": np.array(digest(users)),
           "graph_sha256": np.array(graph_digest(ids, levels, layers, entry)),
           "layer_counts": np.asarray(index.layer_node_counts(), dtype=np.int64),
           "entry_slot": np.int64(entry)}
    _G.update(index=index, model=model, users=users, emb=emb, counter=WorkCounter())
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        for pi, (p, nq) in enumerate(psets):
            t1 = time.time()
            res = pool.map(_search_one, [(q, p) for q in range(nq)], chunksize=1)
            sp = SearchParams(**p)
            for key, val in result_arrays(res, sp.k).items():
                out[f"p{pi}/{key}"] = val
            out[f"p{pi}/params"] = np.array([sp.k, sp.k_parallel, sp.hops, sp.frontier_width])
            out[f"p{pi}/wall_s"] = np.float64(time.time() - t1)
            out[f"p{pi}/procs"] = np.int64(procs)
            print(f"{name} p{pi} {p}: {nq} queries {time.time() - t1:.1f}s "
                  f"evals mean {out[f'p{pi}/res_evals'].mean():.0f}", flush=True)
        t1 = time.time()
        gts = pool.map(_bf_one, range(n_gt), chunksize=1)
        out["gt100"] = np.stack([g[0] for g in gts])
        out["gt100_scores"] = np.stack([g[1] for g in gts])
        print(f"{name} brute force {n_gt} queries {time.time() - t1:.1f}s", flush=True)
    for pi in range(len(psets)):
        got = out[f"p{pi}/res_ids"]
        nq = got.shape[0]
        ng = min(nq, n_gt)
        rec = np.mean([len(set(got[q]) & set(out["gt100"][q])) / 100.0 for q in range(ng)])
        out[f"p{pi}/recall100"] = np.float64(rec)
        print(f"{name} p{pi} recall@100 {rec:.4f} over {ng} queries", flush=True)
    np.savez_compressed(os.path.join(OUT, f"{name}_ref.npz"), **out)
    print(f"{name}: done in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    procs = int(os.environ.get("PROCS", os.cpu_count() or 1))
    for name in sys.argv[1:] or ["cfg1"]:
        make(name, procs)
