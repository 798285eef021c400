"""Native exact index build (csrc/hnsw_build.cpp, gr_hnsw_insert) vs the reference.

Host code only (no GPU): every graph the reference built for the golden fixtures is
rebuilt here from the same vectors and parameters and must be identical node for node
(ids, levels, entry point, every row in stored order).  The reference's own
test_index.py properties are re-run on the native build (build == iterated insert,
insert after reload == uninterrupted build, invariants, duplicate / shape errors).
"""

import hashlib
import os

import numpy as np
import pytest

import golden_io as G
import paper_2502_11490_b200 as P
from paper_2502_11490_b200 import workload


def same_graph(idx, ids, levels, layers, entry):
    n = len(ids)
    gi, gl, glay, ge = idx.graph_view()
    if not (np.array_equal(gi, ids) and np.array_equal(gl, levels) and ge == entry):
        return False
    if len(glay) != len(layers):
        return False
    for (nb, ct), (rn, rc) in zip(glay, layers):
        if not np.array_equal(ct[:n], rc[:n]):
            return False
        mask = np.arange(nb.shape[1])[None, :] < ct[:n, None]
        if not np.array_equal(nb[:n][mask], np.asarray(rn)[:n][:, :nb.shape[1]][mask]):
            return False
    return True


def structure(idx):
    """Reference test_index.py fingerprint: per layer, per id, sorted neighbour ids."""
    ids, _, layers, entry = idx.graph_view()
    out = [int(ids[entry])]
    for l, (nb, ct) in enumerate(layers):
        out.append({int(ids[s]): sorted(int(ids[t]) for t in nb[s, :ct[s]]) for s in range(len(ids))})
    return out


@pytest.mark.parametrize("name,m,heur,shuffle", [
    ("search_d64_z2", 8, False, False),
    ("search_d128_z3", 16, False, False),
    ("search_d32_shuffled", 6, True, True),
])
def test_identical_to_reference_search_fixtures(name, m, heur, shuffle):
    z = G.load(name)
    emb = z["emb"]
    if shuffle:  # make_golden.py: ids = permutation, rows = emb[perm], heuristic selection
        perm = np.random.default_rng(5).permutation(len(emb)).astype(np.int64)
        idx = P.GraphIndex.build(emb[perm].astype(np.float64), ids=perm, m=m, ef_construction=2 * m,
                                 seed=0, select_heuristic=heur)
    else:
        idx = P.GraphIndex.build(emb.astype(np.float64), m=m, ef_construction=2 * m, seed=0,
                                 select_heuristic=heur)
    assert same_graph(idx, z["ids"], z["levels"], G.graph_layers(z), int(z["entry_slot"]))
    idx.validate()


# make_reftests.py: case -> (m, ef_construction, seed) of the reference build
REFTEST_BUILDS = {"complete": (40, 40, 13), "never_twice": (8, 32, 14), "desk": (16, 64, 21),
                  "deterministic": (8, 32, 23), "ties": (6, 24, 25)}
REFTEST_BUILDS.update({f"visited{s}": (8, 32, s) for s in range(20)})
REFTEST_BUILDS.update({f"recall{s}": (8, 32, s) for s in range(20)})


@pytest.mark.parametrize("case", sorted(REFTEST_BUILDS))
def test_identical_to_reference_reftest_graphs(case):
    c = G.ref_case(case)
    m, efc, seed = REFTEST_BUILDS[case]
    idx = P.GraphIndex.build(c.vectors, m=m, ef_construction=efc, seed=seed)
    assert same_graph(idx, c.ids, c.levels, c.layers, c.entry)


def test_reference_written_index_rebuilds_byte_identical(tmp_path):
    path = os.path.join(G.GOLDEN, "euclid_index.nann")
    ref = P.GraphIndex.load(path)
    idx = P.GraphIndex.build(ref._vectors[:len(ref)], ids=ref.item_ids(), m=ref.m,
                             ef_construction=ref.ef_construction, level_prob=ref.level_prob,
                             max_layers=ref.max_layers, seed=ref.seed,
                             select_heuristic=ref.select_heuristic)
    out = str(tmp_path / "rebuilt.nann")
    idx.save(out)
    assert open(out, "rb").read() == open(path, "rb").read()


def clustered(n, d, seed, n_clusters=4):  # reference test_index.py helper shape
    rng = np.random.default_rng(seed)
    centers = rng.normal(scale=5.0, size=(n_clusters, d))
    return centers[rng.integers(0, n_clusters, size=n)] + rng.normal(size=(n, d))


def test_build_equals_iterated_insert():
    vectors = clustered(120, 5, seed=4)
    built = P.GraphIndex.build(vectors, m=5, ef_construction=16, seed=9)
    manual = P.GraphIndex(dim=5, m=5, ef_construction=16, seed=9)
    for i, v in enumerate(vectors):
        manual.insert(i, v)
    assert structure(built) == structure(manual)
    manual.validate()


def test_insert_after_reload_matches_uninterrupted_build(tmp_path):
    vectors = clustered(60, 4, seed=10)
    full = P.GraphIndex.build(vectors, m=4, ef_construction=16, seed=7)
    partial = P.GraphIndex.build(vectors[:40], m=4, ef_construction=16, seed=7)
    path = str(tmp_path / "partial.nann")
    partial.save(path)
    resumed = P.GraphIndex.load(path)
    for i in range(40, 60):
        resumed.insert(i, vectors[i])
    assert structure(resumed) == structure(full)
    resumed.validate()


def test_insert_errors_and_small_cases():
    index = P.GraphIndex(dim=2)
    index.insert(1, np.zeros(2))
    assert index.entry_point == 1 and len(index) == 1
    with pytest.raises(P.InvalidArgumentError):
        index.insert(1, np.ones(2))
    with pytest.raises(P.InvalidArgumentError):
        index.insert(2, np.zeros(3))
    with pytest.raises(P.InvalidArgumentError):
        P.GraphIndex.build(np.zeros((2, 3)), ids=np.array([5, 5]))
    two = P.GraphIndex.build(np.array([[0.0, 0.0], [1.0, 1.0]]), m=2, seed=0)
    assert two.neighbors(0, 0) == [1] and two.neighbors(0, 1) == [0]
    rng = np.random.default_rng(5)
    grown = P.GraphIndex(dim=4, m=4, ef_construction=12, seed=1)
    for i in range(100):
        grown.insert(i, rng.normal(size=4))
    grown.validate()


def test_cfg1_graph_identical_to_reference_build():
    """BASELINE config 1 at full size (100k x 64, m=16, ef_construction=64): the native
    build of the reference's own inputs has the digest the reference build recorded
    (tests/golden/make_cfg_golden.py)."""
    z = G.load("cfg1_ref")
    model, emb, users = workload.reference_inputs("cfg1")
    assert hashlib.sha256(np.ascontiguousarray(emb).tobytes()).hexdigest() == str(z["items_sha256"])
    assert hashlib.sha256(np.ascontiguousarray(users).tobytes()).hexdigest() == str(z["users_sha256"])
    idx = P.GraphIndex.build(emb.astype(np.float64), m=16, ef_construction=64, seed=0)
    assert workload.graph_digest(idx) == str(z["graph_sha256"])
    assert idx.layer_node_counts() == list(z["layer_counts"])


def test_parallel_build_equals_single_thread(monkeypatch):
    """The speculative parallel build (planners + in-order committer) is exact: any thread
    count gives the sequential graph."""
    vectors = clustered(20_000, 16, seed=11, n_clusters=64)
    graphs = []
    for threads in ("1", "3", "8"):
        monkeypatch.setenv("GMPGR_BUILD_THREADS", threads)
        idx = P.GraphIndex.build(vectors, m=8, ef_construction=32, seed=2)
        graphs.append(workload.graph_digest(idx))
    assert graphs[0] == graphs[1] == graphs[2]
