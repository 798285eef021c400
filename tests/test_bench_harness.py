"""Host-side pieces of the benchmark harness (no GPU):

* the exact-graph cache of workload.exact_graph (rank 0 builds and saves, later calls and
  other ranks load) reproduces GraphIndex.build digest for digest;
* the stock-reference harness of bench.py -- the unmodified reference package (nann,
  pip-installed into baseline/_ref) searching a graph this repo built -- agrees with the C
  oracle on ids, scores and evaluation counts.
"""

import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exact_graph_cache_roundtrip(tmp_path, monkeypatch):
    torch = pytest.importorskip("torch")
    from paper_2502_11490_b200 import workload as W
    from paper_2502_11490_b200.index import GraphIndex

    monkeypatch.setenv("GMPGR_CACHE", str(tmp_path))
    items = torch.randn(2500, 12, generator=torch.Generator().manual_seed(3))
    built = W.exact_graph("t", items, 6, rank=0)          # builds + writes the cache
    assert len(list(tmp_path.iterdir())) == 1
    loaded = W.exact_graph("t", items, 6, rank=1)         # another rank: loads it
    ref = GraphIndex.build(items.double().numpy(), m=6, ef_construction=64, seed=0)
    assert W.graph_digest(built) == W.graph_digest(loaded) == W.graph_digest(ref)
    assert loaded.layer_node_counts() == ref.layer_node_counts()


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "nann")),
                    reason="reference package not installed in baseline/_ref")
def test_stock_reference_matches_oracle(tmp_path, monkeypatch):
    import bench
    from paper_2502_11490_b200 import workload as W

    monkeypatch.setenv("GMPGR_CACHE", str(tmp_path))
    wl = W.make_reference("cfg1", device=None)
    nq = 6
    ids, scores, evals, n, _ = bench.stock_reference(wl, range(nq), bench.PARAMS, processes=2)
    assert n == nq
    r, _ = bench.cpu_search(wl, wl.users[:nq], 2)
    par = bench.parity_vs(ids, scores, evals, r["ids"], r["scores"], r["evals"])
    assert par["ids_identical"] == par["scores_identical"] == par["evals_identical"] == 1.0
    assert np.all(evals > 0)
