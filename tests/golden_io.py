"""Helpers to read the committed golden fixtures (tests/golden/*.npz).

The fixtures were written by ``tests/golden/make_golden.py`` from the reference
package itself; nothing here touches ``/root/reference`` at run time.
"""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


def graph_layers(z):
    return [(z[f"nbrs{l}"], z[f"cnts{l}"]) for l in range(int(z["n_layers"]))]


def model_layers(z, prefix=""):
    n = int(z[f"{prefix}n_mlp"])
    return [(z[f"{prefix}W{m}"], z[f"{prefix}b{m}"]) for m in range(n)], z[f"{prefix}A"], \
        bool(z[f"{prefix}relu"])


def param_sets(z):
    out = []
    i = 0
    while f"p{i}/params" in z.files:
        k, kp, hops, ef = (int(v) for v in z[f"p{i}/params"])
        out.append((i, dict(k=k, k_parallel=kp, hops=hops, ef=ef)))
        i += 1
    return out


def expected(z, pi):
    p = f"p{pi}/"
    return {key: z[p + "res_" + key] for key in
            ("ids", "scores", "n", "evals", "visited", "best_hop", "per_layer", "rows",
                         "nbr_ids")}


SEARCH_FIXTURES = ["search_d64_z2", "search_d128_z3", "search_d32_shuffled"]


# ---- tests/golden/reftests.npz: the reference's own test_search.py cases (make_reftests.py)
class RefCase:
    """One recorded case: graph arrays, fp64 vectors/queries, per-parameter-set results."""

    def __init__(self, z, name: str):
        self.name = name
        p = name + "/"
        self.z, self.p = z, p
        self.vectors = z[p + "vectors"]
        self.queries = z[p + "queries"]
        self.ids = z[p + "ids"]
        self.levels = z[p + "levels"]
        self.entry = int(z[p + "entry_slot"])
        self.m = int(z[p + "m"])
        self.layers = [(z[p + f"nbrs{l}"], z[p + f"cnts{l}"]) for l in range(int(z[p + "n_layers"]))]
        self.bf_ids = z[p + "bf_ids"]
        self.bf_scores = z[p + "bf_scores"]

    def params(self):
        out, i = [], 0
        while f"{self.p}p{i}/params" in self.z.files:
            k, kp, hops, ef = (int(v) for v in self.z[f"{self.p}p{i}/params"])
            out.append((i, dict(k=k, k_parallel=kp, hops=hops, ef=ef)))
            i += 1
        return out

    def expected(self, pi):
        pp = f"{self.p}p{pi}/"
        return {k: self.z[pp + k] for k in ("ids", "scores", "n", "evals", "per_layer", "best_hop")}


def ref_cases(prefix: str = ""):
    z = load("reftests")
    names = sorted({k.split("/")[0] for k in z.files if k.endswith("/entry_slot")})
    return [n for n in names if n.startswith(prefix)]


def ref_case(name: str) -> RefCase:
    return RefCase(load("reftests"), name)
