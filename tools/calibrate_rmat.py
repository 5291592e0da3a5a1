"""Finds the RMAT pair budget that gives each config's directed edge count
with exact-V generation: pairs are drawn by the reference's
gen_rmat over n_pad = 2^ceil(log2 V) (a,b,c,d = .45/.22/.22/.11, seed 7),
pairs with an endpoint >= V or self loops are rejected, and the graph is
build_undirected_csr with n_hint = V. m(P) for every prefix P of one long
draw is 2 * #{undirected edges first seen before P}, so one sort suffices.

Output: the budgets hard-coded in bench.py CONFIGS.
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2204_02662_b200 as pg  # noqa: E402

CONFIGS = {  # name: (V, target directed m, max pairs to draw)
    "cora": (2708, 10556, 20000),
    "pubmed": (19717, 88648, 150000),
    "arxiv": (169343, 1166243, 2_000_000),
    "products": (2449029, 61859140, 60_000_000),
    "reddit": (232965, 114615892, 90_000_000),
}


def calibrate(name, V, target, max_pairs):
    t = time.time()
    pairs, n_pad = pg.gen_rmat(V, max_pairs, 0.45, 0.22, 0.22, 0.11, 7)
    u = pairs[:, 0].astype(np.uint64)
    v = pairs[:, 1].astype(np.uint64)
    keep = (u < V) & (v < V) & (u != v)
    idx = np.nonzero(keep)[0]
    lo = np.minimum(u[idx], v[idx])
    hi = np.maximum(u[idx], v[idx])
    key = (lo << np.uint64(32)) | hi
    _, first = np.unique(key, return_index=True)
    first_pair = np.sort(idx[first])  # raw pair index of each edge's first draw
    total = 2 * len(first_pair)
    if total < target:
        print(f"{name}: max_pairs too small: m={total} < {target}")
        return None
    k = (target + 1) // 2  # undirected edges needed
    P = int(first_pair[k - 1]) + 1
    m = 2 * int(np.searchsorted(first_pair, P))
    print(f"{name}: V={V} n_pad={n_pad} pairs={P} -> m={m} (target {target}) [{time.time() - t:.1f}s]", flush=True)
    return P, m


if __name__ == "__main__":
    names = sys.argv[1:] or list(CONFIGS)
    for n in names:
        calibrate(n, *CONFIGS[n])
