"""Pins the oracle's composition of the GCN chain (forward, top_grad,
backward_all_active / backward_ifelse / backward_epp Local+Global) against
the reference's own engine.hpp run on identical inputs (oracle/_ref).
Everything bit-exact: every product keeps the reference's ascending order
with separately rounded mul/add, and expf is the same libm call."""
import numpy as np
import pytest

from conftest import rmat_pairs


def chain_inputs(orc, n_req, m, seed, ratio, L, f, hidden, classes, symnorm=True):
    pairs, n_pad = rmat_pairs(orc, n_req, m, seed)
    g = orc.build_graph(pairs, n_hint=n_pad, symnorm=symnorm)
    vt = orc.sample_training_set(g.n, ratio, 42)
    rng = np.random.default_rng(seed)
    dims = [hidden] * (L - 1) + [classes]
    ins = [f] + dims[:-1]
    x0 = rng.uniform(0, 1, size=(g.n, f)).astype(np.float32)
    ws = [rng.uniform(-0.5, 0.5, size=(ins[l], dims[l])).astype(np.float32) for l in range(L)]
    r = np.zeros((g.n, classes), np.float32)
    r[vt, rng.integers(0, classes, size=len(vt))] = 1.0
    return g, vt, x0, ws, r


def oracle_chain(orc, g, vt, x0, ws, r, mode, gs=4):
    arts = orc.forward(g, x0, ws)
    top = orc.top_grad_f32(arts["x"][-1], r, vt)
    L = len(ws)
    if mode == 0:
        wg, xg, edges = orc.backward_full(g, arts, top, ws)
    elif mode == 1:
        levels = orc.compute_frontiers(g, vt, L)
        wg, xg, edges = orc.backward_full(g, arts, top, ws, levels=levels, gs=gs)
    else:
        levels = orc.compute_frontiers(g, vt, L)
        paths = orc.prepare_all_paths(g, levels)
        wg, xg, edges = orc.backward_epp(paths, levels, arts, top, ws, "local" if mode == 2 else "global")
    return arts, top, wg, xg, edges


def same(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


CASES = [
    # n_req, m, seed, ratio, L, f, hidden, classes, symnorm
    (1024, 8192, 7, 0.1, 2, 24, 16, 4, True),
    (512, 3000, 3, 0.05, 3, 12, 8, 3, False),
    (2048, 9000, 11, 0.5, 2, 40, 33, 7, True),
    (700, 2500, 5, 0.2, 1, 9, 0, 5, True),  # a single layer: no relu, W'^(0) only
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_chain_matches_reference(orc, ref, case, mode):
    n_req, m, seed, ratio, L, f, hidden, classes, symnorm = case
    g, vt, x0, ws, r = chain_inputs(orc, n_req, m, seed, ratio, L, f, hidden, classes, symnorm)
    want = ref.chain_f32(g, vt, x0, ws, r, mode, graph_gs=4, path_gs=2)
    arts, top, wg, xg, edges = oracle_chain(orc, g, vt, x0, ws, r, mode)
    for l in range(L):
        assert same(arts["y"][l], want["y"][l]), f"Y^({l})"
        assert same(arts["pre"][l], want["pre"][l]), f"pre^({l})"
        assert same(arts["x"][l + 1], want["x"][l + 1]), f"X^({l + 1})"
    assert same(top, want["top"])
    for l in range(L):
        assert same(wg[l], want["w_grads"][l]), f"W^({l})' mode {mode}"
    if mode == 0:
        for i in range(L):
            assert same(xg[i], want["x_grads"][i])
    assert edges == want["edges"]
    # non-vacuity: the gradients are not all zero
    assert any(np.abs(w).max() > 0 for w in wg)


def test_ifelse_counters(orc):
    """aggregate_pull_filtered counters: traversed + skipped = m, groups
    executed + skipped = total groups (aggregate.hpp:139-162), traversed =
    sum over N^1 of |N(v) & V_t| (test_engine.cpp:303-340)."""
    g, vt, x0, ws, r = chain_inputs(orc, 1024, 8192, 7, 0.1, 2, 8, 8, 4)
    levels = orc.compute_frontiers(g, vt, 2)
    da = np.zeros(g.n, np.uint8)
    da[levels[1]] = 1
    sa = np.zeros(g.n, np.uint8)
    sa[levels[0]] = 1
    _, c = orc.aggregate_pull_filtered_f32(g.offsets, g.neighbors, g.weights, x0, da, sa, 3)
    deg = np.diff(g.offsets.astype(np.int64))
    assert c["edges_traversed"] + c["edges_skipped"] == g.m
    assert c["groups_executed"] + c["groups_skipped"] == int(((deg + 2) // 3).sum())
    vts = set(levels[0].tolist())
    want = sum(sum(1 for u in g.neighbors[g.offsets[v]:g.offsets[v + 1]] if int(u) in vts) for v in levels[1])
    assert c["edges_traversed"] == want
