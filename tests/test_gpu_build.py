"""GPU parity: graph load, frontiers, execution paths, groups and the gs
selector on device vs the C oracle (and the reference's golden vectors).
Every integer structure and every f64 weight must be bit-exact."""
import os

import numpy as np
import pytest

from conftest import GEX_PAIRS, GEX_VT, random_graph_pairs, rmat_pairs, star_pairs

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


def same_graph(dg, og):
    offs, nb, w = dg.export()
    assert dg.n == og.n and dg.m == og.m
    assert np.array_equal(offs, og.offsets)
    assert np.array_equal(nb, og.neighbors)
    assert np.array_equal(w.view(np.uint64), og.weights.view(np.uint64))


def same_path(dp, op):
    x = dp.export()
    assert (dp.D, dp.S, dp.E) == (op.D, op.S, op.E)
    for f in ("dest", "src", "srcpos", "offsets", "neighbors"):
        assert np.array_equal(x[f], getattr(op, f)), f
    assert np.array_equal(x["weights"].view(np.uint64), op.weights.view(np.uint64))


def cases(orc):
    yield GEX_PAIRS, None, GEX_VT
    yield star_pairs(64), None, np.array([1], np.uint32)
    yield np.array([[0, 1]], np.uint32), 3, np.array([2], np.uint32)  # isolated training vertex
    pairs, n_pad = rmat_pairs(orc, 1024, 8192, 7)
    yield pairs, n_pad, orc.sample_training_set(1024, 0.1, 42)
    for seed in range(3):
        yield random_graph_pairs(200, 800, seed), 200, orc.sample_training_set(200, 0.1, seed)
    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 4, 11)
    yield pairs, n_pad, orc.sample_training_set(4096, 0.5, 3)
    pairs, n_pad = rmat_pairs(orc, 20000, 200000, 5)
    yield pairs, n_pad, orc.sample_training_set(20000, 0.01, 9)  # sparse frontier (push path)
    yield pairs, n_pad, orc.sample_training_set(20000, 1.0, 9)  # full training set


@pytest.mark.parametrize("symnorm", [False, True])
def test_graph_build_bit_exact(pg, orc, symnorm):
    for pairs, n_hint, _ in cases(orc):
        dg = pg.build_undirected_csr(pairs, n_hint=n_hint, weights="symnorm" if symnorm else "unit")
        og = orc.build_graph(pairs, n_hint=n_hint, symnorm=symnorm)
        same_graph(dg, og)
        assert dg.fingerprint() == orc.graph_fingerprint(og)
        assert dg.max_degree() == og.max_degree()


def test_graph_build_edge_cases(pg, orc):
    with pytest.raises(pg.ConfigError):
        pg.build_undirected_csr(np.zeros((0, 2), np.uint32))
    g = pg.build_undirected_csr(np.zeros((0, 2), np.uint32), n_hint=4)
    assert g.n == 4 and g.m == 0
    g = pg.build_undirected_csr(np.array([[5, 5], [1, 0], [0, 1]], np.uint32))
    assert g.n == 2 and g.m == 2  # self loop ignored for n


def test_graph_upload_validation(pg, orc):
    og = orc.build_graph(GEX_PAIRS, symnorm=True)
    dg = pg.graph_from_csr(og.n, og.offsets, og.neighbors, og.weights)
    same_graph(dg, og)
    bad = og.neighbors.copy()
    bad[0] = 4  # 0->4 without 4->0
    with pytest.raises(pg.ConfigError):
        pg.graph_from_csr(og.n, og.offsets, bad, og.weights)
    w = og.weights.copy()
    w[0] = 0.3
    with pytest.raises(pg.ConfigError):
        pg.graph_from_csr(og.n, og.offsets, og.neighbors, w)


def test_frontiers_paths_groups_bit_exact(pg, orc):
    for pairs, n_hint, vt in cases(orc):
        for L in (2, 3, 4):
            og = orc.build_graph(pairs, n_hint=n_hint, symnorm=True)
            dg = pg.build_undirected_csr(pairs, n_hint=n_hint, weights="symnorm")
            lv = orc.compute_frontiers(og, vt, L)
            F = pg.compute_frontiers(dg, vt, L)
            for k in range(L + 1):
                assert np.array_equal(F.level(k), lv[k]), (k, L)
            assert pg.path_fingerprint(dg, vt, L) == orc.path_fingerprint(og, vt, L)
            for dp, op in zip(pg.prepare_all_paths(dg, F), orc.prepare_all_paths(og, lv)):
                assert dp.layer == op.layer
                same_path(dp, op)
                maxdeg = int(np.diff(op.offsets).max(initial=0))
                assert dp.max_degree == maxdeg
                for gs in (1, 2, 3, 9, max(maxdeg, 1), maxdeg + 1):
                    G = pg.group_neighbors(dp, gs)
                    og_ = orc.group_neighbors(op.offsets, gs)
                    x = G.export()
                    assert G.group_count() == len(og_.dest)
                    for f in ("dest", "begin", "end", "dest_groups"):
                        assert np.array_equal(x[f], getattr(og_, f)), (f, gs)
                assert pg.path_regression_gs(dp) == orc.path_regression_gs(op.D, op.E)


def test_frontier_errors(pg):
    g = pg.build_undirected_csr(GEX_PAIRS)
    with pytest.raises(pg.ConfigError):
        pg.compute_frontiers(g, np.array([], np.uint32), 2)
    with pytest.raises(pg.ConfigError):
        pg.compute_frontiers(g, GEX_VT, 0)
    with pytest.raises(pg.ConfigError):
        pg.compute_frontiers(g, np.array([7], np.uint32), 2)
    F = pg.compute_frontiers(g, GEX_VT, 2)
    with pytest.raises(pg.ConfigError):
        pg.extract_execution_path(g, F, 2)
    p = pg.extract_execution_path(g, F, 0)
    with pytest.raises(pg.ConfigError):
        pg.group_neighbors(p, 0)


@pytest.mark.parametrize("dim,W,lam", [(16, 8, 0.25), (602, 3, 0.1), (1, 12, 1.0), (128, 1, 0.0), (16, 5000, 0.25)])
def test_oracle_gs_cost_bit_exact(pg, orc, dim, W, lam):
    for pairs, n_hint, vt in cases(orc):
        og = orc.build_graph(pairs, n_hint=n_hint)
        dg = pg.build_undirected_csr(pairs, n_hint=n_hint)
        F = pg.compute_frontiers(dg, vt, 2)
        for dp, op in zip(pg.prepare_all_paths(dg, F), orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, 2))):
            cands = orc.default_candidates(int(np.diff(op.offsets).max(initial=0)))
            best, table = pg.oracle_gs(dp, dim, W, lam)
            obest, otable = orc.oracle_gs_cost(op.offsets, cands, dim, W, lam)
            assert best == obest
            assert [t[0] for t in table] == cands.tolist()
            assert np.array_equal(np.array([t[1] for t in table]), otable)
            for gs in (1, 4):
                G = pg.group_neighbors(dp, gs)
                assert pg.grouping_cost(G, dim, W, lam) == orc.grouping_cost(op.offsets, gs, dim, W, lam)


def test_hub_oracle_known_answer(pg):
    # test_group_cost.cpp:60-68 on a path that is the star itself: V_t = all
    # leaves' hub neighbourhood. Use the graph grouping cost directly.
    g = pg.build_undirected_csr(star_pairs(64))
    G = pg.group_neighbors(g, 8)
    assert pg.grouping_cost(G, 16, 8, 0.1) == pytest.approx(267.2)


def test_golden_vectors(pg):
    gold = dict(np.load(GOLD))
    n = int(gold["g_n"][0])
    dg = pg.graph_from_csr(n, gold["g_offsets"], gold["g_neighbors"], gold["g_weights"])
    assert dg.fingerprint() == int(gold["g_fp"][0])
    F = pg.compute_frontiers(dg, gold["vt"], 2)
    assert pg.path_fingerprint(dg, gold["vt"], 2) == int(gold["path_fp"][0])
    for k in range(3):
        assert np.array_equal(F.level(k), gold[f"level{k}"])
    for i, p in enumerate(pg.prepare_all_paths(dg, F)):
        x = p.export()
        for f in ("dest", "src", "srcpos", "offsets", "neighbors"):
            assert np.array_equal(x[f], gold[f"p{i}_{f}"])
        assert np.array_equal(x["weights"].view(np.uint64), gold[f"p{i}_weights"].view(np.uint64))
        gs = (2, 9)[i]
        gx = pg.group_neighbors(p, gs).export()
        for f in ("dest", "begin", "end", "dest_groups"):
            assert np.array_equal(gx[f], gold[f"p{i}_g{gs}_{f}"])
        for j, (dim, W, lam) in enumerate(((16, 8, 0.25), (602, 3, 0.1))):
            best, table = pg.oracle_gs(p, dim, W, lam)
            assert best == int(gold[f"p{i}_cost{j}_best"][0])
            assert np.array_equal(np.array([t[1] for t in table]), gold[f"p{i}_cost{j}_table"])
