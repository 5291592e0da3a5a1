"""The oracle against the committed golden vectors produced by the reference
itself (tests/golden/make_golden.py). Runs anywhere (no reference tree)."""
import os

import numpy as np
import pytest

from conftest import rmat_pairs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def test_graph_and_paths(orc, gold):
    pairs, n_pad = rmat_pairs(orc, 1024, 8192, 7)
    g = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
    assert np.array_equal(g.offsets, gold["g_offsets"]) and np.array_equal(g.neighbors, gold["g_neighbors"])
    assert np.array_equal(g.weights.view(np.uint64), gold["g_weights"].view(np.uint64))
    assert orc.graph_fingerprint(g) == int(gold["g_fp"][0])
    vt = orc.sample_training_set(g.n, 0.1, 42)
    assert np.array_equal(vt, gold["vt"])
    assert orc.path_fingerprint(g, vt, 2) == int(gold["path_fp"][0])
    lv = orc.compute_frontiers(g, vt, 2)
    for k in range(3):
        assert np.array_equal(lv[k], gold[f"level{k}"])
    for i, p in enumerate(orc.prepare_all_paths(g, lv)):
        for f in ("dest", "src", "srcpos", "offsets", "neighbors"):
            assert np.array_equal(getattr(p, f), gold[f"p{i}_{f}"]), f
        assert np.array_equal(p.weights.view(np.uint64), gold[f"p{i}_weights"].view(np.uint64))
        gs = (2, 9)[i]
        gr = orc.group_neighbors(p.offsets, gs)
        for f in ("dest", "begin", "end", "dest_groups"):
            assert np.array_equal(getattr(gr, f), gold[f"p{i}_g{gs}_{f}"])
        cands = gold[f"p{i}_cands"]
        assert np.array_equal(orc.default_candidates(int(np.diff(p.offsets).max())), cands)
        for j, (dim, W, lam) in enumerate(((16, 8, 0.25), (602, 3, 0.1))):
            best, table = orc.oracle_gs_cost(p.offsets, cands, dim, W, lam)
            assert best == int(gold[f"p{i}_cost{j}_best"][0])
            assert np.array_equal(table, gold[f"p{i}_cost{j}_table"])
        y = orc.aggregate_pull_f32(p.offsets, p.neighbors, p.weights, gold[f"p{i}_agg_in"])
        assert np.array_equal(y.view(np.uint32), gold[f"p{i}_agg_out"].view(np.uint32))


def test_chain(orc, gold):
    gm = gold["ch_top_g"]
    # the chain fixture runs on the same sym-norm graph and paths
    for i in range(2):
        l = 1 - i
        yg = orc.gemm_a_bt_f32(gm, gold[f"ch_w{l}"])
        assert np.array_equal(yg.view(np.uint32), gold[f"ch_y{i}"].view(np.uint32))
        xg = orc.aggregate_pull_f32(gold[f"p{i}_offsets"], gold[f"p{i}_neighbors"], gold[f"p{i}_weights"],
                                    yg[gold[f"p{i}_srcpos"]])
        assert np.array_equal(xg.view(np.uint32), gold[f"ch_x{i}"].view(np.uint32))
        if l > 0:
            gm = orc.relu_backward_f32(xg, gold["ch_pre0"])
