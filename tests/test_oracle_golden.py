"""Pins the C oracle (oracle/pathgcn_oracle.c) against the reference's own
known-answer tests (proj/tests/unit/*.cpp, proj/tests/acceptance/acceptance.cpp,
proj/tests/cli/test_cli.cpp) and the survey's frozen fixture values."""
import numpy as np
import pytest

from conftest import GEX_PAIRS, GEX_VT, random_graph_pairs, rmat_pairs, star_pairs


def gex(orc, symnorm=False):
    return orc.build_graph(GEX_PAIRS, symnorm=symnorm)


def edges_of(path):
    """test_execution_path.cpp:14-20 path_edges: {(src global, dst global)}"""
    out = set()
    for d in range(path.D):
        for e in range(int(path.offsets[d]), int(path.offsets[d + 1])):
            out.add((int(path.src[path.neighbors[e]]), int(path.dest[d])))
    return out


# ---------------------------------------------------------------- graph ---

def test_gex_degrees(orc):
    g = gex(orc)
    assert g.n == 5 and g.m == 12
    assert np.diff(g.offsets).tolist() == [1, 4, 2, 3, 2]  # fixtures.hpp:17-18


def test_rmat_frozen_fixture(orc):
    # test_rmat.cpp:72-81: rmat_graph(1024, 8192, 7): n 1024, m 15376, maxdeg 214
    pairs, n_pad = rmat_pairs(orc, 1024, 8192, 7)
    g = orc.build_graph(pairs, n_hint=n_pad)
    assert (g.n, g.m, g.max_degree()) == (1024, 15376, 214)
    assert orc.graph_fingerprint(g) == 0x783D36DC470444FA  # SURVEY §8c probe


def test_rmat_degenerate_quadrant(orc):
    # test_rmat.cpp:8-21
    pairs, _ = orc.gen_rmat(4, 3, 1.0, 0.0, 0.0, 0.0, 123)
    assert (pairs == 0).all()


def test_rmat_pads_to_power_of_two(orc):
    # test_rmat.cpp:58-70
    pairs, n_pad = orc.gen_rmat(100, 50, 0.57, 0.19, 0.19, 0.05, 1)
    assert n_pad == 128 and pairs.max() < 128


def test_empty_edge_list_needs_hint(orc):
    with pytest.raises(ValueError):
        orc.build_graph(np.zeros((0, 2), np.uint32))
    g = orc.build_graph(np.zeros((0, 2), np.uint32), n_hint=4)
    assert g.n == 4 and g.m == 0


def test_self_loops_and_duplicates(orc):
    g = orc.build_graph(np.array([[0, 0], [0, 1], [1, 0], [0, 1], [2, 2]], np.uint32))
    assert g.n == 2 and g.m == 2  # n = 1 + max id over non-self-loop pairs


def test_symnorm_weights(orc):
    g = gex(orc, symnorm=True)
    # weight(0->1) = 1/sqrt(1*4)
    assert g.weights[0] == 1.0 / np.sqrt(4.0)
    # symmetric
    for u in range(g.n):
        for e in range(int(g.offsets[u]), int(g.offsets[u + 1])):
            v = g.neighbors[e]
            row = g.neighbors[g.offsets[v]:g.offsets[v + 1]]
            back = int(g.offsets[v]) + int(np.searchsorted(row, u))
            assert g.weights[back] == g.weights[e]


# ------------------------------------------------------------ frontiers ---

def test_frontiers_worked_example(orc):
    # test_frontier.cpp:10-18
    lv = orc.compute_frontiers(gex(orc), GEX_VT, 2)
    assert [x.tolist() for x in lv] == [[2, 4], [1, 3], [0, 1, 2, 3, 4]]


def test_frontiers_walk_semantics(orc):
    # test_frontier.cpp:20-30
    g = orc.build_graph(np.array([[0, 1]], np.uint32))
    lv = orc.compute_frontiers(g, np.array([0], np.uint32), 2)
    assert lv[1].tolist() == [1] and lv[2].tolist() == [0]


def test_frontiers_errors(orc):
    # test_frontier.cpp:32-39
    with pytest.raises(ValueError):
        orc.compute_frontiers(gex(orc), np.array([], np.uint32), 2)
    with pytest.raises(ValueError):
        orc.compute_frontiers(gex(orc), np.array([0], np.uint32), 0)


@pytest.mark.parametrize("seed", range(6))
def test_frontiers_brute_force(orc, seed):
    # test_frontier.cpp:41-57
    g = orc.build_graph(random_graph_pairs(200, 800, seed), n_hint=200)
    vt = orc.sample_training_set(g.n, 0.1, seed)
    lv = orc.compute_frontiers(g, vt, 3)
    cur = set(vt.tolist())
    for k in range(1, 4):
        nxt = set()
        for v in cur:
            nxt.update(g.neighbors[g.offsets[v]:g.offsets[v + 1]].tolist())
        assert lv[k].tolist() == sorted(nxt)
        cur = nxt


# --------------------------------------------------------------- paths ---

def test_path_worked_example(orc):
    # test_execution_path.cpp:23-47, dump string :228-235
    g = gex(orc)
    lv = orc.compute_frontiers(g, GEX_VT, 2)
    sg1 = orc.extract_path(g, lv, 1)
    assert sg1.dest.tolist() == [1, 3] and sg1.offsets.tolist() == [0, 2, 4]
    assert edges_of(sg1) == {(2, 1), (4, 1), (2, 3), (4, 3)}
    assert (sg1.D, sg1.S, sg1.E) == (2, 2, 4)
    sg0 = orc.extract_path(g, lv, 0)
    assert sg0.dest.tolist() == [0, 1, 2, 3, 4] and sg0.E == 7
    assert edges_of(sg0) == {(1, 0), (3, 1), (1, 2), (3, 2), (1, 3), (1, 4), (3, 4)}
    # CLI prepare: SG_1: 2 dests / 4 edges, SG_0: 5 dests / 7 edges (test_cli.cpp:111-131)
    paths = orc.prepare_all_paths(g, lv)
    assert [(p.layer, p.D, p.E) for p in paths] == [(1, 2, 4), (0, 5, 7)]


def test_path_isolated_training_vertex(orc):
    # test_execution_path.cpp:68-82
    g = orc.build_graph(np.array([[0, 1]], np.uint32), n_hint=3)
    lv = orc.compute_frontiers(g, np.array([2], np.uint32), 2)
    paths = orc.prepare_all_paths(g, lv)
    assert paths[0].D == 0 and paths[0].E == 0 and paths[1].D == 0


def test_path_star(orc):
    # test_execution_path.cpp:84-99
    g = orc.build_graph(star_pairs(4))
    lv = orc.compute_frontiers(g, np.array([1], np.uint32), 2)
    sg1 = orc.extract_path(g, lv, 1)
    assert sg1.dest.tolist() == [0] and sg1.E == 1
    sg0 = orc.extract_path(g, lv, 0)
    assert sg0.D == 4 and sg0.E == 4


def test_full_training_set_gives_whole_graph(orc):
    # test_execution_path.cpp:60-66
    pairs, n_pad = rmat_pairs(orc, 256, 1024, 5)
    g = orc.build_graph(pairs, n_hint=n_pad)
    vt = orc.sample_training_set(g.n, 1.0, 0)
    for p in orc.prepare_all_paths(g, orc.compute_frontiers(g, vt, 2)):
        assert p.E == g.m


@pytest.mark.parametrize("seed", range(5))
def test_paths_brute_force(orc, seed):
    # test_execution_path.cpp:101-120
    g = orc.build_graph(random_graph_pairs(128, 512, seed + 100), n_hint=128)
    vt = orc.sample_training_set(g.n, 0.1, seed)
    L = 2 + seed % 2
    lv = orc.compute_frontiers(g, vt, L)
    for l in range(L):
        p = orc.extract_path(g, lv, l)
        dests, parents = set(lv[L - l].tolist()), set(lv[L - l - 1].tolist())
        expect = {(int(u), v) for v in dests for u in g.neighbors[g.offsets[v]:g.offsets[v + 1]] if int(u) in parents}
        assert edges_of(p) == expect
        # src maps bijective, src_pos_in_parent exact (:159-179)
        assert (np.diff(p.src.astype(np.int64)) > 0).all()
        assert set(p.neighbors.tolist()) == set(range(p.S))
        assert (lv[L - l - 1][p.srcpos] == p.src).all()


def test_probe_fixture_values(orc):
    # RMAT(1024, 8192, 7), ratio 0.1 seed 42: |V_t|=102, |N1|=581,
    # |N2|=980; SG_1 E=1474 |S|=99; SG_0 E=13074 |S|=581; regression gs 2 / 9
    pairs, n_pad = rmat_pairs(orc, 1024, 8192, 7)
    g = orc.build_graph(pairs, n_hint=n_pad)
    vt = orc.sample_training_set(g.n, 0.1, 42)
    lv = orc.compute_frontiers(g, vt, 2)
    assert [len(x) for x in lv] == [102, 581, 980]
    sg1, sg0 = orc.prepare_all_paths(g, lv)
    assert (sg1.E, sg1.S, sg0.E, sg0.S) == (1474, 99, 13074, 581)
    assert orc.path_regression_gs(sg1.D, sg1.E) == 2 and orc.path_regression_gs(sg0.D, sg0.E) == 9
    # SG_0 src_pos_in_parent is the identity (every parent vertex referenced)
    assert (sg0.srcpos == np.arange(sg0.S)).all()


# ------------------------------------------------------------- grouping ---

def test_grouping_gex_gs3(orc):
    # test_grouping.cpp:8-18, acceptance C3
    g = gex(orc)
    gr = orc.group_neighbors(g.offsets, 3)
    assert len(gr.dest) == 6
    assert gr.dest_groups[2] - gr.dest_groups[1] == 2
    first, second = int(gr.dest_groups[1]), int(gr.dest_groups[1]) + 1
    assert gr.end[first] - gr.begin[first] == 3 and gr.end[second] - gr.begin[second] == 1


def test_grouping_extremes(orc):
    # test_grouping.cpp:20-33
    g = gex(orc)
    assert len(orc.group_neighbors(g.offsets, g.max_degree()).dest) == 5
    assert len(orc.group_neighbors(g.offsets, 1).dest) == g.m
    with pytest.raises(ValueError):
        orc.group_neighbors(g.offsets, 0)


def test_grouping_coverage(orc):
    # test_grouping.cpp:40-61
    pairs, n_pad = rmat_pairs(orc, 256, 2048, 3)
    g = orc.build_graph(pairs, n_hint=n_pad)
    for gs in range(1, g.max_degree() + 2):
        gr = orc.group_neighbors(g.offsets, gs)
        deg = np.diff(g.offsets)
        assert len(gr.dest) == int(((deg + gs - 1) // gs).sum())
        for v in range(0, g.n, 17):
            cur = g.offsets[v]
            for k in range(int(gr.dest_groups[v]), int(gr.dest_groups[v + 1])):
                assert gr.dest[k] == v and gr.begin[k] == cur and 1 <= gr.end[k] - gr.begin[k] <= gs
                cur = gr.end[k]
            assert cur == g.offsets[v + 1]


# ------------------------------------------------------------ gs models ---

@pytest.mark.parametrize("n,e,gs", [(2708, 5278, 2), (3327, 4552, 2), (19717, 44324, 2), (81306, 1342296, 10),
                                    (88784, 2093195, 12), (410236, 2439437, 6), (875713, 4322051, 9),
                                    (1134890, 2987624, 15)])
def test_regression_published(orc, n, e, gs):
    # test_gs_model.cpp:47-58 / acceptance C4
    assert orc.regression_gs(n, e, e / n) == gs


def test_regression_clamps(orc):
    # test_gs_model.cpp:60-75
    assert orc.regression_gs(0, 0, 0.0) == 1
    for e in (0.0, 1e5, 1e9):
        assert orc.regression_gs(1, int(e), e) >= 1


def test_cost_model_known_answers(orc):
    g = gex(orc)
    # test_group_cost.cpp:7-13
    assert orc.grouping_cost(g.offsets, g.max_degree(), 16, 1, 1.0) == g.m * 16
    # test_group_cost.cpp:15-20
    assert orc.grouping_cost(g.offsets, 1, 1, 12, 1.0) == 8.0


def test_cost_model_hub(orc):
    # test_group_cost.cpp:60-68 / CLI "chosen gs = 8" (test_cli.cpp:150-170)
    g = orc.build_graph(star_pairs(64))
    cands = orc.default_candidates(g.max_degree())
    best, table = orc.oracle_gs_cost(g.offsets, cands, 16, 8, 0.1)
    assert best == 8 and len(table) == 7
    assert table[3] == pytest.approx(267.2)


def test_candidates_and_ties(orc):
    # test_group_cost.cpp:77-84
    assert orc.default_candidates(4).tolist() == [1, 2, 4]
    assert orc.default_candidates(5).tolist() == [1, 2, 4, 8]
    assert orc.default_candidates(1).tolist() == [1]
    assert orc.default_candidates(0).tolist() == [1]
    best, table = orc.oracle_gs_cost(gex(orc).offsets, [3], 4, 4, 0.25)
    assert best == 3 and len(table) == 1


def test_lambda_monotone(orc):
    # test_group_cost.cpp:22-38
    pairs, n_pad = rmat_pairs(orc, 256, 2048, 13)
    for g in (gex(orc), orc.build_graph(pairs, n_hint=n_pad)):
        prev = 0
        cands = orc.default_candidates(g.max_degree())
        for lam in (0.0, 0.05, 0.1, 0.25, 0.5, 1.0, 2.0, 10.0):
            gs, _ = orc.oracle_gs_cost(g.offsets, cands, 16, 8, lam)
            assert gs >= prev
            prev = gs


# ---------------------------------------------------------- aggregation ---

def test_aggregate_hand_sums(orc):
    # test_engine.cpp:72-80
    g = gex(orc)
    x = np.array([[1], [2], [3], [4], [5]], np.float64)
    y = orc.aggregate_pull_f64(g.offsets, g.neighbors, g.weights, x)
    assert y[:, 0].tolist() == [2, 13, 6, 10, 6]
    y32 = orc.aggregate_pull_f32(g.offsets, g.neighbors, g.weights, x.astype(np.float32))
    assert y32[:, 0].tolist() == [2, 13, 6, 10, 6]


def test_aggregate_sg1_hand_case(orc):
    # test_engine.cpp:169-180
    g = gex(orc)
    lv = orc.compute_frontiers(g, GEX_VT, 2)
    sg1 = orc.extract_path(g, lv, 1)
    y = orc.aggregate_pull_f64(sg1.offsets, sg1.neighbors, sg1.weights, np.array([[1.0], [2.0]]))
    assert y[:, 0].tolist() == [3.0, 3.0]


def test_aggregate_zero_and_negative_zero(orc):
    # test_engine.cpp:82-88 and the +T(0) canonicalisation (aggregate.hpp:82)
    g = gex(orc)
    x = -np.zeros((5, 3), np.float32)
    y = orc.aggregate_pull_f32(g.offsets, g.neighbors, g.weights, x)
    assert (y == 0).all() and not np.signbit(y).any()


def test_work_counter_brute_force(orc):
    # test_engine.cpp:303-340: SG_1 edges = sum_{v in N1} |N(v) ∩ Vt|
    pairs, n_pad = rmat_pairs(orc, 1024, 8192, 7)
    g = orc.build_graph(pairs, n_hint=n_pad)
    vt = orc.sample_training_set(g.n, 0.1, 42)
    lv = orc.compute_frontiers(g, vt, 2)
    vts = set(vt.tolist())
    expect = sum(1 for v in lv[1] for u in g.neighbors[g.offsets[v]:g.offsets[v + 1]] if int(u) in vts)
    assert orc.prepare_all_paths(g, lv)[0].E == expect < g.m


def test_gemm_a_bt_ascending_k(orc):
    a = np.array([[1.0, 2.0, 3.0]], np.float32)
    b = np.array([[1.0, 1.0, 1.0], [0.5, 0.0, -1.0]], np.float32)
    assert orc.gemm_a_bt_f32(a, b).tolist() == [[6.0, -2.5]]


def test_fingerprints(orc):
    g = gex(orc)
    a = orc.path_fingerprint(g, GEX_VT, 2)
    assert a != orc.path_fingerprint(g, GEX_VT, 3)
    assert a != orc.path_fingerprint(g, np.array([2], np.uint32), 2)
