"""Parity at BASELINE.json's named configurations (the same synthetic inputs
bench.py builds): Cora-shaped (configs[0]), Pubmed-shaped (configs[1]) and
ogbn-arxiv-shaped (configs[2]) — graph, frontiers, both execution paths,
regression-gs groups and the cost-model gs table bit-exact against the C
oracle; the backward-aggregation stage bit-exact at the config's widths; and
for Cora / Pubmed the whole chain (forward incl. softmax, top_grad,
backward_epp W') at the real feature widths (1433 / 500)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def build(pg, orc, name):
    import bench

    cfg = bench.CONFIGS[name]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    L = len(cfg["dims"])
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    prep = pg.prepare_paths(g, vt, L, bench.agg_dims(cfg))
    og = orc.build_graph(pairs, n_hint=cfg["V"], symnorm=True)
    levels = orc.compute_frontiers(og, vt, L)
    ops = orc.prepare_all_paths(og, levels)
    return cfg, vt, g, prep, og, levels, ops, bench.agg_dims(cfg)


@pytest.mark.parametrize("name", ["cora", "pubmed", "arxiv"])
def test_config_structures_and_stage(pg, orc, name):
    import torch

    cfg, vt, g, prep, og, levels, ops, dims = build(pg, orc, name)
    assert g.n == cfg["V"] and g.m == cfg["m"] == og.m
    offs, nb, w = g.export()
    assert np.array_equal(offs, og.offsets) and np.array_equal(nb, og.neighbors)
    assert np.array_equal(w.view(np.uint64), og.weights.view(np.uint64))
    for k, lv in enumerate(levels):
        assert np.array_equal(prep.frontiers.level(k), lv)
    for i, (p, op) in enumerate(zip(prep.paths, ops)):
        x = p.export()
        for f in ("dest", "src", "srcpos", "offsets", "neighbors"):
            assert np.array_equal(x[f], getattr(op, f)), (name, i, f)
        assert np.array_equal(x["weights"].view(np.uint64), op.weights.view(np.uint64))
        gs = orc.path_regression_gs(op.D, op.E)
        assert prep.gs[i] == gs
        gx = prep.groups[i].export()
        og_ = orc.group_neighbors(op.offsets, gs)
        assert np.array_equal(gx["dest_groups"], og_.dest_groups)
        assert np.array_equal(gx["begin"], og_.begin) and np.array_equal(gx["end"], og_.end)
        best, table = pg.oracle_gs(p, dims[i], 8, 0.25)
        obest, otable = orc.oracle_gs_cost(op.offsets, [c for c, _ in table], dims[i], 8, 0.25)
        assert best == obest and [c for _, c in table] == list(otable)
        # the timed stage (engine.hpp:331-338) at the config's width
        y = np.random.default_rng(i).uniform(-1, 1, size=(p.P, dims[i])).astype(np.float32)
        yd = pg.empty_rows(p.P, dims[i])
        yd.copy_(torch.from_numpy(y))
        xd = pg.empty_rows(p.D, dims[i])
        pg.backward_aggregation(prep.groups[i], yd, xd, overwrite=True)
        torch.cuda.synchronize()
        want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
        assert np.array_equal(bits(xd.cpu().numpy()), bits(want)), (name, i)


@pytest.mark.parametrize("name", ["cora", "pubmed"])
def test_config_chain(pg, orc, name):
    import torch

    cfg, vt, g, prep, og, levels, ops, dims = build(pg, orc, name)
    f, hid = cfg["f"], cfg["dims"]
    rng = np.random.default_rng(11)
    x0 = rng.uniform(0, 1, size=(g.n, f)).astype(np.float32)
    ins = [f] + hid[:-1]
    ws = [rng.uniform(-0.1, 0.1, size=(ins[l], hid[l])).astype(np.float32) for l in range(len(hid))]
    r = np.zeros((g.n, hid[-1]), np.float32)
    r[vt, rng.integers(0, hid[-1], size=len(vt))] = 1

    def dev(a):
        t = pg.empty_rows(a.shape[0], a.shape[1])
        t.copy_(torch.from_numpy(a))
        return t

    wd = [dev(w) for w in ws]
    arts = pg.forward(pg.group_neighbors(g, 4), dev(x0), wd)
    top = pg.empty_rows(g.n, hid[-1])
    pg.top_grad_from_probs(arts.x[-1], dev(r), torch.from_numpy(vt.astype(np.int32)).cuda(), top)
    wg = pg.backward_epp(prep, arts, top, wd)
    torch.cuda.synchronize()
    oa = orc.forward(og, x0, ws)
    otop = orc.top_grad_f32(oa["x"][-1], r, vt)
    owg, _, _ = orc.backward_epp(ops, levels, oa, otop, ws, "local")
    assert np.array_equal(bits(arts.x[-1].cpu().numpy()), bits(oa["x"][-1]))
    assert np.array_equal(bits(top.cpu().numpy()), bits(otop))
    for l in range(len(hid)):
        assert np.array_equal(bits(wg[l].cpu().numpy()), bits(owg[l])), (name, l)
    assert max(float(np.abs(w).max()) for w in owg) > 0
