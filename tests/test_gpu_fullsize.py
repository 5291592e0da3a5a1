"""Full-size parity (BASELINE configs[3], the Reddit-shaped bench workload:
V = 232,965, m = 114,615,892, and configs[4], products-shaped: V = 2,449,029,
m = 61,859,140 at 8 % train — the sparse-frontier regime): at this size the CPU oracle cannot redo the
whole epoch inside a test, so the checks are the size-independent ones —
structural invariants of the device-built paths, bit-exact SpMM rows on a
stride sample of destinations (the oracle restricted to those rows), and
the host-buffer drop-in bit-equal to the device call on every row."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STRIDE = 101


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module", params=["reddit", "products"])
def reddit(pg, request):
    import bench

    cfg = bench.CONFIGS[request.param]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), bench.agg_dims(cfg))
    return cfg, g, vt, prep, bench.agg_dims(cfg)


def test_fullsize_structure(pg, reddit):
    cfg, g, vt, prep, dims = reddit
    assert g.n == cfg["V"] and g.m == cfg["m"]
    F = prep.frontiers
    assert np.array_equal(F.level(0), np.sort(vt))
    for i, p in enumerate(prep.paths):
        x = p.export()
        offs = x["offsets"].astype(np.int64)
        assert p.layer == len(prep.paths) - 1 - i
        assert p.D == F.size(i + 1) and p.P == F.size(i)
        assert np.array_equal(x["dest"], F.level(i + 1))
        deg = np.diff(offs)
        assert offs[0] == 0 and offs[-1] == p.E and (deg >= 1).all()  # walk semantics: every dest keeps an edge
        nb = x["neighbors"].astype(np.int64)
        head = np.zeros(p.E, bool)
        head[offs[:-1]] = True
        assert (np.diff(nb)[~head[1:]] > 0).all()  # strictly ascending local ids per destination
        assert nb.max() < p.S
        src = x["src"].astype(np.int64)
        assert (np.diff(src) > 0).all()
        parent = F.level(i).astype(np.int64)
        assert np.array_equal(parent[x["srcpos"]], src)  # src_pos_in_parent
        if i + 1 == len(prep.paths):  # layer 0: every parent vertex is referenced
            assert p.S == p.P and np.array_equal(x["srcpos"], np.arange(p.P))
        assert np.isfinite(x["weights"]).all() and (x["weights"] > 0).all()
        dg = prep.groups[i].export()["dest_groups"].astype(np.int64)
        gs = prep.gs[i]
        assert np.array_equal(np.diff(dg), (deg + gs - 1) // gs)


def sampled_oracle(orc, x, y, rows):
    offs = x["offsets"].astype(np.int64)
    b, e = offs[rows], offs[rows + 1]
    cnt = e - b
    sub_off = np.zeros(len(rows) + 1, np.uint64)
    sub_off[1:] = np.cumsum(cnt)
    idx = np.repeat(b - sub_off[:-1].astype(np.int64), cnt) + np.arange(int(sub_off[-1]))
    nbr = x["neighbors"][idx]
    w = x["weights"][idx]
    return orc.aggregate_pull_f32(sub_off, x["srcpos"][nbr], w, y)


def test_fullsize_spmm_sampled_rows_bit_exact(pg, orc, reddit):
    import torch

    cfg, g, vt, prep, dims = reddit
    for i, p in enumerate(prep.paths):
        dim = dims[i]
        x = p.export()
        y = np.random.default_rng(17 + i).uniform(-1, 1, size=(p.P, dim)).astype(np.float32)
        yd = pg.empty_rows(p.P, dim)
        yd.copy_(torch.from_numpy(y))
        out = pg.empty_rows(p.D, dim)
        pg.backward_aggregation(prep.groups[i], yd, out, overwrite=True)
        torch.cuda.synchronize()
        rows = np.arange(0, p.D, STRIDE)
        rows = np.union1d(rows, np.argsort(np.diff(x["offsets"].astype(np.int64)))[-16:])  # + the 16 biggest hubs
        got = out[torch.from_numpy(rows).cuda()].cpu().numpy()
        want = sampled_oracle(orc, x, y, rows)
        assert np.array_equal(bits(got), bits(want)), f"path {i}"
        # host-buffer drop-in (pinned, K-segment pipeline) == device call on every row
        yh = torch.from_numpy(y).pin_memory().numpy()
        xh = torch.empty((p.D, dim), dtype=torch.float32).pin_memory().numpy()
        pg.backward_aggregation(prep.groups[i], yh, xh, overwrite=True)
        assert np.array_equal(bits(xh), bits(out.cpu().numpy())), f"host path {i}"
        # other pipeline shapes: source segments K, the last F of them in the chunked last pass
        # (segment balance: 1 equal edges / 0 equal rows; chunk cuts: % edges vs rows)
        for ks, fs, sb, cb, lp in ((3, 1, 0, 100, 0), (4, 2, 1, 50, 0), (3, 3, 1, 0, 40), (5, 2, 0, 0, 40),
                                   (6, 3, 1, 100, 55), (2, 1, 1, 0, 70)):
            knobs = {"host_segs": ks, "host_final_segs": fs, "host_seg_balance": sb, "host_chunk_balance": cb,
                     "host_last_seg_pct": lp}
            for k, v in knobs.items():
                pg.set_tuning(k, v)
            try:
                xh[:] = np.nan
                pg.backward_aggregation(prep.groups[i], yh, xh, overwrite=True)
                assert np.array_equal(bits(xh), bits(out.cpu().numpy())), f"host path {i} {knobs}"
            finally:
                for k in knobs:
                    pg.set_tuning(k, None)
