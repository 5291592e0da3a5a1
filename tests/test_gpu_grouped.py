"""CommitMode::Fast on the group-partitioned kernel (PG_AGG_GROUPED,
aggregate.hpp:84-115) and the measured gs oracle on the device
(train.hpp:35-54). Fast re-associates across the groups
of a destination (atomics), so it is checked against the f64 oracle with the
conditioning-aware fp32 bound; with gs >= max degree every destination owns
one group and the result is bit-equal to Deterministic. The default grouped
kernel (tuning grouped_seg 0) is atomic-free: whole-destination CTA ranges,
records staged by TMA bulk copy, a segmented reduction in group order and a
slice-order fixup for hub destinations — deterministic run to run."""
import numpy as np
import pytest

from conftest import rmat_pairs

pytestmark = pytest.mark.gpu


def setup(pg, orc, n=2048, m=30000, seed=3, ratio=0.2):
    pairs, n_pad = rmat_pairs(orc, n, m, seed)
    g = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
    vt = pg.sample_training_set(n_pad, ratio, 42)
    F = pg.compute_frontiers(g, vt, 2)
    paths = pg.prepare_all_paths(g, F)
    og = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
    ops = orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, 2))
    return g, paths, og, ops


@pytest.mark.parametrize("seg", [0, 1, 2])
@pytest.mark.parametrize("dim", [16, 41, 602])
def test_grouped_within_tolerance(pg, orc, cuda, dim, seg):
    import torch

    pg.set_tuning("grouped_seg", seg)
    g, paths, og, ops = setup(pg, orc)
    for p, op in zip(paths, ops):
        y = np.random.default_rng(dim).uniform(-1, 1, size=(p.P, dim)).astype(np.float32)
        yd = pg.empty_rows(p.P, dim)
        yd.copy_(torch.from_numpy(y))
        yu = y[op.srcpos]
        want64 = orc.aggregate_pull_f64(op.offsets, op.neighbors, op.weights, yu.astype(np.float64))
        absum = orc.aggregate_pull_f64(op.offsets, op.neighbors, np.abs(op.weights), np.abs(yu).astype(np.float64))
        det = pg.empty_rows(p.D, dim)
        pg.backward_aggregation(pg.group_neighbors(p, 1), yd, det, overwrite=True)
        for gs in (1, 3, 16, 64, max(p.max_degree, 1)):
            G = pg.group_neighbors(p, gs)
            x = pg.empty_rows(p.D, dim)
            x.fill_(7.0)  # overwrite zeroes first
            pg.backward_aggregation(G, yd, x, mode=pg.GROUPED, overwrite=True)
            torch.cuda.synchronize()
            xh = x.cpu().numpy()
            err = np.abs(xh.astype(np.float64) - want64)
            assert (err <= 1e-6 + 1e-5 * absum).all(), (gs, dim, float(err.max()))
            if gs >= p.max_degree:  # one group per destination: the serial order, bit for bit
                assert np.array_equal(xh.view(np.uint32), det.cpu().numpy().view(np.uint32))
        # accumulate semantics: out += A y
        G = pg.group_neighbors(p, 8)
        x = pg.empty_rows(p.D, dim)
        x.fill_(1.0)
        pg.backward_aggregation(G, yd, x, mode=pg.GROUPED)
        torch.cuda.synchronize()
        err = np.abs(x.cpu().numpy().astype(np.float64) - (want64 + 1.0))
        assert (err <= 2e-6 + 1e-5 * (absum + 1.0)).all()
    pg.set_tuning("grouped_seg")


def test_grouped_graph_forward_pull(pg, orc, cuda):
    import torch

    g, paths, og, ops = setup(pg, orc)
    dim = 33
    x0 = np.random.default_rng(1).uniform(0, 1, size=(g.n, dim)).astype(np.float32)
    xd = pg.empty_rows(g.n, dim)
    xd.copy_(torch.from_numpy(x0))
    out = pg.empty_rows(g.n, dim)
    pg.aggregate_pull(pg.group_neighbors(g, 5), xd, out, mode=pg.GROUPED, overwrite=True)
    torch.cuda.synchronize()
    want = orc.aggregate_pull_f64(og.offsets, og.neighbors, og.weights, x0.astype(np.float64))
    absum = orc.aggregate_pull_f64(og.offsets, og.neighbors, np.abs(og.weights), x0.astype(np.float64))
    assert (np.abs(out.cpu().numpy() - want) <= 1e-6 + 1e-5 * absum).all()


def test_grouped_rejects_row_ranges(pg, orc, cuda):
    g, paths, og, ops = setup(pg, orc)
    p = paths[1]
    yd = pg.empty_rows(p.P, 16)
    x = pg.empty_rows(10, 16)
    with pytest.raises(pg.ConfigError):
        pg.backward_aggregation(pg.group_neighbors(p, 4), yd, x, mode=pg.GROUPED, rows=(0, 10))


def test_measured_oracle(pg, orc, cuda):
    g, paths, og, ops = setup(pg, orc)
    p = paths[1]
    best, table = pg.oracle_gs_measured(p, 64, repeats=3)
    cands = pg.default_gs_candidates(p.max_degree).tolist()
    assert [gs for gs, _ in table] == cands
    assert best in cands and all(t > 0 for _, t in table)
    tmin = min(t for _, t in table)
    assert dict(table)[best] == tmin
    assert pg.choose_gs("oracle:measured", p, 64) in cands


@pytest.mark.parametrize("dim", [16, 100, 602])
def test_grouped_atomic_free_hubs_and_determinism(pg, orc, cuda, dim):
    """Hub destinations with more groups than a CTA range takes and more
    edges than its staging window (sliced, combined by the fixup kernel),
    odd widths, small and large gs: within tolerance of f64, bit-identical
    across repeated runs (no atomics), and bit-equal to Deterministic when
    every destination owns one group."""
    import torch

    g, paths, og, ops = setup(pg, orc, n=16384, m=16384 * 64, seed=5, ratio=0.5)
    p, op = paths[1], ops[1]
    assert p.max_degree > 4096  # a hub past the 4096-record staging window
    y = np.random.default_rng(dim + 1).uniform(-1, 1, size=(p.P, dim)).astype(np.float32)
    yd = pg.empty_rows(p.P, dim)
    yd.copy_(torch.from_numpy(y))
    yu = y[op.srcpos]
    want64 = orc.aggregate_pull_f64(op.offsets, op.neighbors, op.weights, yu.astype(np.float64))
    absum = orc.aggregate_pull_f64(op.offsets, op.neighbors, np.abs(op.weights), np.abs(yu).astype(np.float64))
    det = pg.empty_rows(p.D, dim)
    pg.backward_aggregation(pg.group_neighbors(p, 1), yd, det, overwrite=True)
    torch.cuda.synchronize()
    for gs in (1, 2, 7, 42, 256, 1 << 20):
        G = pg.group_neighbors(p, gs)
        runs = []
        for _ in range(2):
            x = pg.empty_rows(p.D, dim)
            x.fill_(float("nan"))
            pg.backward_aggregation(G, yd, x, mode=pg.GROUPED, overwrite=True)
            torch.cuda.synchronize()
            runs.append(x.cpu().numpy())
        assert np.array_equal(runs[0].view(np.uint32), runs[1].view(np.uint32)), gs
        # groups handed to workers dynamically (tuning grp_dynamic): the
        # partials and their reduction order are the same, so the same bits
        try:
            for dyn in (0, 1):
                pg.set_tuning("grp_dynamic", dyn)
                x = pg.empty_rows(p.D, dim)
                pg.backward_aggregation(G, yd, x, mode=pg.GROUPED, overwrite=True)
                torch.cuda.synchronize()
                assert np.array_equal(x.cpu().numpy().view(np.uint32), runs[0].view(np.uint32)), (gs, dyn)
        finally:
            pg.set_tuning("grp_dynamic")
        err = np.abs(runs[0].astype(np.float64) - want64)
        assert (err <= 1e-6 + 1e-5 * absum).all(), (gs, float((err / (1e-6 + 1e-5 * absum)).max()))
        if gs >= p.max_degree:
            assert np.array_equal(runs[0].view(np.uint32), det.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("dim", [41, 602])
def test_grouped_source_segments_within_tolerance(pg, orc, cuda, dim):
    """The atomic-free grouped kernel over L2-sized source segments (tuning
    grouped_src_segs, forced here with src_segs = 3): each pass takes every
    group's part of one segment and adds its partials to the output — a
    further re-association, still inside the Fast-mode bound."""
    import torch

    g, paths, og, ops = setup(pg, orc, m=60000)
    try:
        pg.set_tuning("src_segs", 3)
        for p, op in zip(paths, ops):
            y = np.random.default_rng(dim + 5).uniform(-1, 1, size=(p.P, dim)).astype(np.float32)
            yd = pg.empty_rows(p.P, dim)
            yd.copy_(torch.from_numpy(y))
            yu = y[op.srcpos]
            want64 = orc.aggregate_pull_f64(op.offsets, op.neighbors, op.weights, yu.astype(np.float64))
            absum = orc.aggregate_pull_f64(op.offsets, op.neighbors, np.abs(op.weights),
                                           np.abs(yu).astype(np.float64))
            for gs in (32, 64, max(p.max_degree, 32)):
                for segs in (1, 0):
                    pg.set_tuning("grouped_src_segs", segs)
                    x = pg.empty_rows(p.D, dim)
                    x.fill_(7.0)
                    pg.backward_aggregation(pg.group_neighbors(p, gs), yd, x, mode=pg.GROUPED, overwrite=True)
                    torch.cuda.synchronize()
                    err = np.abs(x.cpu().numpy().astype(np.float64) - want64)
                    assert (err <= 1e-6 + 1e-5 * absum).all(), (gs, segs, dim, float(err.max()))
    finally:
        pg.set_tuning("src_segs")
        pg.set_tuning("grouped_src_segs")
