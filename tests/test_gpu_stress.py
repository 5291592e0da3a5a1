"""Randomised parity sweep of the backward-aggregation stage: random RMAT
graphs, training fractions, widths (odd, 16-byte, wide, multi-chunk) and
scheduling knobs (gather batch, item order, L1/L2 loads, heavy-kernel
routing and threshold, source segments), through the device call, a row
range, and the host-buffer drop-in. Every output row bit-exact with the
fp32 oracle (aggregate_pull<float> Deterministic over the same path)."""
import os

import numpy as np
import pytest

from conftest import rmat_pairs

pytestmark = pytest.mark.gpu

WIDTHS = (1, 3, 16, 17, 41, 64, 100, 128, 129, 300, 602)
KNOBS = {
    "vec_u": (0, 4, 8, 16),
    "chunk_major": (0, 1),
    "ld_cg": (0, 2, 7),
    "heavy_narrow": (0, 1),
    "heavy_wide_pipe": (0, 1, 2, 3, 4, 5),
    "wide_lpd": (16, 32),
    "src_segs": (0, 1, 2, 3),
    "src_seg_balance": (0, 50, 100),
    "heavy_tma": (0, 1),
    "rec_window": (0, 1, 2),
    "row_kernel": (0, 0, 1),
    "row_u": (2, 3, 4),
    "row_seg_mb": (8, 56),
    "vec_block": (256, 256, 512, 1024),
    "vec8": (0, 1, 2, 2),
    "vec8_u": (0, 0, 3, 6),
    "range_side_hubs": (1, 1, 0),
    "grp_dynamic": (0, 1),
    "hub_inline": (0, 1, 1),
    "hub_front_min": (0, 0, 16, 256),
}


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# 240 / 384 / 540 caught a pageable-staging bug (a host copy split across
# 16 threads dropped the last n % 16 bytes when n / 16 was a multiple of 64)
@pytest.mark.parametrize("seed", sorted(set(range(int(os.environ.get("PG_STRESS_SEEDS", "64")))) | {240, 384, 540}))
def test_random_stage_parity(pg, orc, seed):
    import torch

    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(300, 6000))
    deg = int(rng.choice([2, 6, 24, 64]))
    pairs, n_pad = rmat_pairs(orc, n, n * deg, 50 + seed)
    vt = orc.sample_training_set(n_pad, float(rng.choice([0.01, 0.1, 0.5, 1.0])), seed)
    L = int(rng.integers(1, 4))
    dg = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm" if seed % 3 else "unit")
    og = orc.build_graph(pairs, n_hint=n_pad, symnorm=bool(seed % 3))
    F = pg.compute_frontiers(dg, vt, L)
    ops = orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, L))
    dps = pg.prepare_all_paths(dg, F)
    knobs = {k: int(rng.choice(v)) for k, v in KNOBS.items()}
    hmin = [None, 0, 8, 64, 1024][int(rng.integers(0, 5))]
    try:
        for k, v in knobs.items():
            pg.set_tuning(k, v)
        pg.set_heavy_min_degree(hmin)
        for dp, op in zip(dps, ops):
            dim = int(rng.choice(WIDTHS))
            G = pg.group_neighbors(dp, int(rng.integers(1, 9)))
            y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
            want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
            yd = pg.empty_rows(dp.P, dim)
            yd.copy_(torch.from_numpy(y))
            xd = pg.empty_rows(dp.D, dim)
            pg.backward_aggregation(G, yd, xd, overwrite=True)
            torch.cuda.synchronize()
            assert np.array_equal(bits(xd.cpu().numpy()), bits(want)), (seed, dim, knobs, hmin)
            if dp.D > 2:  # a row range of the same path
                b, e = sorted(int(v) for v in rng.integers(0, dp.D + 1, size=2))
                xr = pg.empty_rows(e - b, dim)
                pg.backward_aggregation(G, yd, xr, overwrite=True, rows=(b, e))
                torch.cuda.synchronize()
                assert np.array_equal(bits(xr.cpu().numpy()), bits(want[b:e])), (seed, dim, "rows", b, e)
            xh = np.full((dp.D, dim), np.nan, np.float32)  # host-buffer drop-in
            pg.backward_aggregation(G, y, xh, overwrite=True)
            assert np.array_equal(bits(xh), bits(want)), (seed, dim, "host")
    finally:
        for k in knobs:
            pg.set_tuning(k, None)
        pg.set_heavy_min_degree(None)


HOST_KNOBS = {
    "host_segs": (1, 2, 3, 4, 6),
    "host_final_segs": (1, 2, 3),
    "host_seg_balance": (0, 1),
    "host_chunk_balance": (0, 50, 100),
    "host_last_seg_pct": (0, 30, 40, 70),
    "host_chunks": (1, 3, 8, 16),
    "host_chunk_order": (0, 1),
    "host_hub_chunk_side": (0, 1, 2),
    "host_first_chunk_pct": (100, 50, 10),
    "host_seq": (0, 1, 2),
    "host_small_chunks": (0, 2),
    "host_hub_min": (1, 64, 16384),
}


@pytest.mark.parametrize("seed", range(int(os.environ.get("PG_STRESS_HOST_SEEDS", "6"))))
def test_random_host_pipeline(pg, orc, seed):
    """The host-buffer pipeline (source segments under the H2D, chunked last
    pass under the D2H) on paths big enough to engage it, with random
    pipeline knobs, pinned or pageable buffers, overwrite or accumulate."""
    import torch

    rng = np.random.default_rng(5000 + seed)
    n = int(rng.integers(20000, 40000))
    pairs, n_pad = rmat_pairs(orc, n, n * 56, 70 + seed)
    vt = orc.sample_training_set(n_pad, 0.5, seed)
    dg = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
    og = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
    F = pg.compute_frontiers(dg, vt, 2)
    ops = orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, 2))
    dp, op = pg.prepare_all_paths(dg, F)[1], ops[1]
    dim = int(rng.choice([301, 302, 320]))
    knobs = {k: int(rng.choice(v)) for k, v in HOST_KNOBS.items()}
    try:
        for k, v in knobs.items():
            pg.set_tuning(k, v)
        G = pg.group_neighbors(dp, 4)
        y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
        base = rng.uniform(-1, 1, size=(dp.D, dim)).astype(np.float32)
        accumulate = bool(rng.integers(0, 2))
        want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos],
                                      out=base.copy() if accumulate else None)
        pinned = bool(rng.integers(0, 2))
        yh = torch.from_numpy(y).pin_memory().numpy() if pinned else y
        xh = base.copy() if accumulate else np.full((dp.D, dim), np.nan, np.float32)
        if pinned:
            xh = torch.from_numpy(xh).pin_memory().numpy()
        pg.backward_aggregation(G, yh, xh, overwrite=not accumulate)
        assert np.array_equal(bits(xh), bits(want)), (seed, dim, knobs, pinned, accumulate, dp.D, dp.E)
    finally:
        for k in knobs:
            pg.set_tuning(k, None)


@pytest.mark.parametrize("seed", range(int(os.environ.get("PG_STRESS_BUILD_SEEDS", "24"))))
def test_random_build(pg, orc, seed):
    """Graph load, frontiers, execution paths, groupings, regression gs and
    the cost-model gs table on random RMAT graphs and training sets: every
    integer array and table equal to the oracle's."""
    rng = np.random.default_rng(9000 + seed)
    n = int(rng.integers(50, 8000))
    pairs, n_pad = rmat_pairs(orc, n, n * int(rng.choice([1, 4, 16, 48])), 300 + seed)
    ratio = float(rng.choice([0.001, 0.02, 0.3, 0.9, 1.0]))
    vt = orc.sample_training_set(n_pad, ratio, seed)
    L = int(rng.integers(1, 5))
    symnorm = bool(seed % 2)
    dg = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm" if symnorm else "unit")
    og = orc.build_graph(pairs, n_hint=n_pad, symnorm=symnorm)
    offs, nb, w = dg.export()
    assert np.array_equal(offs, og.offsets) and np.array_equal(nb, og.neighbors)
    assert np.array_equal(w.view(np.uint64), og.weights.view(np.uint64))
    F = pg.compute_frontiers(dg, vt, L)
    lv = orc.compute_frontiers(og, vt, L)
    for k in range(L + 1):
        assert np.array_equal(F.level(k), lv[k]), (seed, k)
    for dp, op in zip(pg.prepare_all_paths(dg, F), orc.prepare_all_paths(og, lv)):
        x = dp.export()
        for f in ("dest", "src", "srcpos", "offsets", "neighbors"):
            assert np.array_equal(x[f], getattr(op, f)), (seed, f)
        assert np.array_equal(x["weights"].view(np.uint64), op.weights.view(np.uint64))
        assert pg.path_regression_gs(dp) == orc.path_regression_gs(op.D, op.E)
        gs = int(rng.integers(1, 40))
        gx = pg.group_neighbors(dp, gs).export()
        og_ = orc.group_neighbors(op.offsets, gs)
        for f in ("dest", "begin", "end", "dest_groups"):
            assert np.array_equal(gx[f], getattr(og_, f)), (seed, f, gs)
        dim = int(rng.choice([1, 16, 100, 602]))
        W = int(rng.choice([1, 8, 16]))
        best, table = pg.oracle_gs(dp, dim, W, 0.25)
        obest, otable = orc.oracle_gs_cost(op.offsets, [c for c, _ in table], dim, W, 0.25)
        assert best == obest and [c for _, c in table] == list(otable), (seed, dim, W)


def test_concurrent_host_calls_mixed_buffers(pg, orc):
    """Several host threads issuing host-buffer calls at once on distinct
    groupings, pinned and pageable, of sizes that span several 16 MB staging
    pieces: every result bit-exact (per-device copy streams and staging
    slots are serialised, never shared mid-call)."""
    import threading

    import torch

    rng = np.random.default_rng(4242)
    pairs, n_pad = rmat_pairs(orc, 30000, 30000 * 40, 17)
    vt = orc.sample_training_set(n_pad, 0.5, 3)
    dg = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
    og = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
    F = pg.compute_frontiers(dg, vt, 2)
    ops = orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, 2))
    dps = pg.prepare_all_paths(dg, F)
    jobs = []
    for dp, op in zip(dps, ops):
        for dim, pinned in ((33, False), (301, True), (302, False), (128, False)):
            y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
            want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
            yh = torch.from_numpy(y).pin_memory().numpy() if pinned else y
            jobs.append((pg.group_neighbors(dp, 4), yh, want, pinned))
    errors = []

    def run(G, y, want, pinned):
        try:
            for _ in range(3):
                x = np.full(want.shape, np.nan, np.float32)
                if pinned:
                    x = torch.from_numpy(x).pin_memory().numpy()
                pg.backward_aggregation(G, y, x, overwrite=True)
                if not np.array_equal(bits(x), bits(want)):
                    errors.append((want.shape, pinned))
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    ts = [threading.Thread(target=run, args=j) for j in jobs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_concurrent_calls_share_one_grouping(pg, orc):
    """Host threads calling into ONE grouping at once (the reference's
    aggregate_pull takes a const GroupedCsr and is re-entrant): device calls
    over distinct row ranges (each builds and caches its own schedule),
    whole-path calls (the cached L2-sized source segments) and host-buffer
    calls (the cached host pipeline cuts), every result bit-exact."""
    import threading

    import torch

    rng = np.random.default_rng(777)
    pairs, n_pad = rmat_pairs(orc, 20000, 20000 * 48, 21)
    vt = orc.sample_training_set(n_pad, 0.6, 5)
    dg = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
    og = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
    F = pg.compute_frontiers(dg, vt, 2)
    op = orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, 2))[1]
    dp = pg.prepare_all_paths(dg, F)[1]
    dim = 300
    G = pg.group_neighbors(dp, 8)
    y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
    want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
    yd = pg.empty_rows(dp.P, dim)
    yd.copy_(torch.from_numpy(y))
    cuts = sorted(set(rng.integers(0, dp.D, 24).tolist()) | {0, dp.D})
    ranges = [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1) if cuts[i + 1] > cuts[i]]
    errors = []

    def dev_job(rs):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for rb, re in rs:
                    x = pg.empty_rows(re - rb, dim)
                    pg.backward_aggregation(G, yd, x, overwrite=True, rows=(rb, re), stream=st)
                    st.synchronize()
                    if not np.array_equal(bits(x.cpu().numpy()), bits(want[rb:re])):
                        errors.append(("rows", rb, re))
                x = pg.empty_rows(dp.D, dim)
                pg.backward_aggregation(G, yd, x, overwrite=True, stream=st)
                st.synchronize()
                if not np.array_equal(bits(x.cpu().numpy()), bits(want)):
                    errors.append("whole")
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    def host_job():
        try:
            for _ in range(2):
                x = np.full(want.shape, np.nan, np.float32)
                pg.backward_aggregation(G, y, x, overwrite=True)
                if not np.array_equal(bits(x), bits(want)):
                    errors.append("host")
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    ts = [threading.Thread(target=dev_job, args=(ranges[k::4],)) for k in range(4)]
    ts += [threading.Thread(target=host_job) for _ in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("seed", range(int(os.environ.get("PG_STRESS_SEEDS_TOL", "24"))))
def test_random_tolerance_paths(pg, orc, seed):
    """Randomised sweep of the tolerance-level kernels: the atomic-free grouped
    Fast stage (random gs, widths, training fractions; deterministic run to
    run, within the conditioning-aware fp32 bound of f64, bit-equal to
    Deterministic when gs >= max degree), the f64 stage (bit-exact vs the
    f64 oracle) and the tensor-core GEMMs (random shapes, gathered or not)."""
    import torch

    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(300, 8000))
    pairs, n_pad = rmat_pairs(orc, n, n * int(rng.choice([4, 16, 48])), 900 + seed)
    vt = orc.sample_training_set(n_pad, float(rng.choice([0.05, 0.3, 1.0])), seed)
    dg = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
    og = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
    ops = orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, 2))
    dps = pg.prepare_all_paths(dg, pg.compute_frontiers(dg, vt, 2))
    for dp, op in zip(dps, ops):
        dim = int(rng.choice(WIDTHS))
        gs = int(rng.choice([1, 2, 5, 17, 64, 300, max(dp.max_degree, 1)]))
        G = pg.group_neighbors(dp, gs)
        y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
        yu = y[op.srcpos]
        want64 = orc.aggregate_pull_f64(op.offsets, op.neighbors, op.weights, yu.astype(np.float64))
        absum = orc.aggregate_pull_f64(op.offsets, op.neighbors, np.abs(op.weights), np.abs(yu).astype(np.float64))
        yd = pg.empty_rows(dp.P, dim)
        yd.copy_(torch.from_numpy(y))
        runs = []
        for _ in range(2):
            x = pg.empty_rows(dp.D, dim)
            x.fill_(float("nan"))
            pg.backward_aggregation(G, yd, x, mode=pg.GROUPED, overwrite=True)
            torch.cuda.synchronize()
            runs.append(x.cpu().numpy())
        assert np.array_equal(bits(runs[0]), bits(runs[1])), (seed, gs, dim)
        assert (np.abs(runs[0] - want64) <= 1e-6 + 1e-5 * absum).all(), (seed, gs, dim)
        if gs >= dp.max_degree:
            det = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, yu)
            assert np.array_equal(bits(runs[0]), bits(det)), (seed, "one group per destination")
        # f64 stage, bit-exact
        x64 = np.zeros((dp.D, dim))
        pg.backward_aggregation(G, y.astype(np.float64), x64, overwrite=True)
        assert np.array_equal(x64.view(np.uint64), want64.view(np.uint64)), (seed, dim, "f64")
    # tensor-core GEMMs on random shapes
    for _ in range(2):
        nr, k, m = int(rng.integers(1, 5000)), int(rng.integers(1, 300)), int(rng.integers(1, 700))
        a = rng.uniform(-1, 1, size=(nr, k)).astype(np.float32)
        b = rng.uniform(-1, 1, size=(m, k)).astype(np.float32)
        ad = pg.empty_rows(nr, k)
        ad.copy_(torch.from_numpy(a))
        bd = torch.from_numpy(b).cuda()
        od = pg.empty_rows(nr, m)
        pg.gemm_a_bt(ad, bd, od, tensor_cores=True)
        ind, outd = int(rng.integers(1, 641)), int(rng.integers(1, 257))
        ry = int(rng.integers(1, 4000))
        rows = rng.integers(0, ry, size=int(rng.integers(0, 4000))).astype(np.int32)
        yy = rng.uniform(-1, 1, size=(ry, ind)).astype(np.float32)
        gg = rng.uniform(-1, 1, size=(len(rows), outd)).astype(np.float32)
        yyd = pg.empty_rows(ry, ind)
        yyd.copy_(torch.from_numpy(yy))
        ggd = pg.empty_rows(len(rows), outd)
        ggd.copy_(torch.from_numpy(gg))
        wd = pg.empty_rows(ind, outd)
        if len(rows):
            pg.gemm_at_b(yyd, ggd, wd, a_rows=torch.from_numpy(rows).cuda(), tensor_cores=True)
        torch.cuda.synchronize()
        got, exact = od.cpu().numpy().astype(np.float64), a.astype(np.float64) @ b.astype(np.float64).T
        mag = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64).T
        assert (np.abs(got - exact) <= 1e-6 + 1e-5 * mag).all(), (seed, nr, k, m)
        if len(rows):
            ya = yy[rows].astype(np.float64)
            got, exact = wd.cpu().numpy().astype(np.float64), ya.T @ gg.astype(np.float64)
            mag = np.abs(ya).T @ np.abs(gg).astype(np.float64)
            assert (np.abs(got - exact) <= 1e-6 + 1e-5 * mag).all(), (seed, ind, outd, len(rows))
