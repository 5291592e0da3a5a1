"""GPU parity of the backward-aggregation SpMM (the hot path) and the dense
helpers of backward_epp.

Gate (BASELINE.json north_star): fp32 within 1e-5 relative / 1e-6 absolute of
the reference. The kernel keeps the reference's Deterministic summation order
(ascending edges, unfused mul/add, +0), so it is asserted BIT-EXACT against
the fp32 oracle, and additionally within the conditioning-aware tolerance of
the f64 oracle: |gpu - ref64| <= 1e-6 + 1e-5 * sum_e |w_e * y_e| plus a
normwise check and a non-vacuity check (SURVEY §7 hard part 1).
"""
import os

import numpy as np
import pytest

from conftest import GEX_PAIRS, GEX_VT, rmat_pairs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


def torch_mod():
    import torch

    return torch


def to_dev(x, ld=None):
    torch = torch_mod()
    rows, cols = x.shape
    ld = ld or cols
    buf = torch.zeros((rows, ld), dtype=torch.float32, device="cuda")
    buf[:, :cols] = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    return buf[:, :cols]


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def tol_check(gpu, orc, p, y_used):
    """Conditioning-aware bound against the f64 oracle + normwise + non-vacuity."""
    ref64 = orc.aggregate_pull_f64(p.offsets, p.neighbors, p.weights, y_used.astype(np.float64))
    absmat = orc.aggregate_pull_f64(p.offsets, p.neighbors, np.abs(p.weights), np.abs(y_used).astype(np.float64))
    err = np.abs(gpu.astype(np.float64) - ref64)
    assert (err <= 1e-6 + 1e-5 * absmat).all()
    nrm = np.linalg.norm(ref64)
    if nrm > 0:
        assert np.linalg.norm(gpu - ref64) / nrm <= 1e-5
    return ref64


def build_all(pg, orc, pairs, n_hint, vt, L, symnorm=True):
    og = orc.build_graph(pairs, n_hint=n_hint, symnorm=symnorm)
    dg = pg.build_undirected_csr(pairs, n_hint=n_hint, weights="symnorm" if symnorm else "unit")
    F = pg.compute_frontiers(dg, vt, L)
    ops = orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, L))
    dps = pg.prepare_all_paths(dg, F)
    return og, dg, F, ops, dps


def test_hand_sums(pg, orc):
    # test_engine.cpp:72-80 (graph grouping, input by global id)
    torch = torch_mod()
    g = pg.build_undirected_csr(GEX_PAIRS)
    G = pg.group_neighbors(g, 3)
    x = to_dev(np.arange(1, 6, dtype=np.float32).reshape(5, 1))
    y = torch.zeros((5, 1), device="cuda")
    pg.aggregate_pull(G, x, y)
    assert y[:, 0].tolist() == [2, 13, 6, 10, 6]
    # SG_1 hand case test_engine.cpp:169-180
    F = pg.compute_frontiers(g, GEX_VT, 2)
    sg1 = pg.extract_execution_path(g, F, 1)
    out = np.zeros((2, 1), np.float32)
    pg.aggregate_pull(pg.group_neighbors(sg1, 2), np.array([[1.0], [2.0]], np.float32), out)
    assert out[:, 0].tolist() == [3.0, 3.0]


@pytest.mark.parametrize("dim", [1, 3, 4, 7, 16, 41, 64, 128, 256, 602])
def test_backward_aggregation_bit_exact(pg, orc, dim):
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 8, 7)
    vt = orc.sample_training_set(4096, 0.3, 42)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    rng = np.random.default_rng(dim)
    for dp, op in zip(dps, ops):
        y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)  # parent-frontier rows
        y_used = y[op.srcpos]
        want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y_used)
        for ld in (dim, pg.padded_ld(dim)):
            for gs in (1, 5):
                G = pg.group_neighbors(dp, gs)
                x = to_dev(np.zeros((dp.D, dim), np.float32), ld)
                pg.backward_aggregation(G, to_dev(y, ld), x)
                torch.cuda.synchronize()
                got = x.cpu().numpy()
                assert np.array_equal(bits(got), bits(want)), (dim, ld, gs)
        tol_check(got, orc, op, y_used)


@pytest.mark.parametrize("kern", ["coop", "narrow", "tma", "wide_lat"])
@pytest.mark.parametrize("heavy_min", [1, 0, 64])
@pytest.mark.parametrize("dim", [1, 16, 41, 130, 602])
def test_heavy_ring_kernel_bit_exact(pg, orc, dim, heavy_min, kern):
    """Force every (heavy_min=1), none (0) or some (64) destinations onto the
    TMA bulk-copy ring kernel; results must not change by a bit, including
    accumulate semantics."""
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 8, 13)
    vt = orc.sample_training_set(4096, 0.3, 4)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    rng = np.random.default_rng(dim + heavy_min)
    try:
        pg.set_heavy_min_degree(heavy_min)
        # narrow rows: cooperative tiles (default), scalar-lane latency kernel,
        # or the TMA cp.async.bulk + mbarrier ring; wide rows: pipelined
        # (default) or plain latency kernel
        pg.set_tuning("heavy_narrow", 1 if kern == "narrow" else 0)
        pg.set_tuning("heavy_tma", 1 if kern == "tma" else 0)
        pg.set_tuning("heavy_wide_pipe", 0 if kern == "wide_lat" else 1)
        pg.set_tuning("hub_inline", 0)  # wide rows: the side kernels, not the inlined front
        for dp, op in zip(dps, ops):
            y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
            base = rng.uniform(-1, 1, size=(dp.D, dim)).astype(np.float32)
            want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos], out=base)
            x = to_dev(base, pg.padded_ld(dim))
            pg.backward_aggregation(pg.group_neighbors(dp, 7), to_dev(y, pg.padded_ld(dim)), x)
            torch.cuda.synchronize()
            got = x.cpu().numpy()
            assert np.array_equal(bits(got), bits(want)), (dim, heavy_min)
            b = dp.shard_bounds(3)
            x2 = to_dev(base[b[1]:b[2]], pg.padded_ld(dim))
            pg.backward_aggregation(pg.group_neighbors(dp, 7), to_dev(y, pg.padded_ld(dim)), x2,
                                    rows=(b[1], b[2]))
            torch.cuda.synchronize()
            assert np.array_equal(bits(x2.cpu().numpy()), bits(want[b[1]:b[2]]))
    finally:
        pg.set_heavy_min_degree(None)
        for k in ("heavy_narrow", "heavy_tma", "heavy_wide_pipe", "hub_inline"):
            pg.set_tuning(k)


@pytest.mark.parametrize("variant", [{"row_kernel": 1}, {"row_kernel": 1, "row_u": 3, "row_seg_mb": 8},
                                     {"row_kernel": 1, "row_u": 4, "row_heavy": 64}, {"vec_block": 512},
                                     {"vec_block": 1024}, {"ld_cg": 7}, {"hub_inline": 0, "heavy_wide_pipe": 2},
                                     {"hub_inline": 0}, {"hub_inline": 1, "hub_front_min": 8}, {"rec_window": 2},
                                     {"vec_window": 4}, {"hub_inline": 0, "heavy_wide_pipe": 3},
                                     {"hub_inline": 0, "heavy_wide_pipe": 4}, {"vec8": 1},
                                     {"vec8": 1, "vec_u": 4}, {"vec8": 1, "hub_inline": 0},
                                     {"vec8": 1, "vec8_u": 3}, {"vec8": 1, "vec8_u": 6},
                                     {"range_side_hubs": 0}, {"range_side_hubs": 0, "vec8": 1},
                                     {"hub_inline": 0, "heavy_wide_pipe": 5}])
@pytest.mark.parametrize("dim", [130, 300, 602, 700])
def test_wide_row_schedule_variants_bit_exact(pg, orc, dim, variant):
    """The measured-and-kept-selectable wide-row schedules:
    whole-row warps (k_agg_row) with their L2-sized segments and hub
    threshold, 512/1024-thread CTAs, evict-first record loads, chunk-major hub
    items — bit-identical to the oracle, accumulate semantics and row ranges
    included."""
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 24, 21)
    vt = orc.sample_training_set(4096, 0.5, 8)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    rng = np.random.default_rng(dim)
    try:
        for k, v in variant.items():
            pg.set_tuning(k, v)
        pg.set_heavy_min_degree(64)
        for dp, op in zip(dps, ops):
            y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
            base = rng.uniform(-1, 1, size=(dp.D, dim)).astype(np.float32)
            want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos], out=base)
            x = to_dev(base, pg.padded_ld(dim))
            G = pg.group_neighbors(dp, 3)
            pg.backward_aggregation(G, to_dev(y, pg.padded_ld(dim)), x)
            torch.cuda.synchronize()
            assert np.array_equal(bits(x.cpu().numpy()), bits(want)), (dim, variant)
            b = dp.shard_bounds(3)
            x2 = to_dev(base[b[1]:b[2]], pg.padded_ld(dim))
            pg.backward_aggregation(G, to_dev(y, pg.padded_ld(dim)), x2, rows=(b[1], b[2]))
            torch.cuda.synchronize()
            assert np.array_equal(bits(x2.cpu().numpy()), bits(want[b[1]:b[2]])), (dim, variant, "rows")
    finally:
        pg.set_heavy_min_degree(None)
        for k in variant:
            pg.set_tuning(k)


@pytest.mark.parametrize("vec8", [0, 1])
@pytest.mark.parametrize("dim", [8, 16, 20, 24, 32, 40, 64, 100, 128, 136])
def test_vec8_widths_bit_exact(pg, orc, dim, vec8):
    """256-bit row gathers (k_agg_vec8, forced on small graphs with vec8 = 1)
    at every lane-count instantiation — 2 / 4 / 8 lanes per narrow row,
    16 per 128-column chunk — and the pitches it refuses (20 columns: a
    16-byte pitch, back to k_agg_vec4): bit-identical to the oracle, with
    accumulate semantics and row ranges."""
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 24, 23)
    vt = orc.sample_training_set(4096, 0.5, 8)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    rng = np.random.default_rng(dim)
    try:
        pg.set_tuning("vec8", vec8)
        for dp, op in zip(dps, ops):
            y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
            base = rng.uniform(-1, 1, size=(dp.D, dim)).astype(np.float32)
            want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos], out=base)
            x = to_dev(base, pg.padded_ld(dim))
            G = pg.group_neighbors(dp, 3)
            pg.backward_aggregation(G, to_dev(y, pg.padded_ld(dim)), x)
            torch.cuda.synchronize()
            assert np.array_equal(bits(x.cpu().numpy()), bits(want)), (dim, vec8)
            b = dp.shard_bounds(3)
            x2 = to_dev(base[b[1]:b[2]], pg.padded_ld(dim))
            pg.backward_aggregation(G, to_dev(y, pg.padded_ld(dim)), x2, rows=(b[1], b[2]))
            torch.cuda.synchronize()
            assert np.array_equal(bits(x2.cpu().numpy()), bits(want[b[1]:b[2]])), (dim, vec8, "rows")
    finally:
        pg.set_tuning("vec8")


def test_aggregate_pull_local_and_accumulate(pg, orc):
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 2048, 2048 * 6, 3)
    vt = orc.sample_training_set(2048, 0.05, 1)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    rng = np.random.default_rng(0)
    for dp, op in zip(dps, ops):
        dim = 20
        x = rng.uniform(-1, 1, size=(dp.S, dim)).astype(np.float32)  # local source rows
        base = rng.uniform(-1, 1, size=(dp.D, dim)).astype(np.float32)
        want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, x, out=base)
        G = pg.group_neighbors(dp, 3)
        out = to_dev(base, 32)
        pg.aggregate_pull(G, to_dev(x, 32), out)
        torch.cuda.synchronize()
        assert np.array_equal(bits(out.cpu().numpy()), bits(want))
        # host DenseMatrix drop-in
        host = base.copy()
        cnt = {}
        pg.aggregate_pull(G, x, host, counters=cnt)
        assert np.array_equal(bits(host), bits(want))
        assert cnt["edges_traversed"] == op.E and cnt["groups_executed"] == G.group_count()
        assert cnt["atomic_commits"] == 0
        fc = G.counters(dim, pg.FAST)
        assert fc["atomic_commits"] == orc.fast_atomic_commits(op.offsets, 3, dim)


def test_shape_errors(pg, orc):
    torch = torch_mod()
    g = pg.build_undirected_csr(GEX_PAIRS)
    F = pg.compute_frontiers(g, GEX_VT, 2)
    p = pg.extract_execution_path(g, F, 0)
    G = pg.group_neighbors(p, 2)
    y = torch.zeros((p.P + 1, 4), device="cuda")
    with pytest.raises(pg.ShapeError):
        pg.backward_aggregation(G, y, torch.zeros((p.D, 4), device="cuda"))
    with pytest.raises(pg.ShapeError):
        pg.aggregate_pull(G, np.zeros((p.S, 4), np.float32), np.zeros((p.D, 3), np.float32))


def test_row_shards_concatenate(pg, orc):
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 8, 9)
    vt = orc.sample_training_set(4096, 0.2, 5)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    dim = 48
    for dp, op in zip(dps, ops):
        y = np.random.default_rng(1).uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
        want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
        G = pg.group_neighbors(dp, 4)
        yd = to_dev(y, 64)
        from paper_2204_02662_b200 import dist as pgd

        for world in (1, 2, 3, 8):
            b = dp.shard_bounds(world)
            assert b[0] == 0 and b[-1] == dp.D and (np.diff(b.astype(np.int64)) >= 0).all()
            assert np.array_equal(b.astype(np.int64), pgd.edge_balanced_bounds(op.offsets, world))
            parts = []
            for r in range(world):
                xs = to_dev(np.zeros((int(b[r + 1] - b[r]), dim), np.float32), 64)
                pg.backward_aggregation(G, yd, xs, rows=(b[r], b[r + 1]))
                parts.append(xs)
            torch.cuda.synchronize()
            got = torch.cat(parts).cpu().numpy()
            assert np.array_equal(bits(got), bits(want)), world


@pytest.mark.parametrize("world", [2, 3, 8])
def test_remapped_allgather_layout(pg, orc, world):
    """The multi-GPU data path on one device: y_grad row shards laid out as a
    padded all_gather buffer, the remapped edge stream, per-rank row ranges
    (the heavy kernel forced on for some ranks' hubs)."""
    torch = torch_mod()
    from paper_2204_02662_b200 import dist as pgd

    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 8, 19)
    vt = orc.sample_training_set(4096, 0.25, 6)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    plan = pgd.plan([None, None], [dps[0].P, dps[1].P], world, [p.shard_bounds(world) for p in dps])
    dims = [16, 41]
    try:
        pg.set_heavy_min_degree(256)
        for i, (dp, op) in enumerate(zip(dps, ops)):
            sh = plan[i]
            y = np.random.default_rng(i).uniform(-1, 1, size=(dp.P, dims[i])).astype(np.float32)
            want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
            padded = np.zeros((sh.gathered_rows, dims[i]), np.float32)
            padded[sh.source_map] = y
            G = pg.group_neighbors(dp, 3)
            G.remap_sources(sh.source_map, sh.gathered_rows)
            yd = to_dev(padded, pg.padded_ld(dims[i]))
            parts = []
            for r in range(world):
                db, de = sh.my_dest_rows(r)
                xs = pg.empty_rows(de - db, dims[i])
                pg.backward_aggregation(G, yd, xs, overwrite=True, rows=(db, de))
                parts.append(xs)
            torch.cuda.synchronize()
            got = torch.cat(parts).cpu().numpy()
            assert np.array_equal(bits(got), bits(want))
            with pytest.raises(pg.ConfigError):  # host path refuses a remapped grouping
                pg.backward_aggregation(G, y, np.zeros((dp.D, dims[i]), np.float32))
            G.remap_sources(None, 0)
    finally:
        pg.set_heavy_min_degree(None)


@pytest.mark.parametrize("nseg", [1, 2, 3, 8])
def test_source_segments_bit_exact(pg, orc, nseg):
    """Segments of source rows run as successive accumulate passes must give
    the serial order's bits (edges are sorted by source within each
    destination), including empty segments, row ranges and heavy routing."""
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 8, 29)
    vt = orc.sample_training_set(4096, 0.3, 8)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    rng = np.random.default_rng(nseg)
    for dim, hmin in ((16, None), (602, None), (41, 128)):
        pg.set_heavy_min_degree(hmin)
        for dp, op in zip(dps, ops):
            y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
            base = rng.uniform(-1, 1, size=(dp.D, dim)).astype(np.float32)
            want0 = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
            want1 = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos], out=base)
            cuts = np.unique(np.concatenate([[0, dp.P], rng.integers(0, dp.P + 1, size=nseg - 1)]))
            if nseg == 3:
                cuts = np.array([0, 0, dp.P // 3, dp.P])  # an empty first segment
            G = pg.group_neighbors(dp, 4)
            G.set_segments(cuts)
            yd = to_dev(y, pg.padded_ld(dim))
            x = pg.empty_rows(dp.D, dim)
            for k in range(len(cuts) - 1):
                pg.backward_aggregation(G, yd, x, overwrite=(k == 0), segment=k)
            xa = to_dev(base, pg.padded_ld(dim))
            for k in range(len(cuts) - 1):
                pg.backward_aggregation(G, yd, xa, segment=k)
            b = dp.shard_bounds(2)
            xr = pg.empty_rows(int(b[2] - b[1]), dim)
            for k in range(len(cuts) - 1):
                pg.backward_aggregation(G, yd, xr, overwrite=(k == 0), segment=k, rows=(b[1], b[2]))
            torch.cuda.synchronize()
            assert np.array_equal(bits(x.cpu().numpy()), bits(want0)), (dim, nseg)
            assert np.array_equal(bits(xa.cpu().numpy()), bits(want1)), (dim, nseg)
            assert np.array_equal(bits(xr.cpu().numpy()), bits(want0[b[1]:b[2]])), (dim, nseg)
    pg.set_heavy_min_degree(None)


def test_unit_weights_hub_heavy(pg, orc):
    """Unit weights on a hub-heavy graph: bit-exact with the fp32 reference
    even where the reference itself leaves the 1e-5 tolerance of the exact
    sum."""
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 16384, 16384 * 16, 21)
    vt = orc.sample_training_set(16384, 0.5, 2)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2, symnorm=False)
    dp, op = dps[1], ops[1]
    y = np.random.default_rng(3).uniform(-1, 1, size=(dp.P, 16)).astype(np.float32)
    want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
    x = to_dev(np.zeros((dp.D, 16), np.float32))
    pg.backward_aggregation(pg.group_neighbors(dp, 8), to_dev(y), x)
    torch.cuda.synchronize()
    assert np.array_equal(bits(x.cpu().numpy()), bits(want))


def test_dense_helpers_bit_exact(pg, orc):
    torch = torch_mod()
    rng = np.random.default_rng(5)
    for n, m, k in ((1, 1, 1), (261, 602, 16), (1000, 41, 16), (333, 256, 40), (77, 100, 256), (5, 3, 0)):
        a = rng.uniform(-1, 1, size=(n, k)).astype(np.float32)
        b = rng.uniform(-1, 1, size=(m, k)).astype(np.float32)
        out = to_dev(np.zeros((n, m), np.float32), pg.padded_ld(m))
        pg.gemm_a_bt(to_dev(a), to_dev(b), out)
        torch.cuda.synchronize()
        assert np.array_equal(bits(out.cpu().numpy()), bits(orc.gemm_a_bt_f32(a, b))), (n, m, k)
    g = rng.uniform(-1, 1, size=(100, 37)).astype(np.float32)
    pre = rng.uniform(-1, 1, size=(100, 37)).astype(np.float32)
    pre[0, :5] = 0.0
    out = to_dev(np.zeros_like(g))
    pg.relu_backward(to_dev(g), to_dev(pre), out)
    torch.cuda.synchronize()
    assert np.array_equal(bits(out.cpu().numpy()), bits(orc.relu_backward_f32(g, pre)))
    ids = torch.tensor([3, 0, 99, 3], dtype=torch.int32, device="cuda")
    gout = to_dev(np.zeros((4, 37), np.float32))
    pg.gather_rows(to_dev(g), ids, gout)
    torch.cuda.synchronize()
    assert np.array_equal(gout.cpu().numpy(), g[[3, 0, 99, 3]])


def test_golden_chain_on_device(pg):
    """The reference's real gradient chain (engine.hpp:316-346) replayed on
    device from the golden operands: y = gemm_a_bt(g, W), x = aggregate,
    g = relu_backward(x, pre) — bit-exact at every step."""
    torch = torch_mod()
    gold = dict(np.load(GOLD))
    n = int(gold["g_n"][0])
    dg = pg.graph_from_csr(n, gold["g_offsets"], gold["g_neighbors"], gold["g_weights"])
    F = pg.compute_frontiers(dg, gold["vt"], 2)
    paths = pg.prepare_all_paths(dg, F)
    gm = to_dev(gold["ch_top_g"])
    for i, p in enumerate(paths):
        l = 1 - i
        w = to_dev(gold[f"ch_w{l}"])
        y = pg.empty_rows(gm.shape[0], w.shape[0])
        pg.gemm_a_bt(gm, w, y)
        x = pg.empty_rows(p.D, w.shape[0])
        pg.backward_aggregation(pg.group_neighbors(p, 2), y, x, overwrite=True)
        torch.cuda.synchronize()
        assert np.array_equal(bits(y.cpu().numpy()), bits(gold[f"ch_y{i}"]))
        assert np.array_equal(bits(x.cpu().numpy()), bits(gold[f"ch_x{i}"]))
        if l > 0:
            nxt = pg.empty_rows(p.D, w.shape[0])
            pg.relu_backward(x, to_dev(gold["ch_pre0"]), nxt)
            gm = nxt
    # the golden SpMM vectors (local-indexed input, aggregate_pull)
    for i, p in enumerate(paths):
        G = pg.group_neighbors(p, (2, 9)[i])
        out = np.zeros((p.D, 37), np.float32)
        pg.aggregate_pull(G, gold[f"p{i}_agg_in"], out)
        assert np.array_equal(bits(out), bits(gold[f"p{i}_agg_out"]))


@pytest.mark.slow
def test_large_checksum(pg, orc):
    """A 2M-edge hub-heavy path at width 602 (the Reddit layer-0 width):
    bit-exact against the oracle on every row."""
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 65536, 1_000_000, 17)
    vt = orc.sample_training_set(65536, 0.66, 42)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    dp, op = dps[1], ops[1]
    dim = 602
    y = np.random.default_rng(7).uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
    want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
    G = pg.group_neighbors(dp, pg.path_regression_gs(dp))
    x = pg.empty_rows(dp.D, dim)
    pg.backward_aggregation(G, to_dev(y, pg.padded_ld(dim)), x, overwrite=True)
    torch.cuda.synchronize()
    assert np.array_equal(bits(x.cpu().numpy()), bits(want))
    # host drop-in: flat copies, on-device repack (602 % 4 != 0), chunked
    # D2H overlap; pinned and pageable buffers, overwrite and accumulate
    assert dp.D >= 16384 and dp.D * dim * 4 >= 32 << 20
    for pinned in (True, False):
        yh = torch.from_numpy(y).pin_memory().numpy() if pinned else y.copy()
        xh = np.full((dp.D, dim), np.nan, np.float32)
        pg.backward_aggregation(G, yh, xh, overwrite=True)
        assert np.array_equal(bits(xh), bits(want))
    base = np.random.default_rng(8).uniform(-1, 1, size=(dp.D, dim)).astype(np.float32)
    want2 = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos], out=base)
    xh = base.copy()
    pg.backward_aggregation(G, y, xh)
    assert np.array_equal(bits(xh), bits(want2))
    # a width that is a multiple of 4 takes the no-repack branch
    y4 = y[:, :600].copy()
    want4 = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y4[op.srcpos])
    xh4 = np.zeros((dp.D, 600), np.float32)
    pg.backward_aggregation(G, y4, xh4, overwrite=True)
    assert np.array_equal(bits(xh4), bits(want4))


@pytest.mark.parametrize("dim", [301, 264])
def test_host_drop_in_pageable_and_pinned(pg, orc, dim):
    """The host-buffer drop-in (pg_backward_aggregate_host) on a path big
    enough for the K-segment / R-chunk pipeline, with PAGEABLE buffers (a
    reference DenseMatrix is a std::vector: staged through the library's
    pinned slots, several 16 MB pieces) and pinned ones, overwrite and
    accumulate, odd (repacked) and 16-byte widths: bit-exact with the fp32
    oracle."""
    torch = torch_mod()
    pairs, n_pad = rmat_pairs(orc, 32768, 32768 * 48, 41)
    vt = orc.sample_training_set(32768, 0.5, 9)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    dp, op = dps[1], ops[1]  # the layer-0 path: every frontier vertex, E/D ~ 90
    assert dp.E >= 64 * dp.D and dp.D * dim * 4 >= (32 << 20)
    G = pg.group_neighbors(dp, 4)
    rng = np.random.default_rng(dim)
    y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
    base = rng.uniform(-1, 1, size=(dp.D, dim)).astype(np.float32)
    want0 = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
    want1 = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos], out=base)
    for pinned in (False, True):
        yh = torch.from_numpy(y).pin_memory().numpy() if pinned else y.copy()
        x0 = np.full((dp.D, dim), np.nan, np.float32)
        x1 = base.copy()
        if pinned:
            x0 = torch.from_numpy(x0).pin_memory().numpy()
            x1 = torch.from_numpy(x1).pin_memory().numpy()
        pg.backward_aggregation(G, yh, x0, overwrite=True)
        pg.backward_aggregation(G, yh, x1)
        assert np.array_equal(bits(x0), bits(want0)), ("overwrite", pinned)
        assert np.array_equal(bits(x1), bits(want1)), ("accumulate", pinned)


def test_host_drop_in_concurrent_threads(pg, orc):
    """Distinct groupings may be used from different host threads at once
    (the reference's contract for built objects): concurrent host-buffer
    calls share the per-device copy streams and staging slots safely."""
    import threading

    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 8, 31)
    vt = orc.sample_training_set(4096, 0.3, 5)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    rng = np.random.default_rng(3)
    jobs = []
    for dp, op, dim in ((dps[0], ops[0], 41), (dps[1], ops[1], 602)):
        y = rng.uniform(-1, 1, size=(dp.P, dim)).astype(np.float32)
        want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])
        jobs.append((pg.group_neighbors(dp, 4), y, want, dp.D, dim))
    errors = []

    def run(G, y, want, D, dim):
        try:
            for _ in range(4):
                x = np.full((D, dim), np.nan, np.float32)
                pg.backward_aggregation(G, y, x, overwrite=True)
                if not np.array_equal(bits(x), bits(want)):
                    errors.append(dim)
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    ts = [threading.Thread(target=run, args=j) for j in jobs * 2]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_degenerate_shapes(pg, orc):
    """Empty paths (an isolated training vertex: no edges), zero-width
    rows, and the host-buffer calls on them: no launch failures, outputs
    as the reference leaves them (overwrite -> +0 rows, accumulate ->
    unchanged), counters zero."""
    torch = torch_mod()
    pairs = np.array([[0, 1]], np.uint32)
    vt = np.array([2], np.uint32)  # vertex 2 is isolated
    og, dg, F, ops, dps = build_all(pg, orc, pairs, 3, vt, 2)
    for dp, op in zip(dps, ops):
        assert dp.E == op.E == 0
        G = pg.group_neighbors(dp, 1)
        for dim in (0, 5, 16):
            y = np.ones((dp.P, dim), np.float32)
            x = np.full((dp.D, dim), 7.0, np.float32)
            pg.backward_aggregation(G, y, x)  # accumulate: nothing to add
            assert (x == 7.0).all()
            pg.backward_aggregation(G, y, x, overwrite=True)
            assert np.array_equal(bits(x), bits(np.zeros_like(x)))
            if dp.P and dp.D and dim:
                yd = to_dev(y, pg.padded_ld(dim))
                xd = pg.empty_rows(dp.D, dim)
                xd.fill_(3.0)
                pg.backward_aggregation(G, yd, xd, overwrite=True)
                torch.cuda.synchronize()
                assert (xd.cpu().numpy() == 0).all()
        assert all(int(v) == 0 for v in G.counters(16).values())


def test_launch_counter_counts_library_kernels(pg, orc):
    """pg_launch_count (the bench's gpu_launches): every SpMM call launches
    at least one of this library's kernels, counted."""
    from paper_2204_02662_b200 import _lib

    lib = _lib.load()
    pairs, n_pad = rmat_pairs(orc, 1024, 8192, 7)
    vt = orc.sample_training_set(1024, 0.1, 42)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    G = pg.group_neighbors(dps[1], 4)
    y = pg.empty_rows(dps[1].P, 16)
    x = pg.empty_rows(dps[1].D, 16)
    before = lib.pg_launch_count()
    for _ in range(3):
        pg.backward_aggregation(G, y, x, overwrite=True)
    assert lib.pg_launch_count() - before >= 3


def test_host_call_argument_errors(pg, orc):
    """Host-buffer calls reject what the reference's ShapeError would:
    wrong row counts, wrong widths, non-float32 or strided outputs — and
    leave the output untouched."""
    pairs, n_pad = rmat_pairs(orc, 512, 3000, 3)
    vt = orc.sample_training_set(512, 0.2, 1)
    og, dg, F, ops, dps = build_all(pg, orc, pairs, n_pad, vt, 2)
    dp = dps[1]
    G = pg.group_neighbors(dp, 4)
    y = np.ones((dp.P, 8), np.float32)
    x = np.full((dp.D, 8), 5.0, np.float32)
    with pytest.raises(pg.ConfigError):  # ShapeError is a ConfigError (status 2)
        pg.backward_aggregation(G, np.ones((dp.P + 1, 8), np.float32), x)
    with pytest.raises(pg.ConfigError):
        pg.backward_aggregation(G, y, np.zeros((dp.D, 9), np.float32))
    with pytest.raises(pg.ConfigError):
        pg.backward_aggregation(G, y, np.zeros((dp.D, 8), np.float64))
    with pytest.raises(pg.ConfigError):
        pg.backward_aggregation(G, y, np.zeros((dp.D, 16), np.float32)[:, ::2])
    assert (x == 5.0).all()
