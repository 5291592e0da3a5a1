"""aggregate_pull<double> — the reference's default precision
(run_config.hpp:53 Precision::F64; aggregate.hpp:56-122 with T = double) —
on the device, bit-exact with the f64 oracle (the reference's serial order,
f64 weights, no contraction) through the device call, the host DenseMatrix
<double> drop-in and the timed stage over an execution path."""
import numpy as np
import pytest

from conftest import rmat_pairs

pytestmark = pytest.mark.gpu


def bits64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("knobs", [{}, {"f64_hub_min": 24}, {"f64_hub_min": 24, "src_segs": 2},
                                   {"src_segs": 3}, {"vec8": 0}, {"pitch4": 1, "vec8": 1},
                                   {"pitch4": 1, "vec8": 1, "src_segs": 2}, {"pitch4": 1}])
@pytest.mark.parametrize("dim", [1, 2, 3, 16, 41, 100, 257])
def test_f64_stage_bit_exact(pg, orc, cuda, dim, knobs):
    """Default schedule, the hub kernel forced down to 24-edge lists
    (k_agg_f64_hub: tile-staged gathers, per-column serial fold), forced
    source-segment passes, and the 256-bit k_agg_f64v (4-double pitch,
    vec8 forced on): all bit-identical to the f64 oracle."""
    knobs = dict(knobs)
    pitch4 = knobs.pop("pitch4", 0)
    for k, v in knobs.items():
        pg.set_tuning(k, v)
    try:
        _f64_stage(pg, orc, dim, pitch4)
    finally:
        for k in knobs:
            pg.set_tuning(k)


def _f64_stage(pg, orc, dim, pitch4=0):
    import torch

    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 24, 11)
    g = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
    vt = pg.sample_training_set(n_pad, 0.3, 42)
    paths = pg.prepare_all_paths(g, pg.compute_frontiers(g, vt, 2))
    og = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
    ops = orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, 2))
    for p, op in zip(paths, ops):
        G = pg.group_neighbors(p, 3)
        y = np.random.default_rng(dim).uniform(-1, 1, size=(p.P, dim))
        want = orc.aggregate_pull_f64(op.offsets, op.neighbors, op.weights, y[op.srcpos])
        # host DenseMatrix<double> drop-in
        xh = np.full((p.D, dim), np.nan)
        pg.backward_aggregation(G, y, xh, overwrite=True)
        assert np.array_equal(bits64(xh), bits64(want))
        # device, pitched rows (even ld) and accumulate semantics
        # pitch4: a 4-double pitch (the 256-bit k_agg_f64v path past 32 columns)
        ld = (dim + 3) // 4 * 4 if pitch4 else dim + (dim & 1) + 2
        yd = torch.zeros((p.P, ld), dtype=torch.float64, device="cuda")[:, :dim]
        yd.copy_(torch.from_numpy(y))
        xd = torch.ones((p.D, ld), dtype=torch.float64, device="cuda")[:, :dim]
        pg.backward_aggregation(G, yd, xd)  # accumulate onto 1.0
        torch.cuda.synchronize()
        want_acc = orc.aggregate_pull_f64(op.offsets, op.neighbors, op.weights, y[op.srcpos], out=np.ones((p.D, dim)))
        assert np.array_equal(bits64(xd.cpu().numpy()), bits64(want_acc))
        # aggregate_pull<double> over the path's local sources
        xl = np.zeros((p.D, dim))
        pg.aggregate_pull(G, y[op.srcpos], xl, overwrite=True)
        assert np.array_equal(bits64(xl), bits64(want))


def test_f64_matches_compiled_reference(pg, orc, ref, cuda):
    """Against the reference's own aggregate_pull<double> (oracle/_ref)."""
    pairs, n_pad = rmat_pairs(orc, 2048, 2048 * 16, 5)
    g = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
    vt = pg.sample_training_set(n_pad, 0.25, 42)
    p = pg.prepare_all_paths(g, pg.compute_frontiers(g, vt, 2))[1]
    x = p.export()
    y = np.random.default_rng(3).uniform(-1, 1, size=(p.S, 37))
    want, _ = ref.aggregate_pull(x["offsets"], x["neighbors"], x["weights"], y)
    got = np.zeros((p.D, 37))
    pg.aggregate_pull(pg.group_neighbors(p, 4), y, got, overwrite=True)
    assert np.array_equal(bits64(got), bits64(want))
