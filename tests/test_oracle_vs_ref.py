"""Pins the C oracle against the reference itself, compiled from its own
sources (oracle/_ref/libpathgcn_ref.so), on identical inputs. Integer
structures bit-exact; fp32/f64 aggregation, gemm_a_bt bit-exact too (same
operation order, no FMA contraction on either side)."""
import numpy as np
import pytest

from conftest import random_graph_pairs, rmat_pairs

PATH_FIELDS = ["dest", "src", "srcpos", "offsets", "neighbors", "weights"]


def instances(orc, count=12):
    """acceptance.cpp:70-98 shape: n in {256..4096}, ratios {0.05,0.1,0.5}, L {2,3}."""
    out = []
    seed = 0
    for n in (256, 512, 1024, 2048, 4096):
        for ratio in (0.05, 0.1, 0.5):
            for L in (2, 3):
                if len(out) == count:
                    return out
                pairs, n_pad = rmat_pairs(orc, n, n * 4, 1000 + seed)
                out.append((pairs, n_pad, ratio, seed, L))
                seed += 1
    return out


def test_generators_match(orc, ref):
    for n, m, seed in ((1024, 8192, 7), (100, 50, 1), (5000, 20000, 3)):
        a = orc.gen_rmat(n, m, 0.45, 0.22, 0.22, 0.11, seed)
        b = ref.gen_rmat(n, m, 0.45, 0.22, 0.22, 0.11, seed)
        assert a[1] == b[1] and np.array_equal(a[0], b[0])
    for n, ratio, seed in ((1024, 0.1, 42), (7, 1.0, 0), (232965, 0.66, 42), (19717, 60 / 19717, 42)):
        assert np.array_equal(orc.sample_training_set(n, ratio, seed), ref.sample_training_set(n, ratio, seed))
    x = orc.random_matrix_f32(7, 5, 3)
    assert x.min() >= -1 and x.max() <= 1


@pytest.mark.parametrize("symnorm", [False, True])
def test_graph_build_matches(orc, ref, symnorm):
    for pairs, n_hint in ((rmat_pairs(orc, 2048, 9000, 5)[0], 2048), (random_graph_pairs(300, 900, 4), 300),
                          (np.array([[3, 3], [0, 1], [1, 0]], np.uint32), None)):
        a = orc.build_graph(pairs, n_hint=n_hint, symnorm=symnorm)
        b = ref.build_graph(pairs, n_hint=n_hint, symnorm=symnorm)
        assert a.n == b.n
        assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.neighbors, b.neighbors)
        assert np.array_equal(a.weights.view(np.uint64), b.weights.view(np.uint64))
        assert orc.graph_fingerprint(a) == ref.graph_fingerprint(b)


def test_paths_groups_gs_match(orc, ref):
    for pairs, n_pad, ratio, seed, L in instances(orc):
        g = orc.build_graph(pairs, n_hint=n_pad, symnorm=bool(seed % 2))
        vt = orc.sample_training_set(g.n, ratio, seed)
        assert orc.path_fingerprint(g, vt, L) == ref.path_fingerprint(g, vt, L)
        la = orc.compute_frontiers(g, vt, L)
        lb = ref.compute_frontiers(g, vt, L)
        assert all(np.array_equal(x, y) for x, y in zip(la, lb))
        pa = orc.prepare_all_paths(g, la)
        pb = ref.prepare_all_paths(g, vt, L)
        for x, y in zip(pa, pb):
            for f in PATH_FIELDS:
                assert np.array_equal(getattr(x, f), getattr(y, f)), f
            for gs in (1, 2, 3, 7, max(1, int(np.diff(x.offsets).max(initial=1)))):
                ga, gb = orc.group_neighbors(x.offsets, gs), ref.group_neighbors(y.offsets, gs)
                for f in ("dest", "begin", "end", "dest_groups"):
                    assert np.array_equal(getattr(ga, f), getattr(gb, f))
            cands = orc.default_candidates(int(np.diff(x.offsets).max(initial=0)))
            assert np.array_equal(cands, ref.default_candidates(int(np.diff(x.offsets).max(initial=0))))
            for dim, W, lam in ((16, 8, 0.25), (602, 3, 0.1), (1, 12, 1.0)):
                ba, ta = orc.oracle_gs_cost(x.offsets, cands, dim, W, lam)
                bb, tb = ref.oracle_gs_cost(y.offsets, cands, dim, W, lam)
                assert ba == bb and np.array_equal(ta, tb)


@pytest.mark.parametrize("dim", [1, 3, 16, 41])
def test_aggregate_bit_exact(orc, ref, dim):
    pairs, n_pad = rmat_pairs(orc, 1024, 8192, 7)
    g = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
    vt = orc.sample_training_set(g.n, 0.1, 42)
    for p in orc.prepare_all_paths(g, orc.compute_frontiers(g, vt, 2)):
        x = orc.random_matrix_f32(p.S, dim, 11 + dim)
        a = orc.aggregate_pull_f32(p.offsets, p.neighbors, p.weights, x)
        b, cnt = ref.aggregate_pull(p.offsets, p.neighbors, p.weights, x, gs=5)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        assert cnt[0] == p.E and cnt[1] == len(orc.group_neighbors(p.offsets, 5).dest) and cnt[2] == 0
        # accumulate semantics (aggregate.hpp:50-55)
        a2 = orc.aggregate_pull_f32(p.offsets, p.neighbors, p.weights, x, out=a)
        b2, _ = ref.aggregate_pull(p.offsets, p.neighbors, p.weights, x, gs=5, out=b)
        assert np.array_equal(a2.view(np.uint32), b2.view(np.uint32))
        x64 = x.astype(np.float64)
        c = orc.aggregate_pull_f64(p.offsets, p.neighbors, p.weights, x64)
        d, _ = ref.aggregate_pull(p.offsets, p.neighbors, p.weights, x64, gs=3)
        assert np.array_equal(c.view(np.uint64), d.view(np.uint64))


def test_fast_counters(orc, ref):
    # aggregate.hpp:107-121: Fast counts width atomics per multi-group group
    pairs, n_pad = rmat_pairs(orc, 512, 4096, 7)
    g = orc.build_graph(pairs, n_hint=n_pad)
    x = orc.random_matrix_f32(g.n, 8, 8).astype(np.float64)
    out, cnt = ref.aggregate_pull(g.offsets, g.neighbors, g.weights, x, gs=4, fast=True)
    assert cnt[2] == orc.fast_atomic_commits(g.offsets, 4, 8) > 0
    det = orc.aggregate_pull_f64(g.offsets, g.neighbors, g.weights, x)
    assert np.max(np.abs(out - det) / np.maximum(1, np.maximum(abs(out), abs(det)))) < 1e-12


def test_gemm_a_bt_bit_exact(orc, ref):
    a = orc.random_matrix_f32(301, 16, 1)
    b = orc.random_matrix_f32(602, 16, 2)
    assert np.array_equal(orc.gemm_a_bt_f32(a, b).view(np.uint32), ref.gemm_a_bt(a, b).view(np.uint32))
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    assert np.array_equal(orc.gemm_a_bt_f64(a64, b64).view(np.uint64), ref.gemm_a_bt(a64, b64).view(np.uint64))


def test_chain_restated(orc, ref):
    """The real gradient chain (engine.hpp:316-346) recomposed from oracle
    pieces equals the reference's captured operands bit for bit."""
    pairs, n_pad = rmat_pairs(orc, 1024, 8192, 7)
    g = orc.build_graph(pairs, n_hint=n_pad)
    vt = orc.sample_training_set(g.n, 0.1, 42)
    ch = ref.epp_chain_f32(g, vt, 2, 16, 8, 4, 42)
    lv = ch["levels"]
    paths = orc.prepare_all_paths(g, lv)
    gm = ch["top_g"]
    for i, p in enumerate(paths):
        l = 1 - i
        yg = orc.gemm_a_bt_f32(gm, ch["w"][l])
        assert np.array_equal(yg.view(np.uint32), ch["y_grad"][i].view(np.uint32))
        xg = orc.aggregate_pull_f32(p.offsets, p.neighbors, p.weights, yg[p.srcpos])
        assert np.array_equal(xg.view(np.uint32), ch["x_grad"][i].view(np.uint32))
        if l > 0:
            gm = orc.relu_backward_f32(xg, ch["pre_c"][i])
