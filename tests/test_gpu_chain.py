"""GPU parity of the GCN chain around the backward aggregation (SURVEY
§8f rank 1-3): forward, top_grad_from_probs, backward_epp (Local, fused
relu epilogue and unfused; Global), backward_all_active and backward_ifelse
on the device, bit-exact against the oracle (which tests/test_chain_oracle.py
pins to the reference's engine.hpp)."""
import os

import numpy as np
import pytest

from test_chain_oracle import CASES, chain_inputs, oracle_chain, same
from conftest import rmat_pairs

pytestmark = pytest.mark.gpu


def dev(torch, pg, a):
    t = pg.empty_rows(a.shape[0], a.shape[1])
    t.copy_(torch.from_numpy(np.ascontiguousarray(a, np.float32)))
    return t


def host(t):
    return t.cpu().numpy()


def gpu_setup(pg, orc, case):
    import torch

    n_req, m, seed, ratio, L, f, hidden, classes, symnorm = case
    g_o, vt, x0, ws, r = chain_inputs(orc, n_req, m, seed, ratio, L, f, hidden, classes, symnorm)
    pairs, n_pad = rmat_pairs(orc, n_req, m, seed)
    g = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm" if symnorm else "unit")
    assert g.n == g_o.n and g.m == g_o.m
    Gg = pg.group_neighbors(g, 4)
    agg = [([f] + [hidden] * (L - 1))[L - 1 - i] for i in range(L)]
    prep = pg.prepare_paths(g, vt, L, agg, gs_strategy=("fixed", 2))
    d = dict(x0=dev(torch, pg, x0), ws=[dev(torch, pg, w) for w in ws], r=dev(torch, pg, r),
             vt=torch.from_numpy(vt.astype(np.int32)).cuda())
    return g_o, vt, x0, ws, r, g, Gg, prep, d


@pytest.mark.parametrize("case", CASES)
def test_forward_and_top_grad(pg, orc, cuda, case):
    import torch

    g_o, vt, x0, ws, r, g, Gg, prep, d = gpu_setup(pg, orc, case)
    arts = pg.forward(Gg, d["x0"], d["ws"])
    top = pg.empty_rows(g.n, ws[-1].shape[1])
    pg.top_grad_from_probs(arts.x[-1], d["r"], d["vt"], top)
    torch.cuda.synchronize()
    want = orc.forward(g_o, x0, ws)
    for l in range(len(ws)):
        assert same(host(arts.y[l]), want["y"][l]), f"Y^({l})"
        assert same(host(arts.pre_act[l]), want["pre"][l]), f"pre^({l})"
        assert same(host(arts.x[l + 1]), want["x"][l + 1]), f"X^({l + 1}) (relu / softmax)"
    assert same(host(top), orc.top_grad_f32(want["x"][-1], r, vt))


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_backward_variants(pg, orc, cuda, case, mode):
    import torch

    g_o, vt, x0, ws, r, g, Gg, prep, d = gpu_setup(pg, orc, case)
    L = len(ws)
    arts = pg.forward(Gg, d["x0"], d["ws"])
    top = pg.empty_rows(g.n, ws[-1].shape[1])
    pg.top_grad_from_probs(arts.x[-1], d["r"], d["vt"], top)
    c = {}
    if mode == 0:
        wg = pg.backward_all_active(Gg, arts, top, d["ws"], counters=c)
    elif mode == 1:
        wg = pg.backward_ifelse(Gg, prep.frontiers, arts, top, d["ws"], counters=c)
    else:
        wg = pg.backward_epp(prep, arts, top, d["ws"], gather="local" if mode == 2 else "global", counters=c)
    torch.cuda.synchronize()
    _, _, want_wg, _, want_edges = oracle_chain(orc, g_o, vt, x0, ws, r, mode)
    for l in range(L):
        assert same(host(wg[l]), want_wg[l]), f"W^({l})' mode {mode}"
    assert c["backward_edges_per_layer"] == want_edges


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_backward_x_grads_unfused(pg, orc, cuda, mode):
    """x_grads_out forces the unfused SpMM + relu_backward; same W' and the
    captured X' match the oracle."""
    import torch

    case = CASES[0]
    g_o, vt, x0, ws, r, g, Gg, prep, d = gpu_setup(pg, orc, case)
    L = len(ws)
    arts = pg.forward(Gg, d["x0"], d["ws"])
    top = pg.empty_rows(g.n, ws[-1].shape[1])
    pg.top_grad_from_probs(arts.x[-1], d["r"], d["vt"], top)
    xs = []
    if mode == 0:
        wg = pg.backward_all_active(Gg, arts, top, d["ws"], x_grads_out=xs)
    elif mode == 1:
        wg = pg.backward_ifelse(Gg, prep.frontiers, arts, top, d["ws"], x_grads_out=xs)
    else:
        wg = pg.backward_epp(prep, arts, top, d["ws"], x_grads_out=xs)
    torch.cuda.synchronize()
    _, _, want_wg, want_xg, _ = oracle_chain(orc, g_o, vt, x0, ws, r, mode)
    for l in range(L):
        assert same(host(wg[l]), want_wg[l])
    for i in range(L):
        assert same(host(xs[i]), want_xg[i]), f"X' path {i}"


def test_stale_paths_rejected(pg, orc, cuda):
    case = CASES[0]
    g_o, vt, x0, ws, r, g, Gg, prep, d = gpu_setup(pg, orc, case)
    arts = pg.forward(Gg, d["x0"], d["ws"])
    top = pg.empty_rows(g.n, ws[-1].shape[1])
    pg.top_grad_from_probs(arts.x[-1], d["r"], d["vt"], top)
    with pytest.raises(pg.ConfigError, match="stale"):
        pg.backward_epp(prep, arts, top, d["ws"], expected_fingerprint=prep.fingerprint ^ 1)
    with pytest.raises(pg.ConfigError, match="layer count|depth"):
        pg.backward_epp(prep, arts, top, d["ws"][:1] * 3)


def test_dense_kernels(pg, orc, cuda):
    import torch

    rng = np.random.default_rng(5)
    for packed in (2, 1, 0):  # k_gemm3 (8x8 register tiles), k_gemm2 (FFMA2/FADD2 column pairs), k_gemm
        pg.set_tuning("gemm_packed", packed)
        try:
            for n, k, m in ((1, 1, 1), (37, 602, 16), (300, 16, 41), (65, 33, 130), (129, 35, 63), (200, 7, 100),
                            (70, 5, 33), (257, 47, 256), (130, 256, 100), (128, 32, 128), (383, 19, 602),
                            (64, 3, 129)):
                a = rng.uniform(-1, 1, (n, k)).astype(np.float32)
                b = rng.uniform(-1, 1, (k, m)).astype(np.float32)
                a[0, : min(2, k)] = [0.0, -0.0][: min(2, k)]
                out = pg.empty_rows(n, m)
                pg.gemm(dev(torch, pg, a), dev(torch, pg, b), out)
                assert same(host(out), orc.gemm_f32(a, b)), (packed, n, k, m)
                # op(B) = B^T (gemm_a_bt), unpadded operands
                bt = np.ascontiguousarray(b.T)
                out = pg.empty_rows(n, m)
                pg.gemm_a_bt(torch.from_numpy(a).cuda(), torch.from_numpy(bt).cuda(), out)
                assert same(host(out), orc.gemm_f32(a, b)), ("a_bt", packed, n, k, m)
        finally:
            pg.set_tuning("gemm_packed", None)
    # both W' kernels (copy warp + chain warp, one warp); n around the
    # 64-row stage edges and the 4-slot ring; odd widths take the 4-byte copies
    for split, pairs in ((1, None), (0, None), (1, 1)):  # (1, 1): two A columns per lane everywhere
        pg.set_tuning("atb_split", split)
        pg.set_tuning("atb_pairs", pairs)
        try:
            for n, r_, c in ((1, 1, 1), (1000, 602, 16), (777, 16, 41), (5, 3, 2), (64, 9, 7), (257, 8, 5),
                             (4 * 64 + 1, 20, 33)):
                a = rng.uniform(-1, 1, (n, r_)).astype(np.float32)
                b = rng.uniform(-1, 1, (n, c)).astype(np.float32)
                out = pg.empty_rows(r_, c)
                pg.gemm_at_b(dev(torch, pg, a), dev(torch, pg, b), out)
                assert same(host(out), orc.gemm_at_b_f32(a, b)), (split, n, r_, c)
                # fused row gather
                big = rng.uniform(-1, 1, (n * 2, r_)).astype(np.float32)
                rows = np.sort(rng.choice(n * 2, n, replace=False)).astype(np.int32)
                out = pg.empty_rows(r_, c)
                pg.gemm_at_b(dev(torch, pg, big), dev(torch, pg, b), out, a_rows=torch.from_numpy(rows).cuda())
                assert same(host(out), orc.gemm_at_b_f32(big[rows], b)), (split, n, r_, c)
                # unpadded operands (ld = cols, rows not 16-byte aligned): the 4-byte copy path
                out = pg.empty_rows(r_, c)
                pg.gemm_at_b(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), out)
                assert same(host(out), orc.gemm_at_b_f32(a, b)), ("unpadded", split, n, r_, c)
        finally:
            pg.set_tuning("atb_split", None)
            pg.set_tuning("atb_pairs", None)
    x = rng.uniform(-2, 2, (513, 47)).astype(np.float32)
    x[0, :3] = [0.0, -0.0, np.float32(1e-40)]
    out = pg.empty_rows(*x.shape)
    pg.relu(dev(torch, pg, x), out)
    assert same(host(out), orc.relu_f32(x))
    # past 32768 rows: each thread takes 8 rows per step (the last step partial)
    x = rng.uniform(-2, 2, (32768 * 8 + 32768 * 3 + 5, 21)).astype(np.float32)
    out = pg.empty_rows(*x.shape)
    pg.relu(dev(torch, pg, x), out)
    assert same(host(out), orc.relu_f32(x))


def test_row_softmax_bit_exact(pg, orc, cuda):
    """expf emulation == glibc expf: wide-range logits incl. underflow; the
    shared-memory-tiled kernel (<= 95 columns, a partial last tile of rows)
    and the thread-per-row one past it."""
    import torch

    rng = np.random.default_rng(9)
    for cols, scale in ((41, 1.0), (7, 30.0), (3, 200.0), (47, 0.01), (1, 5.0), (95, 3.0), (96, 3.0),
                        (130, 1.0)):
        x = (rng.standard_normal((4099, cols)) * scale).astype(np.float32)
        out = pg.empty_rows(*x.shape)
        pg.row_softmax(dev(torch, pg, x), out)
        torch.cuda.synchronize()
        assert same(host(out), orc.row_softmax_f32(x)), (cols, scale)


def test_aggregate_pull_filtered(pg, orc, cuda):
    import torch

    case = CASES[0]
    g_o, vt, x0, ws, r, g, Gg, prep, d = gpu_setup(pg, orc, case)
    levels = orc.compute_frontiers(g_o, vt, 2)
    for dim in (16, 37, 602):
        y = np.random.default_rng(dim).uniform(-1, 1, (g.n, dim)).astype(np.float32)
        for dl, sl in ((1, 0), (2, 1), (2, 0)):
            out = pg.empty_rows(g.n, dim)
            out.zero_()
            c = {}
            pg.aggregate_pull_filtered(Gg, prep.frontiers, dl, sl, dev(torch, pg, y), out, counters=c)
            da = np.zeros(g.n, np.uint8)
            da[levels[dl]] = 1
            sa = np.zeros(g.n, np.uint8)
            sa[levels[sl]] = 1
            want, wc = orc.aggregate_pull_filtered_f32(g_o.offsets, g_o.neighbors, g_o.weights, y, da, sa, 4)
            assert same(host(out), want), (dim, dl, sl)
            assert c == wc


def test_filtered_unaligned_rows_scalar_path(pg, orc, cuda):
    """aggregate_pull_filtered on rows whose pitch is not a multiple of 4
    floats (the scalar kernel) — same bits as the oracle."""
    import torch

    case = CASES[0]
    g_o, vt, x0, ws, r, g, Gg, prep, d = gpu_setup(pg, orc, case)
    levels = orc.compute_frontiers(g_o, vt, 2)
    dim = 7
    y = np.random.default_rng(3).uniform(-1, 1, (g.n, dim)).astype(np.float32)
    yd = torch.from_numpy(y).cuda()  # ld = 7: unaligned rows
    out = torch.zeros((g.n, dim), dtype=torch.float32, device="cuda")
    c = {}
    pg.aggregate_pull_filtered(Gg, prep.frontiers, 2, 1, yd, out, counters=c)
    da = np.zeros(g.n, np.uint8)
    da[levels[2]] = 1
    sa = np.zeros(g.n, np.uint8)
    sa[levels[1]] = 1
    want, wc = orc.aggregate_pull_filtered_f32(g_o.offsets, g_o.neighbors, g_o.weights, y, da, sa, 4)
    assert same(host(out), want) and c == wc


@pytest.mark.parametrize("seed", range(int(os.environ.get("PG_STRESS_SEEDS_CHAIN", "16"))))
def test_random_chains(pg, orc, cuda, seed):
    """Random depths / widths / training fractions, knob settings of the
    chain GEMMs (W' copy-warp or one-warp kernel, two A columns per lane,
    packed or scalar y_grad GEMM): forward + every backward variant's W'
    bit-exact with the oracle's composition of the reference."""
    import torch

    rng = np.random.default_rng(77 + seed)
    L = int(rng.integers(1, 4))
    f, hidden, classes = (int(rng.choice(v)) for v in ((3, 17, 64, 130), (4, 16, 33), (2, 7, 41)))
    hidden = hidden if L > 1 else 0
    n_req = int(rng.integers(200, 3000))
    case = (n_req, n_req * int(rng.choice([3, 8, 20])), 90 + seed, float(rng.choice([0.05, 0.3, 1.0])), L, f,
            hidden, classes, bool(seed % 2))
    knobs = {"atb_split": int(rng.integers(0, 2)), "atb_pairs": int(rng.choice([1, 224])),
             "atb_depth": int(rng.integers(0, 3)), "atb_quad": int(rng.integers(0, 4)),
             "gemm_packed": int(rng.integers(0, 3)), "wgrad_fork": int(rng.integers(0, 2)),
             "gemm3_rows": int(rng.choice([8, 16])), "gemm_beside_wgrad": int(rng.integers(0, 2)),
             "vec8": int(rng.integers(0, 3))}
    try:
        for k, v in knobs.items():
            pg.set_tuning(k, v)
        g_o, vt, x0, ws, r, g, Gg, prep, d = gpu_setup(pg, orc, case)
        arts = pg.forward(Gg, d["x0"], d["ws"])
        top = pg.empty_rows(g.n, ws[-1].shape[1])
        pg.top_grad_from_probs(arts.x[-1], d["r"], d["vt"], top)
        for mode in (0, 2, 3):
            if mode == 0:
                wg = pg.backward_all_active(Gg, arts, top, d["ws"])
            else:
                wg = pg.backward_epp(prep, arts, top, d["ws"], gather="local" if mode == 2 else "global")
            torch.cuda.synchronize()
            _, _, want_wg, _, _ = oracle_chain(orc, g_o, vt, x0, ws, r, mode)
            for l in range(L):
                assert same(host(wg[l]), want_wg[l]), (seed, mode, l, knobs, case)
    finally:
        for k in knobs:
            pg.set_tuning(k, None)


@pytest.mark.parametrize("rows, cols", [(1, 1), (1000, 602), (233, 16), (4097, 41), (300, 128), (0, 5)])
def test_mat_upload_download(pg, cuda, rows, cols):
    """pg_mat_upload / pg_mat_download (the C++ DeviceMatrix::upload /
    download): a host DenseMatrix (ld = cols) to a pitched device matrix and
    back in one flat copy + repack, bit-exact, padding untouched."""
    import ctypes as C
    import time

    import torch

    from paper_2204_02662_b200 import _lib
    from paper_2204_02662_b200.pathgcn import _mat

    lib = _lib.load()
    rng = np.random.default_rng(rows * 7 + cols)
    h = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
    d = pg.empty_rows(rows, cols)
    full = d.as_strided((rows, d.stride(0)), (d.stride(0), 1)) if rows else None
    if rows:
        full.fill_(7.0)
    fp = C.POINTER(C.c_float)
    t = time.perf_counter()
    assert lib.pg_mat_upload(0, _mat(d, "d"), h.ctypes.data_as(fp)) == 0
    up_ms = (time.perf_counter() - t) * 1e3
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy().view(np.uint32), h.view(np.uint32))
    if rows and d.stride(0) > cols:
        assert (full[:, cols:].cpu().numpy() == 7.0).all()  # pitch padding untouched
    back = np.full((rows, cols), np.nan, np.float32)
    assert lib.pg_mat_download(0, back.ctypes.data_as(fp), _mat(d, "d")) == 0
    assert np.array_equal(back.view(np.uint32), h.view(np.uint32))
    assert up_ms < 1000  # one copy, not one per row
