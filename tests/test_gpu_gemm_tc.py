"""Tensor-core gemm_a_bt (dense_matrix.hpp:78-95, y_grad = g W^T):
tcgen05.mma kind::tf32 with 3xTF32 operand splitting (gemm_tc.cu). It
re-associates the K sum, so the gate is the reference's fp32 tolerance
against the exact (f64) product, made conditioning-aware like the SpMM's
(SURVEY §8c): |out - exact| <= 1e-6 + 1e-5 * sum_k |a_ik b_jk| element-wise,
plus a normwise relative error <= 1e-5 and a non-vacuity check. The
bit-exact FFMA2 kernel stays the default (PG_GEMM_TF32X3 off)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(pg, n, m, k, seed, lda_pad=0, ldo_pad=0, scale=1.0):
    import torch

    rng = np.random.default_rng(seed)
    a = (rng.uniform(-1, 1, size=(n, k)) * scale).astype(np.float32)
    b = rng.uniform(-1, 1, size=(m, k)).astype(np.float32)
    lda = (k + 3) // 4 * 4 + lda_pad  # TMA: 16-byte row pitch
    ad = torch.zeros((n, lda), dtype=torch.float32, device="cuda")[:, :k]
    ad.copy_(torch.from_numpy(a))
    bd = torch.from_numpy(b).cuda()
    od = torch.full((n, m + ldo_pad), float("nan"), dtype=torch.float32, device="cuda")[:, :m]
    pg.gemm_a_bt(ad, bd, od, tensor_cores=True)
    torch.cuda.synchronize()
    got = od.cpu().numpy().astype(np.float64)
    exact = a.astype(np.float64) @ b.astype(np.float64).T
    mag = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64).T
    return got, exact, mag


def _gate(got, exact, mag, normwise_ref="exact"):
    """Element-wise |got - exact| <= 1e-6 + 1e-5 sum|a b| (the conditioning-
    aware fp32 bound), plus a normwise relative error <= 1e-5 — relative to
    the exact product, or (normwise_ref="mag", for the 1M-row W' sums whose
    random terms cancel to ~1/1000 of sum|a b|) to the magnitude matrix:
    there the reference's own serial fp32 chain is farther from exact."""
    assert np.isfinite(got).all()
    err = np.abs(got - exact)
    bound = 1e-6 + 1e-5 * mag
    worst = float((err / bound).max()) if err.size else 0.0
    assert (err <= bound).all(), f"worst {worst:.3f} x tolerance"
    ref = exact if normwise_ref == "exact" else mag
    nrm = np.linalg.norm(got - exact) / max(np.linalg.norm(ref), 1e-30)
    assert nrm <= 1e-5, nrm
    assert np.median(np.abs(exact)) >= 100 * 1e-6  # non-vacuous
    return worst


@pytest.mark.parametrize("n,m,k", [(1, 1, 1), (127, 16, 41), (128, 602, 16), (300, 100, 256), (1000, 47, 256),
                                   (513, 256, 47), (4097, 257, 33), (2000, 602, 16), (777, 8, 7), (5000, 130, 100)])
def test_tc_gemm_tolerance(pg, n, m, k):
    got, exact, mag = _case(pg, n, m, k, seed=n * 7 + m + k)
    _gate(got, exact, mag)


def test_tc_gemm_pitched_and_unpadded_output(pg):
    """A with a padded pitch (TMA stride), output with ld = cols = 602 (rows
    not 16-byte aligned: scalar stores) and with a padded ld."""
    for ldo_pad in (0, 6):
        got, exact, mag = _case(pg, 1500, 602, 16, seed=5, lda_pad=4, ldo_pad=ldo_pad)
        _gate(got, exact, mag)


def test_tc_gemm_products_shape(pg):
    """The products-shaped layer-0 product: 2.11M x 256 (g) times 100 x 256
    (W) — the case the tensor cores are for (FP32-pipe bound on CUDA cores)."""
    got, exact, mag = _case(pg, 300_000, 100, 256, seed=11)
    _gate(got, exact, mag)


def test_tc_gemm_rejects_unaligned(pg):
    import torch

    a = torch.zeros((10, 7), dtype=torch.float32, device="cuda")  # ld 7: not 16-byte rows
    b = torch.zeros((5, 7), dtype=torch.float32, device="cuda")
    o = torch.zeros((10, 5), dtype=torch.float32, device="cuda")
    with pytest.raises(pg.ConfigError):
        pg.gemm_a_bt(a, b, o, tensor_cores=True)


def test_chain_with_tc_y_grad_within_tolerance(pg, orc):
    """backward_epp with the tensor-core y_grad (tuning gemm_tc = 1): every
    W' within the fp32 tolerance of the bit-exact chain's (the SpMM and W'
    GEMMs themselves stay exact; only y_grad re-associates)."""
    import torch

    from conftest import rmat_pairs

    pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 16, 3)
    vt = orc.sample_training_set(n_pad, 0.3, 9)
    g = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
    rng = np.random.default_rng(2)
    f, dims = 64, [48, 7]

    def dev(a):
        t = pg.empty_rows(a.shape[0], a.shape[1])
        t.copy_(torch.from_numpy(a))
        return t

    x0 = dev(rng.uniform(0, 1, (g.n, f)).astype(np.float32))
    ws = [dev(rng.uniform(-0.5, 0.5, (f, dims[0])).astype(np.float32)),
          dev(rng.uniform(-0.5, 0.5, (dims[0], dims[1])).astype(np.float32))]
    arts = pg.forward(pg.group_neighbors(g, 4), x0, ws)
    top = dev(rng.uniform(-1, 1, (g.n, dims[1])).astype(np.float32))
    prep = pg.prepare_paths(g, vt, 2, [dims[0], f])
    exact = [w.cpu().numpy().astype(np.float64) for w in pg.backward_epp(prep, arts, top, ws)]
    pg.set_tuning("gemm_tc", 1)
    try:
        tc = [w.cpu().numpy().astype(np.float64) for w in pg.backward_epp(prep, arts, top, ws)]
    finally:
        pg.set_tuning("gemm_tc", None)
    for e, t in zip(exact, tc):
        assert np.linalg.norm(t - e) <= 1e-5 * np.linalg.norm(e)


def _atb_case(pg, n, rows_y, in_dim, out_dim, seed, gathered=True):
    import torch

    rng = np.random.default_rng(seed)
    y = rng.uniform(-1, 1, size=(rows_y, in_dim)).astype(np.float32)
    g = rng.uniform(-1, 1, size=(n, out_dim)).astype(np.float32)
    ids = np.sort(rng.choice(rows_y, size=n, replace=False)).astype(np.int32) if gathered else None
    yd = pg.empty_rows(rows_y, in_dim)
    yd.copy_(torch.from_numpy(y))
    gd = pg.empty_rows(n, out_dim)
    gd.copy_(torch.from_numpy(g))
    od = pg.empty_rows(in_dim, out_dim)
    od.fill_(float("nan"))
    idd = None if ids is None else torch.from_numpy(ids).cuda()
    pg.gemm_at_b(yd, gd, od, a_rows=idd, tensor_cores=True)
    torch.cuda.synchronize()
    ya = (y[ids] if gathered else y).astype(np.float64)
    exact = ya.T @ g.astype(np.float64)
    mag = np.abs(ya).T @ np.abs(g).astype(np.float64)
    return od.cpu().numpy().astype(np.float64), exact, mag


@pytest.mark.parametrize("n,rows_y,in_dim,out_dim", [(7, 9, 33, 5), (1000, 1500, 100, 256), (50_000, 60_000, 602, 16),
                                                     (20_000, 20_000, 16, 41), (5_000, 8_000, 256, 47),
                                                     (40_000, 50_000, 128, 40), (333, 400, 640, 32)])
def test_tc_gemm_at_b_tolerance(pg, n, rows_y, in_dim, out_dim):
    """W' = gather_rows(Y, rows)^T g (dense_matrix.hpp:57-76 + engine.hpp:
    323-324) on the tensor cores: split-K 3xTF32, CTA partials added in a
    fixed order."""
    got, exact, mag = _atb_case(pg, n, rows_y, in_dim, out_dim, seed=n + in_dim)
    _gate(got, exact, mag)


def test_tc_gemm_at_b_products_shape_deterministic(pg):
    """The products layer-0 W' (1.2M gathered rows, 100 x 256): within
    tolerance and bit-identical run to run (no atomics in the reduction)."""
    import torch

    got, exact, mag = _atb_case(pg, 1_198_008, 2_449_029, 100, 256, seed=3)
    _gate(got, exact, mag, normwise_ref="mag")
    got2, _, _ = _atb_case(pg, 1_198_008, 2_449_029, 100, 256, seed=3)
    assert np.array_equal(got.view(np.uint64), got2.view(np.uint64))


def test_tc_gemm_at_b_ungathered_and_empty(pg):
    import torch

    got, exact, mag = _atb_case(pg, 3000, 3000, 50, 20, seed=9, gathered=False)
    _gate(got, exact, mag)
    a = pg.empty_rows(0, 8)
    b = pg.empty_rows(0, 4)
    o = pg.empty_rows(8, 4)
    o.fill_(1.0)
    pg.gemm_at_b(a, b, o, tensor_cores=True)  # no rows: W' = 0
    torch.cuda.synchronize()
    assert (o.cpu().numpy() == 0).all()
