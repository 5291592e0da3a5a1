"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and its host-only entry points (input synthesis, gs
regression, candidate lists) agree with the oracle. No device compute."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2204_02662_b200 import _lib


def test_header_symbols_exported():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 40
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), set(declared) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    so = _lib.build()
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_version_and_errors():
    lib = _lib.load()
    assert lib.pg_version() == 2
    h = C.c_void_p()
    # null handles are config errors, reported through pg_last_error
    rc = lib.pg_graph_info(None, None, None, None, None)
    assert rc == 2
    buf = C.create_string_buffer(256)
    lib.pg_last_error(buf, 256)
    assert b"null handle" in buf.value
    line = C.c_uint64(7)
    assert lib.pg_last_error_kind(C.byref(line)) == 1 and line.value == 0  # PG_KIND_CONFIG
    del h


def test_error_kinds_cross_the_abi(tmp_path):
    """pg_last_error_kind carries the exact error.hpp type (no guessing from
    the message text): ParseError with its line number, IoError, ShapeError —
    and a ConfigError whose message mentions "rows" stays a ConfigError."""
    import paper_2204_02662_b200 as pg

    lib = _lib.load()
    bad = tmp_path / "bad.txt"
    bad.write_text("# header\n0 1\n2 x\n")
    with pytest.raises(pg.ParseError) as ei:
        pg.load_edge_list_file(str(bad))
    assert ei.value.line_number == 3 and "(line 3)" in str(ei.value)
    line = C.c_uint64()
    assert lib.pg_last_error_kind(C.byref(line)) == 4 and line.value == 3
    with pytest.raises(pg.IoError):
        pg.load_edge_list_file(str(tmp_path / "missing.txt"))
    assert lib.pg_last_error_kind(None) == 5
    # gemm_a_bt with lda < k: ShapeError (dense_matrix.hpp:80), checked before any device work
    f = C.POINTER(C.c_float)()
    rc = lib.pg_gemm_a_bt(f, 2, f, 4, f, 4, 1, 1, 4, None)
    assert rc == 2 and lib.pg_last_error_kind(None) == 2
    # a ConfigError mentioning "rows": the kind, not the text, decides
    rc = lib.pg_training_set_size(0, 0.5, C.byref(C.c_uint64()))
    assert rc == 2 and lib.pg_last_error_kind(None) == 1


def test_host_generators_match_oracle(orc):
    import paper_2204_02662_b200 as pg

    for n, m, seed in ((1024, 8192, 7), (100, 50, 1)):
        a, na = pg.gen_rmat(n, m, 0.45, 0.22, 0.22, 0.11, seed)
        b, nb = orc.gen_rmat(n, m, 0.45, 0.22, 0.22, 0.11, seed)
        assert na == nb and np.array_equal(a, b)
    for n, ratio, seed in ((1024, 0.1, 42), (232965, 0.66, 42)):
        assert np.array_equal(pg.sample_training_set(n, ratio, seed), orc.sample_training_set(n, ratio, seed))
    with pytest.raises(pg.ConfigError):
        pg.sample_training_set(10, 1.5, 0)
    with pytest.raises(pg.ConfigError):
        pg.gen_rmat(0, 1)


@pytest.mark.parametrize("n,e", [(2708, 5278), (1134890, 2987624), (0, 0), (1, 10**9), (261686, 78511609)])
def test_regression_matches_oracle(orc, n, e):
    import paper_2204_02662_b200 as pg

    avg = 0.0 if n == 0 else e / n
    assert pg.regression_gs(n, e, avg) == orc.regression_gs(n, e, avg)


def test_candidates_match_oracle(orc):
    import paper_2204_02662_b200 as pg

    for md in (0, 1, 4, 5, 214, 52471, 2**31):
        assert np.array_equal(pg.default_gs_candidates(md), orc.default_candidates(md))


def test_tuning_keys(pg):
    """pg_set_tuning: scheduling knobs by name; unknown keys are config errors."""
    for key in ("vec_u", "chunk_major", "heavy_tma", "host_segs", "host_chunks", "host_trace", "heavy_narrow",
                "wide_lpd", "src_segs", "ld_cg", "host_chunk_order", "grouped_seg", "heavy_wide_pipe",
                "host_final_segs", "host_pitch2d", "host_copy_prio", "host_seg_balance",
                "host_chunk_balance", "atb_split", "atb_pairs", "gemm_packed", "host_last_seg_pct", "wgrad_fork",
                "gemm_tc", "rec_window", "src_seg_balance", "host_min_mb", "row_kernel", "row_u", "row_seg_mb",
                "row_heavy", "vec_block", "hub_inline", "hub_front_min", "gemm3_rows", "gemm_beside_wgrad", "host_hub_chunk_side", "vec_window", "host_hub_min", "grouped_src_segs", "narrow_u", "atb_depth",
                "host_first_chunk_pct", "host_seq", "atb_quad",
                "host_small_chunks", "vec8", "f64_hub_min", "grp_dynamic", "vec8_u", "range_side_hubs"):
        pg.set_tuning(key, None)
    import pytest

    with pytest.raises(pg.ConfigError):
        pg.set_tuning("no_such_knob", 1)


def test_compute_fails_loudly_without_gpu(pg):
    """No CPU fallback: on a machine without a usable GPU every compute entry
    point raises DeviceError (status 5) instead of computing on the host."""
    import numpy as np
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(pg.DeviceError):
        pg.build_undirected_csr(np.array([[0, 1], [1, 2]], np.uint32))
    lib = _lib.load()
    out = C.c_void_p()
    offs = np.array([0, 1, 2], np.uint64)
    nbrs = np.array([1, 0], np.uint32)
    w = np.ones(2, np.float64)
    rc = lib.pg_graph_create(0, 2, offs.ctypes.data_as(C.POINTER(C.c_uint64)),
                             nbrs.ctypes.data_as(C.POINTER(C.c_uint32)),
                             w.ctypes.data_as(C.POINTER(C.c_double)), 0, C.byref(out))
    assert rc == 5
