import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a path)")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built (reference tree absent at build time)")
    return Ref()


@pytest.fixture(scope="session")
def pg():
    """The product package; on a GPU box the CUDA path must load (no fallback)."""
    import paper_2204_02662_b200 as pkg

    pkg._lib.load()
    return pkg


@pytest.fixture(scope="session")
def cuda():
    import torch

    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    return torch.device("cuda:0")


# ---- reference fixtures (proj/tests/unit/fixtures.hpp) as edge lists ----

GEX_PAIRS = np.array([[0, 1], [1, 2], [1, 3], [1, 4], [2, 3], [3, 4]], np.uint32)  # fixtures.hpp:19-25
GEX_VT = np.array([2, 4], np.uint32)  # fixtures.hpp:28-33


def star_pairs(leaves):
    """fixtures.hpp:36-42"""
    return np.array([[0, i] for i in range(1, leaves + 1)], np.uint32)


def rmat_pairs(orc, n, m, seed):
    """fixtures.hpp:44-57 (a,b,c,d = .45/.22/.22/.11)."""
    pairs, n_pad = orc.gen_rmat(n, m, 0.45, 0.22, 0.22, 0.11, seed)
    return pairs, n_pad


def random_graph_pairs(n, m, seed):
    """fixtures.hpp:60-73 — uniform_int_distribution<VertexId>(0, n-1) pairs."""
    import ctypes as C

    from oracle.oracle import Oracle

    st = Oracle().L  # the oracle's restated mt19937_64 + uniform_int_distribution
    st.orc_mt64_seed.argtypes = [C.c_void_p, C.c_uint64]
    st.orc_uniform_int.restype = C.c_uint64
    st.orc_uniform_int.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
    rng = C.create_string_buffer(8 * 313)  # orc_mt64
    st.orc_mt64_seed(rng, seed)
    out = []
    for _ in range(m):
        u = st.orc_uniform_int(rng, 0, n - 1)
        v = st.orc_uniform_int(rng, 0, n - 1)
        if u != v:
            out.append((u, v))
    if not out:
        out.append((0, n - 1))
    return np.array(out, np.uint32)
