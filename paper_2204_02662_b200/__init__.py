"""paper_2204_02662_b200 — B200-native execution-path backward aggregation
(arXiv 2204.02662), a drop-in for the reference pathgcn's graph load,
execution-path build, group partition and backward aggregate.

The compute lives in libpathgcn_b200.so (sm_100a CUDA behind the C ABI in
include/pathgcn_b200.h); ``pathgcn`` mirrors the reference operator API.
"""
from . import _lib
from .pathgcn import *  # noqa: F401,F403

__all__ = [n for n in dir() if not n.startswith("_")]


def build(force: bool = False):
    """Compile libpathgcn_b200.so for sm_100a (in-tree)."""
    return _lib.build(force=force)
