"""Shared by tests/golden/make_fullsize_digests.py (run here, against the
REFERENCE compiled from /root/reference) and tests/test_gpu_fullsize.py (run
on the B200): the exact inputs of the benchmarked configs and the digest
format. Test infrastructure only.

Digest of an array: SHA-256 of its little-endian C-order bytes (float arrays
as their bit patterns), plus the SHA-256 of each of CHUNKS equal row blocks
so a mismatch names the rows that differ."""
import hashlib
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CHUNKS = 32
CONFIGS = ("reddit", "products", "arxiv", "pubmed", "cora")


def digest_path(config):
    return os.path.join(HERE, f"fullsize_{config}.json")


def y_grad(P, dim, i):
    """The stage input of path i: bench.grad_input (U(-1,1) fp32, P x dim),
    the same bytes on both sides and in the benchmark."""
    import bench

    return bench.grad_input(P, dim, i)


def _bytes(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8).reshape(-1) if a.size else np.zeros(0, np.uint8)


def digest(a):
    a = np.ascontiguousarray(a)
    out = {"dtype": str(a.dtype), "shape": list(a.shape), "sha256": hashlib.sha256(_bytes(a)).hexdigest()}
    n = a.shape[0] if a.ndim else 0
    if n >= CHUNKS:
        cuts = [n * k // CHUNKS for k in range(CHUNKS + 1)]
        out["chunks"] = [hashlib.sha256(_bytes(a[cuts[k]:cuts[k + 1]])).hexdigest()[:16] for k in range(CHUNKS)]
    return out


def compare(name, want, got_arr):
    """None when equal, else a message naming the first differing row block."""
    d = digest(got_arr)
    if d["dtype"] != want["dtype"] or d["shape"] != want["shape"]:
        return f"{name}: dtype/shape {d['dtype']}{d['shape']} != {want['dtype']}{want['shape']}"
    if d["sha256"] == want["sha256"]:
        return None
    bad = [k for k, (a, b) in enumerate(zip(d.get("chunks", []), want.get("chunks", []))) if a != b]
    n = d["shape"][0] if d["shape"] else 0
    rows = [(n * k // CHUNKS, n * (k + 1) // CHUNKS) for k in bad[:4]]
    return f"{name}: digest differs (row blocks {rows}{' ...' if len(bad) > 4 else ''} of {n})"
